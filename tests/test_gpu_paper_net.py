"""The paper's network (R24: hash encoding + 1..3
hidden layers of 64 -> sigma, rgb; positions only) on the mixed GPU path vs the
oracle: per-block gradients within 2e-2 norm-relative of fp64 (BASELINE, fp16
path; the 2- and 3-layer Table 4 variants: see GRAD_TOL), every block and every
hash level within 1e-2 of the fp16 precision model (tests/mixed_model.py),
losses within 1e-2, a few training steps, density query and render."""
import numpy as np
import pytest

import oracle as O
import scenes
from gpu_common import flat_W, make_pair, norm_rel

pytestmark = pytest.mark.gpu

R = pytest.importorskip("paper_2304_05735_b200.romap")

SMALL = dict(levels=8, log2_T=12, base_res=16, finest_res=2048.0, res_cap=128, samples_per_ray=32, rays_per_iter=256,
             precision=1, seed=3, network=1)
# T = 2^16, N_max = 2048, 4096 rays x N = 32, single hidden layer of 64
PAPER = dict(levels=16, log2_T=16, base_res=16, finest_res=2048.0, res_cap=0, samples_per_ray=32, rays_per_iter=4096,
             precision=1, seed=1, network=1, hidden_layers=1)


@pytest.fixture(scope="module")
def ctx():
    c = R.Context(0)
    yield c
    c.close()


# GPU vs the fp16 model: both round at the same points, but fp32 (GPU) and fp64
# (model) accumulation still move a few pre-activations across a ReLU kink or an
# fp16 rounding boundary, and one flipped unit of one sample shifts a coarse level's
# cancelling sum by up to ~0.7 % (measured, N = 16); a wrong corner index or
# scatter on a level moves that level by O(1)
MODEL_TOL = 1e-2


def _grads(ctx, h, st, tol=2e-2):
    import mixed_model
    stats = ctx.forward_backward([h])[0]
    L, g, dbg = O.loss_and_grads(st, 1)
    assert stats["hit_rays"] == L["hit_rays"] and stats["samples"] == L["samples"]
    assert abs(stats["l_total"] - L["l_total"]) <= 1e-2 * L["l_total"]
    gt = ctx.get_params(h, R.BLOCK_GRAD_TABLE).reshape(-1, 2)
    e_tab = norm_rel(gt, g["table"])
    gm = ctx.get_params(h, R.BLOCK_GRAD_MLP)
    _, gmod = mixed_model.mixed_loss_and_grads(st, 1)
    errs, e_mod, off = [], [], 0
    for w, wm in zip(g["W"], gmod["W"]):
        errs.append(norm_rel(gm[off:off + w.size], w))
        e_mod.append(norm_rel(gm[off:off + w.size], wm))
        off += w.size
    assert off == gm.size
    e_mod += [norm_rel(gt[l.offset:l.offset + l.size], gmod["table"][l.offset:l.offset + l.size])
              for l in O.level_table(st.cfg)]
    assert e_tab < tol and max(errs) < tol, (e_tab, errs)
    assert max(e_mod) < MODEL_TOL, e_mod


# gradient tolerance against fp64 per hidden-layer count: 2e-2 (BASELINE, fp16
# path) for the paper's single layer.  The Table 4 variants with 2 / 3 hidden
# layers are an explicit deviation from north_star's 2e-2:
# the fp16 precision model (tests/mixed_model.py) puts the fp64 gap of the table
# gradient at 1.0-1.1 % / 2.0-2.1 % / 2.5-2.7 % for 1 / 2 / 3 layers with the
# backward deltas exact (rounding the deltas adds < 0.05 %): it comes from the fp16
# FORWARD operands (features, weights, activations) through the deeper ReLU chain,
# so fp32 deltas cannot close it.  The kernel itself is held to the model (1e-2).
GRAD_TOL = {1: 2e-2, 2: 3.5e-2, 3: 5e-2}


@pytest.mark.parametrize("hl", [1, 2, 3])
def test_paper_net_grads_query_render(ctx, hl):
    sc = scenes.sphere_scene(0, depth_per_view=2)
    h, st = make_pair(R, ctx, sc, dict(SMALL, hidden_layers=hl), avoid_kinks=False)
    assert len(st.params["W"]) == hl + 1
    _grads(ctx, h, st, GRAD_TOL[hl])
    # density query: sigma of the whole MLP within the fp16 tolerance
    pts = np.random.default_rng(4).uniform(-0.6, 0.6, (8000, 3)).astype(np.float32)
    s = ctx.query_density(h, pts)
    so = O.query_density(st.cfg, st.box_a, st.params, pts)
    assert np.array_equal(s == 0, so == 0)
    ins = so != 0
    assert np.abs(s[ins] / so[ins] - 1).max() < 2e-2
    # render (midpoints, over black)
    fr = sc.frames[1]
    rgb, dep, opa = ctx.render(h, fr.T_wc, fr.K, 48, 48, 32)
    orgb, odep, oopa = O.render(st.cfg, st.box_t, st.box_yaw, st.box_a, st.params, fr.T_wc, fr.K, 48, 48, 32)
    assert np.abs(rgb - orgb).max() < 2e-2 and np.abs(opa - oopa).max() < 2e-2
    ctx.optimizer_step([h])
    ctx.destroy_object(h)


def test_paper_net_training_tracks_oracle(ctx):
    sc = scenes.sphere_scene(0)
    h, st = make_pair(R, ctx, sc, dict(SMALL, hidden_layers=2), param_seed=9, avoid_kinks=False)
    for it in range(8):
        s = ctx.train_step([h], 1)[0]
        o, _, _ = O.train_iteration(st)
        assert abs(s["l_total"] - o["l_total"]) <= 5e-2 * o["l_total"], (it, s, o)
    ctx.destroy_object(h)


def test_paper_net_full_size_grads(ctx):
    # the paper's configuration at full size in bench.py --network paper's launch configuration
    sc = scenes.object_scene(1, n_views=20)
    h, st = make_pair(R, ctx, sc, PAPER, avoid_kinks=False)
    _grads(ctx, h, st)
    ctx.destroy_object(h)


def test_paper_net_rejects_fp32_and_bad_layers(ctx):
    with pytest.raises(R.RomapError):
        ctx.create_object([0, 0, 0], 0.0, [1, 1, 1], R.model_config(network=1, precision=0), 1)
    with pytest.raises(R.RomapError):
        ctx.create_object([0, 0, 0], 0.0, [1, 1, 1], R.model_config(network=1, precision=1, hidden_layers=4), 1)


def test_paper_net_largest_table_grads(ctx):
    """Table 4's largest table (T = 2^20: 16 levels of up to 1 M
    entries, 64 MB fp16 / 128 MB fp32) on a ragged batch (777 rays x 32): geometry
    bit-exact (the fused kernel's corner entries), every block within the fp64
    tolerance and every level within the fp16 model's"""
    sc = scenes.sphere_scene(0, depth_per_view=2)
    kw = dict(PAPER, log2_T=20, rays_per_iter=777)
    h, st = make_pair(R, ctx, sc, kw, avoid_kinks=False)
    _grads(ctx, h, st)
    rs = O.forward_rays(st, 1)
    _, idx, _ = O.hash_encode(rs["u"][rs["hit"]].reshape(-1, 3), st.params["table"], st.cfg)
    gi = ctx.debug_dump(h, R.DUMP_HASH_IDX).reshape(777, 32, 16, 8)[rs["hit"]].reshape(-1, 16, 8)
    assert np.array_equal(gi.astype(np.int64), idx)
    ctx.destroy_object(h)
