"""The paper's network (R24: hash encoding + 1..3
hidden layers of 64 -> sigma, rgb; positions only) on the mixed GPU path vs the
oracle: per-block gradients within 2e-2 norm-relative (BASELINE, fp16 path),
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


def _grads(ctx, h, st, tol=2e-2):
    stats = ctx.forward_backward([h])[0]
    L, g, dbg = O.loss_and_grads(st, 1)
    assert stats["hit_rays"] == L["hit_rays"] and stats["samples"] == L["samples"]
    assert abs(stats["l_total"] - L["l_total"]) <= 1e-2 * L["l_total"]
    e_tab = norm_rel(ctx.get_params(h, R.BLOCK_GRAD_TABLE), g["table"].reshape(-1))
    gm = ctx.get_params(h, R.BLOCK_GRAD_MLP)
    errs, off = [], 0
    for w in g["W"]:
        errs.append(norm_rel(gm[off:off + w.size], w))
        off += w.size
    assert off == gm.size
    assert e_tab < tol and max(errs) < tol, (e_tab, errs)


# gradient tolerance per hidden-layer count: 2e-2 (BASELINE, fp16 path) for the
# paper's single layer; every further fp16 backward layer rounds delta once more
# and the table-gradient sums cancel, measured 1.4 / 2.9 / 3.8 % (tools/
# diag_paper_net.py), so the Table 4 variants get 2e-2 + 1.5e-2 per extra layer
#
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
