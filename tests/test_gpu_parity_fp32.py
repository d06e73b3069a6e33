"""GPU (CUDA path through the C ABI) vs CPU oracle, fp32 path (BASELINE cfg0).

Tolerances (BASELINE north_star / DESIGN.md "Tolerances"): bit-exact pixels,
classes, rays, segments, sample distances, normalized positions and hash
indices; features <= 1e-6 of the table scale; field (sigma, rgb) <= 1e-5 rel;
losses <= 1e-5 rel; gradients <= 1e-4 norm-relative per parameter block;
rendered colour / opacity <= 1e-4 abs.
"""
import numpy as np
import pytest

import oracle as O
import scenes
from gpu_common import flat_W, make_pair, norm_rel

pytestmark = pytest.mark.gpu

from paper_2304_05735_b200 import romap as R  # noqa: E402  (fails loudly if the library is missing)

CFG0 = dict(levels=8, log2_T=12, base_res=16, finest_res=2048.0, res_cap=128, samples_per_ray=32, rays_per_iter=256,
            precision=0, seed=0)


@pytest.fixture(scope="module")
def ctx():
    c = R.Context(0)
    yield c
    c.close()


@pytest.fixture(scope="module")
def scene0():
    return scenes.sphere_scene(0, depth_per_view=2)


def _fwdbwd(ctx, scene, kw, **k):
    h, st = make_pair(R, ctx, scene, kw, **k)
    stats = ctx.forward_backward([h])[0]
    L, g, dbg = O.loss_and_grads(st, 1)
    return h, st, stats, L, g, dbg


def _check_rays(ctx, h, dbg):
    rd = ctx.debug_dump(h, R.DUMP_RAYS)
    rs = dbg["rays"]
    assert np.array_equal(rd["kf"], rs["k"])
    assert np.array_equal(rd["px"], rs["px"]) and np.array_equal(rd["py"], rs["py"])
    assert np.array_equal(rd["cls"], rs["cls"])
    assert np.array_equal(rd["hit"].astype(bool), rs["hit"])
    assert np.array_equal(rd["has_depth"].astype(bool), rs["has_depth"])
    for a, b in [("o", "o"), ("d", "d"), ("t_near", "tn"), ("t_far", "tf"), ("target", "tgt"), ("bg", "bg"),
                 ("depth", "depth_t")]:
        assert np.array_equal(rd[a].view(np.uint32), np.asarray(rs[b], np.float32).view(np.uint32)), a
    return rd


def _check_samples(ctx, h, st, dbg):
    N = st.cfg.samples_per_ray
    rs = dbg["rays"]
    hit = rs["hit"]
    sd = ctx.debug_dump(h, R.DUMP_SAMPLES).reshape(rs["R"], N, 5)
    assert np.array_equal(sd[hit, :, 0].view(np.uint32), rs["dist"][hit].view(np.uint32))
    assert np.array_equal(sd[hit, :, 1].view(np.uint32), rs["delta"][hit].view(np.uint32))
    assert np.array_equal(sd[hit, :, 2:].view(np.uint32), rs["u"][hit].view(np.uint32))
    hi = ctx.debug_dump(h, R.DUMP_HASH_IDX).reshape(rs["R"], N, st.cfg.levels, 8)
    assert np.array_equal(hi[hit].reshape(-1, st.cfg.levels, 8), dbg["idx"])


def test_cfg0_rays_samples_hash_bit_exact(ctx, scene0):
    h, st, stats, L, g, dbg = _fwdbwd(ctx, scene0, CFG0)
    rd = _check_rays(ctx, h, dbg)
    assert rd["has_depth"].sum() > 0                      # the parity fixture carries sparse depth
    _check_samples(ctx, h, st, dbg)
    ctx.destroy_object(h)


def test_cfg0_features_field_loss_grads(ctx, scene0):
    h, st, stats, L, g, dbg = _fwdbwd(ctx, scene0, CFG0)
    N = st.cfg.samples_per_ray
    hit = dbg["rays"]["hit"]
    R_ = dbg["rays"]["R"]
    fe = ctx.debug_dump(h, R.DUMP_FEATURES).reshape(R_, N, -1)[hit].reshape(-1, 16)
    assert np.abs(fe - dbg["feat"]).max() <= 1e-6 * 0.1 * 8
    fl = ctx.debug_dump(h, R.DUMP_FIELD).reshape(R_, N, 4)[hit].reshape(-1, 4)
    assert np.allclose(fl[:, 0], dbg["fw"]["sigma"], rtol=1e-5, atol=1e-7)
    assert np.allclose(fl[:, 1:], dbg["fw"]["rgb"], rtol=1e-5, atol=1e-7)
    for k in ("l_rgb", "l_rr", "l_depth", "l_density", "l_total"):
        assert abs(stats[k] - L[k]) <= 1e-5 * max(abs(L[k]), 1e-6), (k, stats[k], L[k])
    assert stats["hit_rays"] == L["hit_rays"] and stats["samples"] == L["samples"]
    rg = ctx.debug_dump(h, R.DUMP_RAY_GRADS).reshape(R_, N, 4)[hit]
    assert norm_rel(rg[..., 0], dbg["dsigma"]) < 1e-4
    assert norm_rel(rg[..., 1:], dbg["drgb"]) < 1e-4
    gt = ctx.get_params(h, R.BLOCK_GRAD_TABLE).reshape(-1, 2)
    assert norm_rel(gt, g["table"]) < 1e-4
    gm = ctx.get_params(h, R.BLOCK_GRAD_MLP)
    off = 0
    for w in g["W"]:
        assert norm_rel(gm[off:off + w.size], w) < 1e-4
        off += w.size
    # untouched entries received exactly zero gradient
    assert np.array_equal(gt == 0, g["table"] == 0)
    ctx.destroy_object(h)


def test_cfg0_render_64(ctx, scene0):
    h, st = make_pair(R, ctx, scene0, CFG0)
    fr = scene0.frames[0]
    rgb, dep, opa = ctx.render(h, fr.T_wc, fr.K, 64, 64, 32)
    orgb, odep, oopa = O.render(st.cfg, st.box_t, st.box_yaw, st.box_a, st.params, fr.T_wc, fr.K, 64, 64, 32)
    assert np.abs(rgb - orgb).max() < 1e-4
    assert np.abs(opa - oopa).max() < 1e-4
    assert np.abs(dep - odep).max() < 1e-4 * 3.0
    assert (oopa > 0.1).sum() > 100
    ctx.destroy_object(h)


def test_cfg0_query_density(ctx, scene0):
    h, st = make_pair(R, ctx, scene0, CFG0)
    g = np.random.default_rng(3)
    pts = g.uniform(-0.6, 0.6, (5000, 3)).astype(np.float32)
    pts[:10] = [[0.5, 0.5, 0.5], [-0.5, -0.5, -0.5], [0.5, 0, 0], [0.50001, 0, 0], [0, 0, 0], [0, -0.5, 0.2],
                [0.6, 0.6, 0.6], [-0.5, 0.49, 0.3], [0.1, 0.2, 0.3], [0.25, -0.25, 0.125]]
    s = ctx.query_density(h, pts)
    so = O.query_density(st.cfg, st.box_a, st.params, pts)
    assert np.array_equal(s == 0, so == 0)
    assert np.allclose(s, so, rtol=1e-5, atol=1e-7)
    assert ctx.query_density(h, np.zeros((0, 3), np.float32)).shape == (0,)
    ctx.destroy_object(h)


def test_adam_on_identical_gradients(ctx, scene0):
    h, st = make_pair(R, ctx, scene0, CFG0)
    g = np.random.default_rng(9)
    ne = O.table_entries(st.cfg)
    for t in range(1, 4):
        gt = np.zeros((ne, 2), np.float32)
        pick = g.choice(ne, size=ne // 3, replace=False)
        gt[pick] = g.normal(0, 1e-3, (pick.size, 2)).astype(np.float32)
        gw = [g.normal(0, 1e-2, w.shape).astype(np.float32) for w in st.params["W"]]
        if t > 1:                                # the MLP is dense (R18): exact zeros still move p, m, v
            for w in gw:
                w[g.random(w.shape) < 0.2] = 0.0
        ctx.set_params(h, R.BLOCK_GRAD_TABLE, gt)
        ctx.set_params(h, R.BLOCK_GRAD_MLP, flat_W(gw))
        ctx.optimizer_step([h])
        O.adam_update(st.params["table"], gt.astype(np.float64), st.m["table"], st.v["table"], t, st.cfg, sparse=True)
        for k in range(5):
            O.adam_update(st.params["W"][k], gw[k].astype(np.float64), st.m["W"][k], st.v["W"][k], t, st.cfg, sparse=False)
    p = ctx.get_params(h, R.BLOCK_TABLE).reshape(-1, 2)
    m = ctx.get_params(h, R.BLOCK_M_TABLE).reshape(-1, 2)
    v = ctx.get_params(h, R.BLOCK_V_TABLE).reshape(-1, 2)
    # fp32 Adam: each of the t updates rounds at |p| ~ 0.1 -> absolute error ~ t * ulp(0.1)
    assert np.allclose(p, st.params["table"], rtol=1e-6, atol=3e-8)
    # fp32 moments: relative 1e-5, with an absolute floor of ~1e-6 of the size of the
    # terms being summed (m ~ (1-b1)|g| ~ 1e-4, v ~ (1-b2) g^2 ~ 1e-8) for cancellations
    for name, a, b, floor in (("m", m, st.m["table"], 1e-10), ("v", v, st.v["table"], 1e-14)):
        err = np.abs(a - b) / (np.abs(b) + floor / 1e-5)
        i = np.unravel_index(err.argmax(), err.shape)
        assert err.max() < 1e-5, (name, i, a[i], b[i], gt[i])
    untouched = (st.m["table"] == 0)
    assert np.all(m[untouched] == 0) and np.all(v[untouched] == 0)
    pm = ctx.get_params(h, R.BLOCK_MLP)
    assert np.allclose(pm, flat_W(st.params["W"]), rtol=1e-6, atol=3e-8)
    # MLP moments (g ~ 1e-2: m ~ 1e-3, v ~ 1e-7), absolute floors ~1e-6 of those for cancellations
    assert np.allclose(ctx.get_params(h, R.BLOCK_M_MLP), flat_W(st.m["W"]), rtol=1e-5, atol=1e-9)
    assert np.allclose(ctx.get_params(h, R.BLOCK_V_MLP), flat_W(st.v["W"]), rtol=1e-5, atol=1e-13)
    assert ctx.get_params(h, R.BLOCK_STEP)[0] == 3
    assert np.all(ctx.get_params(h, R.BLOCK_GRAD_TABLE) == 0)
    ctx.destroy_object(h)


def test_cfg0_five_training_steps(ctx, scene0):
    h, st = make_pair(R, ctx, scene0, CFG0)
    for it in range(5):
        s = ctx.train_step([h], 1)[0]
        o, _, _ = O.train_iteration(st)
        assert abs(s["l_total"] - o["l_total"]) <= 1e-3 * abs(o["l_total"]), (it, s, o)
        assert s["step"] == it + 1
    ctx.destroy_object(h)


def test_cfg0d_dense_levels_and_ragged(ctx, scene0):
    # cfg0 with T = 2^16: levels 16 and 32 become dense (17^3, 33^3 <= 65536); 77 rays (ragged tail)
    kw = dict(CFG0, log2_T=16, rays_per_iter=77)
    h, st, stats, L, g, dbg = _fwdbwd(ctx, scene0, kw)
    assert ctx.object_info(h)["n_dense_levels"] == 2
    _check_rays(ctx, h, dbg)
    _check_samples(ctx, h, st, dbg)
    assert abs(stats["l_total"] - L["l_total"]) <= 1e-5 * L["l_total"]
    assert norm_rel(ctx.get_params(h, R.BLOCK_GRAD_TABLE).reshape(-1, 2), g["table"]) < 1e-4
    assert norm_rel(ctx.get_params(h, R.BLOCK_GRAD_MLP), flat_W(g["W"])) < 1e-4
    ctx.destroy_object(h)


def test_cfg1_shape_fp32_several_tiles(ctx):
    # BASELINE cfg1 grid (L=16, T=2^16, 16->512, N=64) on a small object scene,
    # 301 rays = 151 tiles of 2 rays incl. a ragged tail, with occluders absent
    sc = scenes.object_scene(1, n_views=20, W=160, H=120, f=131.25, depth_per_view=8)   # >16 keyframes: table growth
    kw = dict(levels=16, log2_T=16, base_res=16, finest_res=512.0, res_cap=0, samples_per_ray=64,
              rays_per_iter=301, precision=0, seed=1)
    h, st, stats, L, g, dbg = _fwdbwd(ctx, sc, kw)
    _check_rays(ctx, h, dbg)
    _check_samples(ctx, h, st, dbg)
    assert abs(stats["l_total"] - L["l_total"]) <= 1e-5 * L["l_total"]
    assert norm_rel(ctx.get_params(h, R.BLOCK_GRAD_TABLE).reshape(-1, 2), g["table"]) < 1e-4
    gm = ctx.get_params(h, R.BLOCK_GRAD_MLP)
    off = 0
    for w in g["W"]:
        assert norm_rel(gm[off:off + w.size], w) < 1e-4
        off += w.size
    ctx.destroy_object(h)


def test_occluders_and_multi_object_batch(ctx):
    # two objects of a room trained together == each alone; occluder rays dropped
    sc = scenes.room_scene(4, n_objects=3, n_frames=6, W=160, H=120, f=131.25, room_half=1.5)
    kw = dict(CFG0, rays_per_iter=128, seed=4)
    ids = [o.instance_id for o in sc.objects[:2]]
    hs, sts = [], []
    for k, iid in enumerate(ids):
        h, st = make_pair(R, ctx, sc, kw, param_seed=10 + k, inst=iid, obj_id=100 + k)
        hs.append(h)
        sts.append(st)
    stats = ctx.forward_backward(hs)
    for k in range(2):
        L, g, dbg = O.loss_and_grads(sts[k], 1)
        _check_rays(ctx, hs[k], dbg)
        assert abs(stats[k]["l_total"] - L["l_total"]) <= 1e-5 * L["l_total"]
        assert norm_rel(ctx.get_params(hs[k], R.BLOCK_GRAD_MLP), flat_W(g["W"])) < 1e-4
    # alone
    alone = ctx.forward_backward([hs[1]])[0]
    assert abs(alone["l_total"] - stats[1]["l_total"]) <= 1e-6 * stats[1]["l_total"]
    for h in hs:
        ctx.destroy_object(h)


def test_error_paths(ctx, scene0):
    ob = scene0.objects[0]
    with pytest.raises(R.RomapError) as e:
        ctx.create_object(ob.t, 0.0, ob.a, R.model_config(feats=4), 1)
    assert e.value.status == R.E_INVALID
    with pytest.raises(R.RomapError) as e:
        ctx.create_object(ob.t, 0.0, [0.5, 0.0, 0.5], R.model_config(), 1)
    assert e.value.status == R.E_INVALID
    with pytest.raises(R.RomapError) as e:
        ctx.create_object(ob.t, 0.0, ob.a, R.model_config(samples_per_ray=48), 1)
    assert e.value.status == R.E_INVALID
    h1 = ctx.create_object(ob.t, 0.0, ob.a, R.model_config(), 1)
    h2 = ctx.create_object(ob.t, 0.0, ob.a, R.model_config(log2_T=14), 1)
    with pytest.raises(R.RomapError) as e:
        ctx.train_step([h1], 1)
    assert e.value.status == R.E_STATE
    fr = scene0.frames[0]
    ctx.add_observation(h1, fr.rgb, fr.mask, fr.T_wc, fr.K)
    ctx.add_observation(h2, fr.rgb, fr.mask, fr.T_wc, fr.K)
    with pytest.raises(R.RomapError) as e:
        ctx.train_step([h1, h2], 1)
    assert e.value.status == R.E_CONFIG_MISMATCH
    with pytest.raises(R.RomapError) as e:
        ctx.train_step([12345], 1)
    assert e.value.status == R.E_NOT_FOUND
    with pytest.raises(R.RomapError) as e:
        ctx.add_observation(h1, fr.rgb, np.zeros_like(fr.mask), fr.T_wc, fr.K)
    assert e.value.status == R.E_INVALID
    with pytest.raises(R.RomapError) as e:
        ctx.set_params(h1, R.BLOCK_TABLE, np.zeros(7, np.float32))
    assert e.value.status == R.E_INVALID
    assert ctx.object_info(h1)["n_keyframes"] == 1
    ctx.train_step([h1], 2)
    assert ctx.object_info(h1)["step"] == 2
    ctx.destroy_object(h1)
    ctx.destroy_object(h2)


def test_fp32_deterministic_batch_equals_alone_and_oracle():
    """fp32 path in the deterministic-reduction mode (romap_set_deterministic): the
    gradients of two room objects computed in one batch equal each object's alone
    bit for bit, a rerun is bitwise identical, and the result keeps
    the fp32 tolerance against the oracle (1e-4 norm-relative per block)"""
    c = R.Context(0)
    c.set_deterministic(True)
    sc = scenes.room_scene(4, n_objects=3, n_frames=6, W=160, H=120, f=131.25, room_half=1.5)
    kw = dict(CFG0, rays_per_iter=128, seed=4)
    hs, sts = [], []
    for k, ob in enumerate(sc.objects[:2]):
        h, st = make_pair(R, c, sc, kw, param_seed=10 + k, inst=ob.instance_id, obj_id=100 + k)
        hs.append(h)
        sts.append(st)
    grads = lambda h: (c.get_params(h, R.BLOCK_GRAD_TABLE), c.get_params(h, R.BLOCK_GRAD_MLP))
    sb = c.forward_backward(hs)
    gb = [grads(h) for h in hs]
    for k in range(2):
        L, g, _ = O.loss_and_grads(sts[k], 1)
        assert abs(sb[k]["l_total"] - L["l_total"]) <= 1e-5 * L["l_total"]
        assert norm_rel(gb[k][0].reshape(-1, 2), g["table"]) < 1e-4
        assert norm_rel(gb[k][1], flat_W(g["W"])) < 1e-4
    for k in range(2):
        sa = c.forward_backward([hs[k]])[0]
        ga = grads(hs[k])
        assert sa["l_total"] == sb[k]["l_total"] and sa["l_rgb"] == sb[k]["l_rgb"]
        assert np.array_equal(ga[0].view(np.uint32), gb[k][0].view(np.uint32))
        assert np.array_equal(ga[1].view(np.uint32), gb[k][1].view(np.uint32))
    c.close()
