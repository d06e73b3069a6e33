"""render_scene (R20) on the GPU vs the oracle:
several objects of a room, per-pixel segments sorted by t_near, composited front
to back over black.  Tolerance as the single-object render (BASELINE north_star:
<= 1e-4 abs on rendered colour / opacity, fp32 path)."""
import numpy as np
import pytest

import oracle as O
import scenes
from gpu_common import make_pair

pytestmark = pytest.mark.gpu

R = pytest.importorskip("paper_2304_05735_b200.romap")

CFG0 = dict(levels=8, log2_T=12, base_res=16, finest_res=2048.0, res_cap=128, samples_per_ray=32,
            rays_per_iter=128, precision=0, seed=4)


@pytest.fixture(scope="module")
def ctx():
    c = R.Context(0)
    yield c
    c.close()


def _scene_objects(ctx, sc, n):
    hs, objs = [], []
    for k, ob in enumerate(sc.objects[:n]):
        h, st = make_pair(R, ctx, sc, CFG0, param_seed=20 + k, inst=ob.instance_id, obj_id=200 + k,
                          avoid_kinks=False)
        hs.append(h)
        objs.append((st.cfg, st.box_t, st.box_yaw, st.box_a, st.params, h))
    return hs, objs


def test_render_scene_three_objects():
    c = R.Context(0)
    sc = scenes.room_scene(5, n_objects=3, n_frames=6, W=96, H=72, f=78.75, room_half=1.5)
    hs, objs = _scene_objects(c, sc, 3)
    fr = sc.frames[0]
    W, H, N = 96, 72, 16
    rgb, dep, opa = c.render_scene(list(reversed(hs)), fr.T_wc, fr.K, W, H, N)   # order of the list is irrelevant
    orgb, odep, oopa = O.render_scene(objs, fr.T_wc, fr.K, W, H, N)
    assert np.abs(rgb - orgb).max() < 1e-4
    assert np.abs(opa - oopa).max() < 1e-4
    assert np.abs(dep - odep).max() < 3e-4
    # several objects really overlap in the image (the sort matters)
    hits = np.zeros((H, W), int)
    for (_, bt, yaw, ba, params, oid) in objs:
        _, _, o = O.render(objs[0][0], bt, yaw, ba, params, fr.T_wc, fr.K, W, H, N)
        hits += o > 0
    assert (hits >= 1).sum() > 200
    # one object: render_scene == render (opacity comes back as 1 - (1 - A): 1 ulp)
    r1, d1, a1 = c.render_scene([hs[1]], fr.T_wc, fr.K, W, H, N)
    r2, d2, a2 = c.render(hs[1], fr.T_wc, fr.K, W, H, N)
    assert np.array_equal(r1, r2) and np.array_equal(d1, d2)
    assert np.abs(a1 - a2).max() < 1e-6
    # errors: unknown object, duplicate, bad sample count
    with pytest.raises(R.RomapError):
        c.render_scene([hs[0], 12345], fr.T_wc, fr.K, W, H, N)
    with pytest.raises(R.RomapError):
        c.render_scene([hs[0], hs[0]], fr.T_wc, fr.K, W, H, N)
    with pytest.raises(R.RomapError):
        c.render_scene(hs, fr.T_wc, fr.K, W, H, 0)
    c.close()


def test_render_scene_camera_inside_and_miss():
    # a pose looking away from every box: all-black, zero opacity, zero depth
    c = R.Context(0)
    sc = scenes.room_scene(5, n_objects=2, n_frames=6, W=64, H=48, f=52.5, room_half=1.5)
    hs, objs = _scene_objects(c, sc, 2)
    T = np.array([[1, 0, 0, 0], [0, 0, 1, 0], [0, -1, 0, 50.0]], np.float32)   # 50 m above, looking up
    K = (52.5, 52.5, 32.0, 24.0)
    rgb, dep, opa = c.render_scene(hs, T, K, 64, 48, 8)
    assert not rgb.any() and not dep.any() and not opa.any()
    orgb, odep, oopa = O.render_scene(objs, T, K, 64, 48, 8)
    assert not orgb.any() and not oopa.any()
    c.close()


def test_render_scene_batched_mixed_and_fp32_groups():
    """the batched path with three model groups in one scene (4 mixed-precision
    objects of the BASELINE network, one of the paper's network with 2 hidden layers,
    R24, and one fp32 object: one forward launch per group, segments of all objects in one
    composite), a sample count that is not a power of two (object ranges padded to
    128-sample tile boundaries), against the oracle: hit pixels identical (bit-exact
    geometry), colour / opacity within the mixed path's 2e-2 (fp32-only pixels 1e-4)"""
    c = R.Context(0)
    sc = scenes.room_scene(8, n_objects=6, n_frames=6, W=120, H=90, f=98.4, room_half=1.8)
    hs, objs = [], []
    for k, ob in enumerate(sc.objects[:6]):
        kw = dict(CFG0, precision=0 if k == 2 else 1)
        if k == 4:
            kw.update(network=1, hidden_layers=2)
        h, st = make_pair(R, c, sc, kw, param_seed=30 + k, inst=ob.instance_id, obj_id=600 + k, avoid_kinks=False)
        hs.append(h)
        objs.append((st.cfg, st.box_t, st.box_yaw, st.box_a, st.params, h))
    W, H, N = 120, 90, 24
    # every group is on screen in some frame (the paper-network object included)
    for k in (2, 4):
        cf, bt, yaw, ba, params, _ = objs[k]
        assert any(O.render(cf, bt, yaw, ba, params, fr.T_wc, fr.K, W, H, N)[2].max() > 0 for fr in sc.frames[:3]), k
    for fr in sc.frames[:3]:
        rgb, dep, opa = c.render_scene(hs, fr.T_wc, fr.K, W, H, N)
        orgb, odep, oopa = O.render_scene(objs, fr.T_wc, fr.K, W, H, N)
        assert np.array_equal(opa > 0, oopa > 0)
        assert np.abs(rgb - orgb).max() < 2e-2 and np.abs(opa - oopa).max() < 2e-2
    # the fp32 object alone through the batched path keeps the fp32 tolerance
    r1, d1, a1 = c.render_scene([hs[2]], sc.frames[0].T_wc, sc.frames[0].K, W, H, N)
    o1 = O.render_scene([objs[2]], sc.frames[0].T_wc, sc.frames[0].K, W, H, N)
    assert np.abs(r1 - o1[0]).max() < 1e-4 and np.abs(a1 - o1[2]).max() < 1e-4
    c.close()
