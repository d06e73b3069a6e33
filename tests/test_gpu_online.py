"""f3 online policy (R25) through the C ABI: the
Eq. 5 keyframe gate decides exactly as the oracle, accepted frames add 300
pending iterations, and the scheduler trains the objects with budget left in
batched launches exactly as the oracle's schedule says, stopping objects whose
budget is spent."""
import numpy as np
import pytest

import oracle as O
import scenes

pytestmark = pytest.mark.gpu

R = pytest.importorskip("paper_2304_05735_b200.romap")

CFG = dict(levels=8, log2_T=12, base_res=16, finest_res=2048.0, res_cap=128, samples_per_ray=32, rays_per_iter=128,
           precision=1, seed=2)


def test_gate_budget_and_scheduler():
    c = R.Context(0)
    sc = scenes.room_scene(7, n_objects=2, n_frames=24, W=160, H=120, f=131.25, room_half=1.5)
    hs, expect = [], {}
    for k, ob in enumerate(sc.objects[:2]):
        h = c.create_object(ob.t, ob.yaw, ob.a, R.model_config(**CFG), ob.instance_id, obj_id=500 + k)
        hs.append(h)
        last, n_acc = None, 0
        stride = 1 + k                       # object 1 sees every other frame: fewer keyframes
        for fr in sc.frames[::stride]:
            if not (fr.mask == ob.instance_id).any():
                continue
            acc, alpha = c.offer_observation(h, fr.rgb, fr.mask, fr.T_wc, fr.K, alpha_deg=25.0)
            ok, oalpha = O.keyframe_gate(last, fr.T_wc, np.asarray(ob.t, np.float64), 25.0)
            assert acc == ok, (k, alpha, oalpha)
            if oalpha is not None:
                assert alpha == pytest.approx(oalpha, abs=1e-3)
            if ok:
                last = O.camera_centre(fr.T_wc)
                n_acc += 1
        assert n_acc >= 2
        assert c.pending_iters(h) == 300 * n_acc
        expect[h] = 300 * n_acc
    # scheduler: batched chunks exactly as the oracle's schedule, capped per call
    batches, rest = O.schedule_budgets(expect, chunk=100, max_iters=250)
    ran = c.train_pending(chunk=100, max_iters=250)
    want = {}
    for objs, n in batches:
        for o in objs:
            want[o] = want.get(o, 0) + n
    assert ran == want
    for h in hs:
        assert c.pending_iters(h) == rest[h]
        assert int(c.get_params(h, R.BLOCK_STEP)[0]) == want[h]        # Adam steps taken
    # the rest: objects stop when their budget is spent
    ran2 = c.train_pending(chunk=100)
    for h in hs:
        assert c.pending_iters(h) == 0
        assert ran2.get(h, 0) == rest[h]
    assert c.train_pending(chunk=100) == {}
    # a repeated view is rejected and adds nothing
    fr = sc.frames[0]
    for h, ob in zip(hs, sc.objects[:2]):
        if (fr.mask == ob.instance_id).any():
            acc, _ = c.offer_observation(h, fr.rgb, fr.mask, fr.T_wc, fr.K)
            assert c.pending_iters(h) == (300 if acc else 0)
    c.close()


def test_set_box_matches_oracle():
    """f3 box update: parameters stay in normalized box coordinates (R6), so after
    romap_set_box the rays, samples and losses follow the new box exactly as the
    oracle with the same box; bad boxes are rejected without side effects."""
    from gpu_common import make_pair, norm_rel
    c = R.Context(0)
    sc = scenes.sphere_scene(0, n_views=8)
    kw = dict(CFG, rays_per_iter=256)
    h, st = make_pair(R, c, sc, kw)
    for _ in range(3):
        s = c.train_step([h], 1)[0]
        o, _, _ = O.train_iteration(st)
    ob = sc.objects[0]
    t2 = np.asarray(ob.t, np.float64) + [0.05, -0.03, 0.02]
    yaw2 = float(ob.yaw) + 0.2
    a2 = np.asarray(ob.a, np.float64) * 1.15
    with pytest.raises(R.RomapError):
        c.set_box(h, t2, yaw2, [a2[0], -1.0, a2[2]])
    c.set_box(h, t2, yaw2, a2)
    st.box_t = np.asarray(t2, np.float32)
    st.box_yaw = float(np.float32(yaw2))
    st.box_a = np.asarray(a2, np.float32)
    # gradients at identical parameters: the oracle takes the GPU's current ones
    # (3 mixed-precision Adam steps leave them slightly apart)
    W = c.get_params(h, R.BLOCK_MLP).astype(np.float64)
    Ws, off = [], 0
    for w in st.params["W"]:
        Ws.append(W[off:off + w.size].reshape(w.shape))
        off += w.size
    st.params = {"table": c.get_params(h, R.BLOCK_TABLE).reshape(-1, 2).astype(np.float64), "W": Ws}
    s = c.forward_backward([h])[0]
    L, g, dbg = O.loss_and_grads(st, 4)              # the 4th iteration's rays (3 steps taken)
    for k in ("l_total", "l_rgb", "l_rr", "l_density"):
        assert abs(s[k] - L[k]) <= 1e-2 * max(abs(L[k]), 1e-4), (k, s[k], L[k])
    assert s["hit_rays"] == L["hit_rays"] and s["samples"] == L["samples"]
    gt = c.get_params(h, R.BLOCK_GRAD_TABLE).reshape(-1, 2)
    assert norm_rel(gt, g["table"]) < 2e-2
    # training continues on the new box and tracks the oracle
    for _ in range(3):
        s = c.train_step([h], 1)[0]
        o, _, _ = O.train_iteration(st)
        assert abs(s["l_total"] - o["l_total"]) <= 5e-2 * o["l_total"], (s, o)
    c.close()


def test_all_rays_miss_after_box_moves_away():
    """Degenerate batch: the box moved behind every camera, so no ray hits it.
    The fused step must see zero hit rays, produce zero losses and gradients
    without non-finite values, and Adam must still apply the dense MLP update
    with zero gradients (momentum) exactly like the oracle,
    leaving the sparse table untouched."""
    from gpu_common import make_pair, norm_rel
    c = R.Context(0)
    sc = scenes.sphere_scene(0, n_views=8)
    kw = dict(CFG, rays_per_iter=256)
    h, st = make_pair(R, c, sc, kw)
    for _ in range(2):
        c.train_step([h], 1)
        O.train_iteration(st)
    t_far = np.asarray(sc.objects[0].t, np.float64) + [0.0, 0.0, 50.0]
    c.set_box(h, t_far, sc.objects[0].yaw, sc.objects[0].a)
    st.box_t = np.asarray(t_far, np.float32)
    table0 = c.get_params(h, R.BLOCK_TABLE).copy()
    for _ in range(2):
        s = c.train_step([h], 1)[0]
        o, _, _ = O.train_iteration(st)
        assert s["hit_rays"] == o["hit_rays"] == 0
        assert s["samples"] == 0 and s["l_total"] == 0.0
    assert s["step"] == 4
    assert np.array_equal(c.get_params(h, R.BLOCK_TABLE), table0)    # sparse: untouched
    W = c.get_params(h, R.BLOCK_MLP).astype(np.float64)
    Wo = np.concatenate([w.reshape(-1) for w in st.params["W"]])
    assert norm_rel(W, Wo) < 5e-2                                      # momentum steps as the oracle
    c.close()


def test_scheduler_with_two_model_configurations():
    """R25 scheduler over objects of different model configurations (one batched
    train_step per configuration per round, the round length n = min(chunk,
    smallest pending) over ALL objects with budget): per-object iteration counts and
    Adam steps follow the oracle's schedule, and each object trained in its group
    equals the same object trained alone (deterministic mode, bitwise)."""
    sc = scenes.room_scene(7, n_objects=3, n_frames=24, W=160, H=120, f=131.25, room_half=1.5)
    cfgs = [dict(CFG), dict(CFG), dict(CFG, seed=9, precision=0)]     # groups {0, 1} and {2}
    budgets = [130, 70, 100]

    def setup(c, ks):
        hs = {}
        for k in ks:
            ob = sc.objects[k]
            h = c.create_object(ob.t, ob.yaw, ob.a, R.model_config(**cfgs[k]), ob.instance_id, obj_id=700 + k)
            fr = [f for f in sc.frames if (f.mask == ob.instance_id).any()][0]
            acc, _ = c.offer_observation(h, fr.rgb, fr.mask, fr.T_wc, fr.K, iters_per_update=budgets[k])
            assert acc
            hs[k] = h
        return hs

    c = R.Context(0)
    c.set_deterministic(True)
    hs = setup(c, range(3))
    batches, rest = O.schedule_budgets({hs[k]: budgets[k] for k in range(3)}, chunk=40, max_iters=1000)
    ran = c.train_pending(chunk=40)
    assert ran == {hs[k]: budgets[k] for k in range(3)} and all(v == 0 for v in rest.values())
    assert len(batches) > 2
    got = {k: (c.get_params(hs[k], R.BLOCK_TABLE).copy(), int(c.get_params(hs[k], R.BLOCK_STEP)[0])) for k in range(3)}
    c.close()
    for k in range(3):
        assert got[k][1] == budgets[k]
        # alone: the same iterations in the same chunk lengths as the schedule gave it
        a = R.Context(0)
        a.set_deterministic(True)
        h = setup(a, [k])[k]
        for objs, n in batches:
            if hs[k] in objs:
                a.train_step([h], n)
        assert np.array_equal(a.get_params(h, R.BLOCK_TABLE).view(np.uint32), got[k][0].view(np.uint32)), k
        a.close()
