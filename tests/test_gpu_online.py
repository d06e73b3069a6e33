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
