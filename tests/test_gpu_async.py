"""f3 asynchronous online trainer (R25): frames offered
while the worker trains are queued without waiting for the GPU, every frame goes
through the Eq. 5 gate exactly as in the synchronous path, and stopping with
finish_pending trains every accepted frame's 300 iterations."""
import time

import numpy as np
import pytest

import oracle as O
import scenes

pytestmark = pytest.mark.gpu

R = pytest.importorskip("paper_2304_05735_b200.romap")

CFG = dict(levels=8, log2_T=12, base_res=16, finest_res=2048.0, res_cap=128, samples_per_ray=32, rays_per_iter=256,
           precision=1, seed=3)


def test_async_producer_never_blocks_and_trains_everything():
    c = R.Context(0)
    sc = scenes.room_scene(7, n_objects=2, n_frames=24, W=160, H=120, f=131.25, room_half=1.5)
    objs = sc.objects[:2]
    hs = [c.create_object(ob.t, ob.yaw, ob.a, R.model_config(**CFG), ob.instance_id, obj_id=700 + k)
          for k, ob in enumerate(objs)]
    # the oracle's gate decisions for the same frame stream
    expect = {}
    for h, ob in zip(hs, objs):
        last, n = None, 0
        for fr in sc.frames:
            if (fr.mask == ob.instance_id).any():
                ok, _ = O.keyframe_gate(last, fr.T_wc, np.asarray(ob.t, np.float64), 25.0)
                if ok:
                    last, n = O.camera_centre(fr.T_wc), n + 1
        expect[h] = n
    c.async_start(chunk=50, queue_cap=256)
    with pytest.raises(R.RomapError):              # the worker owns the context
        c.train_step(hs, 1)
    worst = 0.0
    for fr in sc.frames:
        for h, ob in zip(hs, objs):
            if (fr.mask == ob.instance_id).any():
                t0 = time.perf_counter()
                assert c.async_offer(h, fr.rgb, fr.mask, fr.T_wc, fr.K)
                worst = max(worst, time.perf_counter() - t0)
        time.sleep(0.002)                          # frames arrive while training runs
    st = c.async_stop(finish_pending=True)
    assert st["dropped"] == 0 and st["accepted"] == sum(expect.values())
    assert worst < 0.05, worst                     # a queue push, not a training step
    for h in hs:
        assert c.pending_iters(h) == 0
        assert int(c.get_params(h, R.BLOCK_STEP)[0]) == 300 * expect[h]
    c.close()


def test_async_queue_full_drops_without_blocking():
    c = R.Context(0)
    sc = scenes.sphere_scene(0, n_views=8)
    ob = sc.objects[0]
    h = c.create_object(ob.t, ob.yaw, ob.a, R.model_config(**CFG), ob.instance_id)
    c.async_start(chunk=50, queue_cap=2)
    res = [c.async_offer(h, fr.rgb, fr.mask, fr.T_wc, fr.K) for fr in sc.frames * 4]
    st = c.async_stop(finish_pending=False)
    assert st["offered"] == len(res) and st["dropped"] == res.count(False)
    c.close()


def test_async_bad_frames_are_rejected_and_the_worker_goes_on():
    """a frame for an unknown object, or one whose mask does not contain the
    instance, is rejected (counted) and changes nothing; the worker keeps taking
    and training the good frames"""
    c = R.Context(0)
    sc = scenes.sphere_scene(0, n_views=8)
    ob = sc.objects[0]
    h = c.create_object(ob.t, ob.yaw, ob.a, R.model_config(**CFG), ob.instance_id)
    c.async_start(chunk=50, queue_cap=64)
    fr0 = sc.frames[0]
    assert c.async_offer(h + 77, fr0.rgb, fr0.mask, fr0.T_wc, fr0.K)             # unknown object
    assert c.async_offer(h, fr0.rgb, np.zeros_like(fr0.mask), fr0.T_wc, fr0.K)   # instance not visible
    for fr in sc.frames:
        assert c.async_offer(h, fr.rgb, fr.mask, fr.T_wc, fr.K)
    st = c.async_stop(finish_pending=True)
    assert st["rejected"] == 2 and st["accepted"] >= 1
    assert c.object_info(h)["n_keyframes"] == st["accepted"]
    assert int(c.get_params(h, R.BLOCK_STEP)[0]) == 300 * st["accepted"]
    c.close()
