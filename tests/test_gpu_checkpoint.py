"""Checkpoint / resume (romap_save_object / romap_load_object):
an object saved after some training and loaded into a fresh context continues
EXACTLY like the original (deterministic-reduction mode: bitwise losses,
parameters and Adam moments), keeps its keyframes, step and online-policy budget;
bad files are rejected without side effects."""
import os

import numpy as np
import pytest

import scenes

pytestmark = pytest.mark.gpu

R = pytest.importorskip("paper_2304_05735_b200.romap")

CFG = dict(levels=8, log2_T=12, base_res=16, finest_res=2048.0, res_cap=128, samples_per_ray=32, rays_per_iter=256,
           precision=1, seed=5)
BLOCKS = (R.BLOCK_TABLE, R.BLOCK_MLP, R.BLOCK_M_TABLE, R.BLOCK_M_MLP, R.BLOCK_V_TABLE, R.BLOCK_V_MLP, R.BLOCK_STEP)


VARIANTS = {"mixed": {}, "fp32": dict(precision=0), "paper net, 2 layers": dict(network=1, hidden_layers=2),
            "softplus, obj_bg=1": dict(density_act=1, obj_bg=1, lambda_density=0.03)}


@pytest.mark.parametrize("variant", list(VARIANTS))
def test_save_load_resume_bitwise(tmp_path, variant):
    sc = scenes.sphere_scene(0, n_views=8, depth_per_view=2)
    ob = sc.objects[0]
    a = R.Context(0)
    a.set_deterministic(True)
    h = a.create_object(ob.t, ob.yaw, ob.a, R.model_config(**dict(CFG, **VARIANTS[variant])), ob.instance_id,
                        obj_id=41)
    for fr in sc.frames[:6]:
        a.add_observation(h, fr.rgb, fr.mask, fr.T_wc, fr.K, fr.depth.get(ob.instance_id))
    fr = sc.frames[6]
    acc, _ = a.offer_observation(h, fr.rgb, fr.mask, fr.T_wc, fr.K, alpha_deg=1.0, iters_per_update=77)
    assert acc
    a.train_step([h], 20)
    a.set_box(h, [ob.t[0] + 0.01, ob.t[1], ob.t[2]], ob.yaw + 0.02, [x * 1.05 for x in ob.a])   # R27: the box round-trips
    a.train_step([h], 3)
    path = str(tmp_path / "obj41.romap")
    a.save_object(h, path)
    b = R.Context(0)
    b.set_deterministic(True)
    h2 = b.load_object(path)
    assert h2 == 41
    ia, ib = a.object_info(h), b.object_info(h2)
    assert ia == ib
    assert a.pending_iters(h) == b.pending_iters(h2) == 77
    for blk in BLOCKS:
        assert np.array_equal(a.get_params(h, blk), b.get_params(h2, blk))
    sa = a.train_step([h], 17)[0]
    sb = b.train_step([h2], 17)[0]
    for k in ("l_total", "l_rgb", "l_rr", "l_depth", "l_density", "hit_rays", "step"):
        assert sa[k] == sb[k], (k, sa[k], sb[k])
    for blk in BLOCKS:
        x, y = a.get_params(h, blk), b.get_params(h2, blk)
        assert np.array_equal(x.view(np.uint8), y.view(np.uint8)), blk
    # under another id in the same context; an existing id and bad files are rejected
    h3 = a.load_object(path, obj_id=99)
    assert h3 == 99 and a.object_info(h3)["n_keyframes"] == ia["n_keyframes"]
    with pytest.raises(R.RomapError):
        a.load_object(path, obj_id=99)
    bad = tmp_path / "bad.romap"
    bad.write_bytes(b"not a checkpoint" * 4)
    with pytest.raises(R.RomapError):
        b.load_object(str(bad))
    trunc = tmp_path / "trunc.romap"
    trunc.write_bytes(open(path, "rb").read()[:4096])
    with pytest.raises(R.RomapError):
        b.load_object(str(trunc), obj_id=7)
    with pytest.raises(R.RomapError):
        b.object_info(7)                        # nothing was created
    assert os.path.getsize(path) > 4 * 32768 * 2 * 4
    a.close()
    b.close()
