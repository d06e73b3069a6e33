"""Full-size multi-object geometry in the launch configuration bench.py times
(BASELINE cfg2 / cfg3 shapes: 640x480 keyframes, cfg1 model, 4096-ray objects of
edge lengths U(0.2, 1.5) m batched in ONE train_step with rays split by mask
area): after a multi-iteration train_step (graph chunk + plain tail), every
object's ray records equal the oracle's bit for bit (pixel, class, ray, segment,
targets, background colour), and for the largest object also the sample records
and the corner entries the fused kernel consumed (SURVEY 8(c) "bit-exact hash
indices, sample positions and ray-box segments")."""
import numpy as np
import pytest

import oracle as O
import scenes
from gpu_common import ocfg_from

pytestmark = pytest.mark.gpu

R = pytest.importorskip("paper_2304_05735_b200.romap")

KW = dict(levels=16, log2_T=16, base_res=16, finest_res=512.0, res_cap=0, samples_per_ray=64, rays_per_iter=4096,
          precision=1, seed=2)


def test_cfg2_shape_batch_full_size_geometry():
    sc = scenes.room_scene(2, n_objects=8, n_frames=40)          # 640 x 480, f = 525
    objs, kfs = [], []
    for ob in sc.objects:
        vis = scenes.visible_frames(sc, ob.instance_id, min_frac=0.01)
        if vis:
            objs.append(ob)
            kfs.append(vis[:12])
    assert len(objs) >= 4
    areas = np.array([sum(int((sc.frames[i].mask == ob.instance_id).sum()) for i in k) for ob, k in zip(objs, kfs)],
                     float)
    total = 4096 * len(objs)
    share = total * areas / areas.sum()
    rays = np.maximum(np.floor(share).astype(int), 128)
    rays[np.argsort(-(share - np.floor(share)))[: max(0, total - rays.sum())]] += 1
    c = R.Context(0)
    hs, sts = [], []
    for j, (ob, k, r) in enumerate(zip(objs, kfs, rays)):
        kw = dict(KW, rays_per_iter=int(r))
        h = c.create_object(ob.t, ob.yaw, ob.a, R.model_config(**kw), ob.instance_id, obj_id=900 + j)
        st = O.ObjectState(ocfg_from(kw), np.asarray(ob.t, np.float32), float(np.float32(ob.yaw)),
                           np.asarray(ob.a, np.float32), 900 + j, {"table": np.zeros((1, 2)), "W": []})
        for i in k:
            fr = sc.frames[i]
            c.add_observation(h, fr.rgb, fr.mask, fr.T_wc, fr.K)
            st.kfs.append(O.ingest_observation(fr.rgb, fr.mask, fr.T_wc, fr.K, ob.instance_id))
        hs.append(h)
        sts.append(st)
    n_it = 19                                                      # one 16-iteration graph chunk + 3 plain
    out = c.train_step(hs, n_it)
    big = int(np.argmax(rays))
    for j, (h, st) in enumerate(zip(hs, sts)):
        rs = O.forward_rays(st, n_it)
        rd = c.debug_dump(h, R.DUMP_RAYS)
        assert len(rd) == rays[j]
        assert np.array_equal(rd["kf"], rs["k"]) and np.array_equal(rd["px"], rs["px"])
        assert np.array_equal(rd["py"], rs["py"]) and np.array_equal(rd["cls"], rs["cls"])
        assert np.array_equal(rd["hit"].astype(bool), rs["hit"])
        for a, b in [("o", "o"), ("d", "d"), ("t_near", "tn"), ("t_far", "tf"), ("target", "tgt"), ("bg", "bg")]:
            x = rd[a]
            y = np.asarray(rs[b], np.float32)
            if a in ("t_near", "t_far"):
                x, y = x[rs["hit"]], y[rs["hit"]]
            assert np.array_equal(x.view(np.uint32), y.view(np.uint32)), (j, a)
        assert out[j]["step"] == n_it
        if j == big:
            N = KW["samples_per_ray"]
            hit = rs["hit"]
            sm = c.debug_dump(h, R.DUMP_SAMPLES).reshape(rays[j], N, 5)[hit]
            for col, key in ((0, "dist"), (1, "delta")):
                assert np.array_equal(np.ascontiguousarray(sm[..., col]).view(np.uint32), rs[key][hit].view(np.uint32))
            assert np.array_equal(np.ascontiguousarray(sm[..., 2:5]).view(np.uint32), rs["u"][hit].view(np.uint32))
            _, idx, _ = O.hash_encode(rs["u"][hit].reshape(-1, 3), np.zeros((O.table_entries(st.cfg), 2)), st.cfg)
            gi = c.debug_dump(h, R.DUMP_HASH_IDX).reshape(rays[j], N, 16, 8)[hit].reshape(-1, 16, 8)
            assert np.array_equal(gi.astype(np.int64), idx)
    c.close()
