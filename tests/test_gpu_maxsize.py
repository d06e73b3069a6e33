"""Maximum sizes (the edge case list of the parity bar): a batch of 4 cfg1-model
objects with 2^18 rays x 64 samples each -- 67 M samples per iteration, 1.3 GB of
sample records, 2^19 tiles of the fused kernel, 64x cfg1 -- trained through
train_step.  Every object's statistics are finite and its hit-ray count equals
the oracle's; the last object's ray records (pixel, class, ray, segment, targets,
background) and the sample records the fused kernel consumed are bit-exact with
the oracle's at that size (no 32-bit index overflows on the path)."""
import numpy as np
import pytest

import oracle as O
import scenes
from gpu_common import ocfg_from

pytestmark = pytest.mark.gpu

R = pytest.importorskip("paper_2304_05735_b200.romap")

KW = dict(levels=16, log2_T=16, base_res=16, finest_res=512.0, res_cap=0, samples_per_ray=64, rays_per_iter=1 << 18,
          precision=1, seed=12)
N_OBJ = 4
N_IT = 2


def test_four_objects_of_2e18_rays_geometry_bit_exact():
    sc = scenes.object_scene(1, n_views=20)
    ob = sc.objects[0]
    c = R.Context(0)
    hs = []
    for j in range(N_OBJ):
        h = c.create_object(ob.t, ob.yaw, ob.a, R.model_config(**KW), ob.instance_id, obj_id=500 + j)
        for fr in sc.frames:
            c.add_observation(h, fr.rgb, fr.mask, fr.T_wc, fr.K)
        hs.append(h)
    stats = c.train_step(hs, N_IT)
    assert all(s["step"] == N_IT for s in stats)
    assert all(np.isfinite(s["l_total"]) for s in stats)
    # the oracle's rays of the last object, last iteration (t = N_IT)
    st = O.ObjectState(ocfg_from(KW), np.asarray(ob.t, np.float32), float(np.float32(ob.yaw)),
                       np.asarray(ob.a, np.float32), 500 + N_OBJ - 1, {"table": np.zeros((1, 2)), "W": []})
    for fr in sc.frames:
        st.kfs.append(O.ingest_observation(fr.rgb, fr.mask, fr.T_wc, fr.K, ob.instance_id))
    rs = O.forward_rays(st, N_IT)
    h = hs[-1]
    rd = c.debug_dump(h, R.DUMP_RAYS)
    assert len(rd) == KW["rays_per_iter"]
    assert np.array_equal(rd["kf"], rs["k"]) and np.array_equal(rd["px"], rs["px"]) and np.array_equal(rd["py"], rs["py"])
    assert np.array_equal(rd["cls"], rs["cls"]) and np.array_equal(rd["hit"].astype(bool), rs["hit"])
    for a, b in [("o", "o"), ("d", "d"), ("target", "tgt"), ("bg", "bg")]:
        assert np.array_equal(rd[a].view(np.uint32), np.asarray(rs[b], np.float32).view(np.uint32)), a
    hit = rs["hit"]
    # hit rays of the last iteration (the count in the statistics sums the call's iterations)
    assert hit.sum() > KW["rays_per_iter"] // 4
    for a, b in [("t_near", "tn"), ("t_far", "tf")]:
        assert np.array_equal(rd[a][hit].view(np.uint32), np.asarray(rs[b], np.float32)[hit].view(np.uint32)), a
    N = KW["samples_per_ray"]
    sm = c.debug_dump(h, R.DUMP_SAMPLES).reshape(KW["rays_per_iter"], N, 5)[hit]
    assert np.array_equal(np.ascontiguousarray(sm[..., 0]).view(np.uint32), rs["dist"][hit].view(np.uint32))
    assert np.array_equal(np.ascontiguousarray(sm[..., 1]).view(np.uint32), rs["delta"][hit].view(np.uint32))
    assert np.array_equal(np.ascontiguousarray(sm[..., 2:5]).view(np.uint32), rs["u"][hit].view(np.uint32))
    # per-object hit counts over both iterations against the oracle's (t = 1 and 2)
    for j in range(N_OBJ):
        st.obj_id = 500 + j
        n_hit = sum(int(O.forward_rays(st, t)["hit"].sum()) for t in range(1, N_IT + 1)) if j < N_OBJ - 1 else \
            int(O.forward_rays(st, 1)["hit"].sum()) + int(hit.sum())
        assert stats[j]["hit_rays"] == n_hit, (j, stats[j]["hit_rays"], n_hit)
    c.close()
