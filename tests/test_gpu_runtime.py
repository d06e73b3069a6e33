"""Runtime calls of the ABI that the parity tests do not exercise: the per-object
ray quota (romap_set_rays_per_iter, the host policy of R9 / cfg2), per-stage
profiling (romap_profile_enable / stages / read), the L2 flush of the bench's
timing rule (romap_set_l2_flush) and romap_sync.  Geometry after a quota change
is bit-exact with the oracle drawing the new number of rays; the flush and the
profiler change no result (deterministic mode, bitwise)."""
import numpy as np
import pytest

import oracle as O
import scenes
from gpu_common import make_pair

pytestmark = pytest.mark.gpu

R = pytest.importorskip("paper_2304_05735_b200.romap")

CFG0M = dict(levels=8, log2_T=12, base_res=16, finest_res=2048.0, res_cap=128, samples_per_ray=32, rays_per_iter=256,
             precision=1, seed=5)


def test_set_rays_per_iter_changes_the_draw():
    sc = scenes.sphere_scene(0)
    c = R.Context(0)
    h, st = make_pair(R, c, sc, CFG0M)
    c.train_step([h], 2)
    c.set_rays_per_iter(h, 77)                        # ragged: not a multiple of the 4 rays per tile
    out = c.train_step([h], 1)[0]
    assert out["rays"] == 77 and out["step"] == 3
    rs = O.forward_rays(st, 3, rays_per_iter=77)
    rd = c.debug_dump(h, R.DUMP_RAYS)
    assert len(rd) == 77
    assert np.array_equal(rd["px"], rs["px"]) and np.array_equal(rd["py"], rs["py"])
    assert np.array_equal(rd["hit"].astype(bool), rs["hit"])
    assert np.array_equal(rd["bg"].view(np.uint32), np.asarray(rs["bg"], np.float32).view(np.uint32))
    assert out["hit_rays"] == int(rs["hit"].sum())
    with pytest.raises(R.RomapError):
        c.set_rays_per_iter(h, 0)
    with pytest.raises(R.RomapError):
        c.set_rays_per_iter(12345, 64)
    c.close()


def _trained(flush, profile):
    sc = scenes.sphere_scene(0)
    c = R.Context(0)
    c.set_deterministic(True)
    h, _ = make_pair(R, c, sc, CFG0M)
    if flush:
        c.set_l2_flush(64 << 20)
    if profile:
        c.profile_enable(True, stages=["fused_mixed", "l2_flush"])
    st = c.train_step([h], 5)[0]
    c.sync()
    prof = c.profile_read()
    out = (c.get_params(h, R.BLOCK_TABLE).copy(), c.get_params(h, R.BLOCK_MLP).copy(), st, prof)
    c.close()
    return out


def test_profiler_and_l2_flush_change_no_result():
    t0, w0, s0, p0 = _trained(False, False)
    t1, w1, s1, p1 = _trained(True, True)
    assert np.array_equal(t0.view(np.uint32), t1.view(np.uint32)) and np.array_equal(w0.view(np.uint32), w1.view(np.uint32))
    assert s0["l_total"] == s1["l_total"] and s0["step"] == s1["step"] == 5
    # launch counters are always kept; events only for the selected stages
    assert p1["fused_mixed"]["launches"] == 5 and p1["adam"]["launches"] == 5 and p1["l2_flush"]["launches"] == 5
    assert p1["fused_mixed"]["ms"] > 0 and p1["l2_flush"]["ms"] > 0 and p1["adam"]["ms"] == 0
    assert p0["l2_flush"]["launches"] == 0 and p0["fused_mixed"]["launches"] == 5
    # without per-stage events the 5 iterations replay a graph chunk
    assert p0["graph_replay"]["launches"] >= 1 and p1["graph_replay"]["launches"] == 0


def test_query_density_device_pointers_equal_host():
    """ROMAP_DEVICE_PTRS: a CUDA tensor in, a CUDA tensor out, in stream order on
    the context's stream -- bitwise the host-buffer result (both paths)"""
    import torch
    sc = scenes.sphere_scene(0)
    g = np.random.default_rng(4)
    pts = g.uniform(-0.6, 0.6, (70001, 3)).astype(np.float32)      # ragged last tile, points outside the box
    for precision in (0, 1):
        c = R.Context(0)
        h, _ = make_pair(R, c, sc, dict(CFG0M, precision=precision))
        host = c.query_density(h, pts)
        dev = c.query_density(h, torch.from_numpy(pts).cuda()).cpu().numpy()
        assert np.array_equal(host.view(np.uint32), dev.view(np.uint32)), precision
        assert (host == 0).any() and (host > 0).any()
        c.close()
