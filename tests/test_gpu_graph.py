"""the iteration driver replays a CUDA graph of K training
iterations (mixed path, timing events off).  A multi-iteration train_step must
train exactly like K single iterations: the oracle tracks it, and the graph
replay equals plain launches (profiling on disables the graph) BITWISE in the
deterministic-reduction mode (romap_set_deterministic; SURVEY 8(c) tolerances,
SPEC.md:436,452).  With fp32 atomics (the default) graph and plain runs may
differ only as much as two plain runs differ from each other."""
import numpy as np
import pytest

import oracle as O
import scenes
from gpu_common import make_pair, norm_rel

pytestmark = pytest.mark.gpu

from paper_2304_05735_b200 import romap as R  # noqa: E402

CFG0M = dict(levels=8, log2_T=12, base_res=16, finest_res=2048.0, res_cap=128, samples_per_ray=32, rays_per_iter=256,
             precision=1, seed=0)
STATE_BLOCKS = (R.BLOCK_TABLE, R.BLOCK_MLP, R.BLOCK_M_TABLE, R.BLOCK_M_MLP, R.BLOCK_V_TABLE, R.BLOCK_V_MLP)


def _scene():
    return scenes.sphere_scene(0, n_views=8)


def _graph_replays(c):
    return c.profile_read()["graph_replay"]["launches"]


def test_graph_chunks_track_the_oracle():
    c = R.Context(0)
    sc = _scene()
    h, st = make_pair(R, c, sc, CFG0M)
    n_iters = 40                                   # 2 graph chunks of 16 + an 8-iteration tail
    s = c.train_step([h], n_iters)[0]
    assert _graph_replays(c) == 2                   # the graph really ran (a9)
    for _ in range(n_iters):
        o, _, _ = O.train_iteration(st)
    assert s["step"] == n_iters
    # losses of the last iteration, 40 Adam steps in: fp16 operands, same samples
    assert abs(s["l_total"] - o["l_total"]) <= 5e-2 * o["l_total"], (s, o)
    t = c.get_params(h, R.BLOCK_TABLE).reshape(-1, 2)
    assert norm_rel(t, st.params["table"]) < 5e-2
    c.close()


def _run(sc, graph, det, calls=(32, 17)):
    c = R.Context(0)
    if det:
        c.set_deterministic(True)
    h, _ = make_pair(R, c, sc, CFG0M, param_seed=7)
    if not graph:
        c.profile_enable(True)                     # per-stage events: no graph
    stats = [c.train_step([h], n)[0] for n in calls]   # 32: two chunks; 17: one chunk + 1 plain iteration
    replays = _graph_replays(c)
    state = [c.get_params(h, b) for b in STATE_BLOCKS]
    c.close()
    return stats, state, replays


def test_graph_equals_plain_launches_bitwise_deterministic():
    sc = _scene()
    (g1, g2), gst, g_rep = _run(sc, graph=True, det=True)
    (p1, p2), pst, p_rep = _run(sc, graph=False, det=True)
    assert g_rep == 3 and p_rep == 0
    assert g2["step"] == p2["step"] == 49
    for a, b in ((g1, p1), (g2, p2)):
        for k in ("l_total", "l_rgb", "l_rr", "l_depth", "l_density", "hit_rays", "samples"):
            assert a[k] == b[k], (k, a[k], b[k])
    for x, y in zip(gst, pst):
        assert np.array_equal(x.view(np.uint32), y.view(np.uint32))
    # and the deterministic mode is reproducible run to run
    (q1, q2), qst, _ = _run(sc, graph=True, det=True)
    assert q2["l_total"] == g2["l_total"]
    for x, y in zip(gst, qst):
        assert np.array_equal(x.view(np.uint32), y.view(np.uint32))


def test_graph_matches_plain_launches_atomics():
    """Default mode (fp32 atomics): the fp32 summation order changes run to run and
    49 Adam steps amplify it, so the graph-vs-plain gap is bounded by the measured
    plain-vs-plain gap (losses and parameters), not by a fixed tolerance."""
    sc = _scene()
    (g1, g2), gst, g_rep = _run(sc, graph=True, det=False)
    (a1, a2), ast, _ = _run(sc, graph=False, det=False)
    (b1, b2), bst, _ = _run(sc, graph=False, det=False)
    assert g_rep == 3
    # same rays and samples (the RNG is keyed by the device step counters)
    assert g1["hit_rays"] == a1["hit_rays"] and g2["hit_rays"] == a2["hit_rays"] == b2["hit_rays"]
    # (floor 2e-2: the mixed path's loss tolerance; two plain runs can land closer to
    # each other by chance than the spread of the summation order allows, the
    # round-1 failure was such a 1.005 % graph-vs-plain gap; the exact check is the
    # deterministic-mode test above)
    for k in ("l_total", "l_rgb", "l_density"):
        d_gp = abs(g2[k] - a2[k])
        d_pp = abs(b2[k] - a2[k])
        assert d_gp <= 3.0 * d_pp + 2e-2 * abs(a2[k]), (k, g2[k], a2[k], b2[k])
    d_gp = max(norm_rel(gst[0], ast[0]), norm_rel(gst[1], ast[1]))
    d_pp = max(norm_rel(bst[0], ast[0]), norm_rel(bst[1], ast[1]))
    assert d_gp <= 3.0 * d_pp + 5e-3, (d_gp, d_pp)


def test_graph_multi_object_with_keyframe_appends():
    """Three objects batched, 20 iterations per call (one graph chunk of 16 + a
    4-iteration tail), keyframes appended between calls: the cached graph is
    replayed with the new descriptors, the geometry stays bit-exact (hit counts
    summed over each call) and the losses track the oracle."""
    import dataclasses
    c = R.Context(0)
    sc = scenes.room_scene(6, n_objects=3, n_frames=8, W=160, H=120, f=131.25, room_half=1.5)
    half = sc.frames[: len(sc.frames) // 2]
    sc_half = dataclasses.replace(sc, frames=half)
    kw = dict(CFG0M, rays_per_iter=128, seed=6)
    hs, sts = [], []
    for k, ob in enumerate(sc.objects[:3]):
        h, st = make_pair(R, c, sc_half, kw, param_seed=60 + k, inst=ob.instance_id, obj_id=400 + k,
                          avoid_kinks=False)
        hs.append(h)
        sts.append(st)
    for call in range(2):
        if call == 1:
            for k, ob in enumerate(sc.objects[:3]):
                for fr in sc.frames[len(half):]:
                    if (fr.mask == ob.instance_id).any():
                        c.add_observation(hs[k], fr.rgb, fr.mask, fr.T_wc, fr.K)
                        sts[k].kfs.append(O.ingest_observation(fr.rgb, fr.mask, fr.T_wc, fr.K, ob.instance_id))
        s = c.train_step(hs, 20)
        for k in range(3):
            hits = 0
            for _ in range(20):
                o, _, _ = O.train_iteration(sts[k])
                hits += o["hit_rays"]
            assert s[k]["hit_rays"] == hits, (call, k, s[k]["hit_rays"], hits)
            assert s[k]["step"] == 20 * (call + 1)
            assert abs(s[k]["l_total"] - o["l_total"]) <= 5e-2 * o["l_total"], (call, k, s[k], o)
    assert _graph_replays(c) == 2
    c.close()


def test_graph_rebuilt_when_the_batch_changes():
    """The cached graph is keyed by the batch (objects, slots, buffers): one object,
    then two (the ray buffers grow), then the other alone -- every call replays a
    graph built for its own batch, with geometry bit-exact against the oracle."""
    c = R.Context(0)
    sc = scenes.room_scene(7, n_objects=2, n_frames=6, W=160, H=120, f=131.25, room_half=1.5)
    kw = dict(CFG0M, rays_per_iter=128, seed=7)
    pairs = [make_pair(R, c, sc, kw, param_seed=70 + k, inst=ob.instance_id, obj_id=500 + k, avoid_kinks=False)
             for k, ob in enumerate(sc.objects[:2])]
    (h1, s1), (h2, s2) = pairs
    for batch in ([0], [0, 1], [1]):
        hs = [pairs[k][0] for k in batch]
        out = c.train_step(hs, 18)                 # one 16-iteration chunk + 2
        for k, st in zip(batch, out):
            hits = 0
            for _ in range(18):
                o, _, _ = O.train_iteration(pairs[k][1])
                hits += o["hit_rays"]
            assert st["hit_rays"] == hits, (batch, k, st["hit_rays"], hits)
            assert abs(st["l_total"] - o["l_total"]) <= 5e-2 * o["l_total"], (batch, k, st, o)
    assert _graph_replays(c) == 3
    assert c.object_info(h1)["step"] == 36 and c.object_info(h2)["step"] == 36
    c.close()
