"""Multi-GPU host logic on CPU (gloo, world_size 2), SURVEY.md 8(e):
object partition, global-id keyed results invariant to the number of ranks, and
the single end-of-run reduction (max time, sum samples).  The data path runs the
CPU oracle here (no GPU in this container); the GPU box runs the same policy
through bench.py --gpus N with NCCL."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle as O
import scenes
from paper_2304_05735_b200.shard import partition, reduce_throughput

TINY = dict(levels=2, log2_T=6, base_res=2, finest_res=4.0, res_cap=0, samples_per_ray=8, rays_per_iter=24, seed=7)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _train_objects(ids, iters=2):
    """oracle training of objects with global ids `ids` (seeded per id); returns
    {id: [l_total per iteration]} and the ray-sample count"""
    sc = scenes.sphere_scene(0, n_views=3, size=16, f=16.0)
    ob = sc.objects[0]
    cfg = O.ModelConfig(**TINY)
    out, samples = {}, 0
    for gid in ids:
        st = O.ObjectState(cfg, ob.t, ob.yaw, ob.a, gid, O.init_params(cfg, gid))
        for fr in sc.frames:
            st.kfs.append(O.ingest_observation(fr.rgb, fr.mask, fr.T_wc, fr.K, ob.instance_id))
        losses = []
        for _ in range(iters):
            L, _, _ = O.train_iteration(st)
            losses.append(L["l_total"])
            samples += L["samples"]
        out[gid] = losses
    return out, samples


def _worker(rank, world, port, costs, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    mine = partition(costs, world)[rank]
    res, samples = _train_objects(mine)
    elapsed = 10.0 + rank                       # stand-in device times (ms) of the ranks
    tmax, ntot, thr = reduce_throughput(elapsed, samples, dist)
    q.put((rank, mine, res, samples, tmax, ntot, thr))
    dist.barrier()
    dist.destroy_process_group()


def test_partition_lpt():
    assert partition([1, 1, 1, 1], 2) == [[0, 2], [1, 3]]
    p = partition([5, 1, 4, 2, 3], 2)
    assert sorted(sum(p, [])) == [0, 1, 2, 3, 4]
    loads = [sum([5, 1, 4, 2, 3][i] for i in r) for r in p]
    assert max(loads) - min(loads) <= 1
    assert partition([3, 3], 4) == [[0], [1], [], []]
    with pytest.raises(ValueError):
        partition([1], 0)


def test_two_ranks_match_one_rank():
    costs = [2048 * 64] * 3 + [1024 * 64]
    ref, ref_samples = _train_objects(range(len(costs)))
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, costs, q)) for r in range(2)]
    for p in procs:
        p.start()
    outs = [q.get(timeout=600) for _ in range(2)]
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    got, seen = {}, []
    for rank, mine, res, samples, tmax, ntot, thr in outs:
        seen += mine
        got.update(res)
        assert tmax == 11.0                       # MAX over ranks
        assert ntot == ref_samples                # SUM over ranks
        assert thr == pytest.approx(ref_samples / 11e-3)
    assert sorted(seen) == list(range(len(costs)))
    for gid, losses in ref.items():               # sharding-invariant (global-id keyed RNG, R13)
        assert np.array_equal(np.asarray(got[gid]), np.asarray(losses))


def test_bench_launcher_two_ranks_dry_run():
    """bench.py --gpus 2 launched the way the driver does without torchrun: the
    script starts its own 2 ranks (torch.distributed.run, rendezvous on 127.0.0.1),
    partitions cfg3's 64 objects by LPT, reduces (max time, sum samples) over gloo and
    rank 0 prints ONE JSON line (--dry-run: no GPU, no kernels)"""
    import json
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    r = subprocess.run([sys.executable, os.path.join(root, "bench.py"), "--gpus", "2", "--dry-run", "--steps", "3",
                        "--warmup", "3"], capture_output=True, text=True, timeout=300, env=env, cwd=root)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, r.stdout
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["config"]["workload"] == "cfg3" and d["config"]["objects"] == 64
    assert sorted(sum(d["partition"], [])) == list(range(64))
    assert [len(p) for p in d["partition"]] == [32, 32]
    assert d["max_ms"] == 2.0                                    # MAX over ranks (1 + rank)
    assert d["total_samples"] == 64 * 2048 * 64 * 3              # SUM over ranks
