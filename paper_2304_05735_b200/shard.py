"""Object sharding across the GPUs of one box.

Objects are independent: each rank trains its own subset with
no data-path collective.  This module holds the host-side policy only:

* ``partition``: static LPT (longest processing time first) assignment of objects
  to ranks by per-iteration cost (rays x samples); deterministic, so every rank
  computes the same map without communication.  Objects keep their GLOBAL ids
  (the RNG of the method is keyed by the global id, R13), so per-object
  results do not depend on the number of ranks.
* ``reduce_throughput``: the single end-of-run reduction: MAX of elapsed device
  time and SUM of processed ray-samples over ranks (one all_reduce each, NCCL on
  the GPU box, gloo in the CPU tests); whole-job throughput = sum / max.
"""
from __future__ import annotations

import heapq


def partition(costs, world: int):
    """LPT: objects in decreasing cost (ties -> smaller id first) go to the rank with
    the smallest load so far (ties -> smaller rank).  Returns, per rank, the list of
    object indices in ascending order."""
    if world < 1:
        raise ValueError("world must be >= 1")
    order = sorted(range(len(costs)), key=lambda i: (-costs[i], i))
    heap = [(0, r) for r in range(world)]
    out = [[] for _ in range(world)]
    for i in order:
        load, r = heapq.heappop(heap)
        out[r].append(i)
        heapq.heappush(heap, (load + costs[i], r))
    return [sorted(o) for o in out]


def reduce_throughput(elapsed_ms: float, samples: float, dist=None, device=None):
    """(max elapsed ms, sum samples, samples/s) over ranks; `dist` = torch.distributed
    (initialised) or None for a single process."""
    import torch

    t = torch.tensor([float(elapsed_ms)], dtype=torch.float64, device=device)
    n = torch.tensor([float(samples)], dtype=torch.float64, device=device)
    if dist is not None and dist.is_initialized() and dist.get_world_size() > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        dist.all_reduce(n, op=dist.ReduceOp.SUM)
    tmax, ntot = float(t.item()), float(n.item())
    return tmax, ntot, (ntot / (tmax * 1e-3) if tmax > 0 else 0.0)
