#!/usr/bin/env python
"""bench.py -- RO-MAP multi-object NeRF training throughput on B200.

Metric (BASELINE.json): NeRF train ray-samples/s (and seconds to the paper's
~2 s per-object budget).  A step = one training iteration of every object on
the rank: ray sampling -> hash encode -> MLP -> volume render + loss -> backward
-> Adam, run through the C ABI (libromap.so).

Workload (default, N=1): BASELINE cfg1 -- one object, L=16, F=2, T=2^16,
resolutions 16->512, density + SH colour MLP, 4096 rays x 64 stratified samples
per iteration, 20 keyframes of 640x480 of a seeded box-union-torus SDF object.
With --gpus N each rank trains its own cfg1-family object (weak scaling: objects
are independent, no data-path collective; one NCCL all_reduce of the timings at
the end).

Timing: W warm-up iterations, then exactly K iterations in ONE train_step call,
bracketed by barrier + cuda.synchronize on both sides and CUDA events on the
library's stream; L2 is flushed before every iteration by the library's
measurement hook (romap_set_l2_flush, 512 MiB) and the flush time -- timed by the
library's own events -- is subtracted.  Max over ranks.

--impl reference runs the CPU oracle (oracle/, the "reference arm" of this tier)
on a bounded sample of the same workload, on the host cores.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

PAPER_SAMPLES_PER_S = 4096 * 32 / 0.706e-3     # PAPER.md:222,307 (RTX 4090; context only)
BUDGET_SAMPLES = 2833 * 4096 * 32               # ~2 s / 0.706 ms iterations
FLUSH_BYTES = 512 << 20


def cfg1_kwargs(precision):
    return dict(levels=16, log2_T=16, base_res=16, finest_res=512.0, res_cap=0, samples_per_ray=64,
                rays_per_iter=4096, precision=precision, seed=1)


# the paper's own configuration (R24): T = 2^16, N_max = 2048,
# single hidden layer of 64 on positions only, 4096 rays x N = 32; Table 4 varies T and layers
PAPER_MS = {(16, 1): 0.706, (14, 1): 0.658, (18, 1): 0.921, (20, 1): 1.495, (16, 2): 0.862, (16, 3): 1.052}


def paper_kwargs(log2_T=16, hidden_layers=1):
    return dict(levels=16, log2_T=log2_T, base_res=16, finest_res=2048.0, res_cap=0, samples_per_ray=32,
                rays_per_iter=4096, precision=1, seed=1, network=1, hidden_layers=hidden_layers)


def workload_kwargs(args, precision):
    if args.network == "paper":
        return paper_kwargs(args.log2_T or 16, args.hidden_layers)
    kw = cfg1_kwargs(precision)
    if args.log2_T:
        kw["log2_T"] = args.log2_T
    if args.rays_per_iter:
        kw["rays_per_iter"] = args.rays_per_iter      # cfg3: 2048 rays per object
    return kw


def paper_baseline_samples_per_s(kw):
    """the paper's ray-samples/s for exactly this workload (4096 x 32 per
    iteration / Table 3-4 iteration time on an RTX 4090), or None"""
    if kw.get("network") != 1:
        return None
    ms = PAPER_MS.get((kw["log2_T"], kw["hidden_layers"]))
    return None if ms is None else 4096 * 32 / (ms * 1e-3)


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def start_clock_sampler(dev_index):
    fields = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")
    f = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
    try:
        p = subprocess.Popen(["nvidia-smi", "-i", str(dev_index), f"--query-gpu={fields}", "--format=csv,noheader,nounits",
                              "-lms", os.environ.get("BENCH_CLOCK_MS", "200")], stdout=f, stderr=subprocess.DEVNULL)
    except FileNotFoundError:
        return None, f.name
    return p, f.name


def stop_clock_sampler(p, path):
    if p is not None:
        p.terminate()
        try:
            p.wait(timeout=5)
        except Exception:
            p.kill()
    rows = []
    try:
        for line in open(path):
            parts = [x.strip() for x in line.split(",")]
            if len(parts) < 8:
                continue
            try:
                rows.append((float(parts[0]), float(parts[1]), parts[3:]))
            except ValueError:
                pass
        os.unlink(path)
    except OSError:
        pass
    if not rows:
        return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
    loaded = [r for r in rows if r[0] > 300] or rows
    names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
    reasons = sorted({names[i] for r in loaded for i, v in enumerate(r[2][1:5]) if v.lower().startswith("active")})
    return {"sm_mhz": statistics.median(r[0] for r in loaded), "sm_max_mhz": max(r[1] for r in rows),
            "reasons": reasons, "samples": len(loaded)}


def visible_index(local_rank):
    cvd = os.environ.get("CUDA_VISIBLE_DEVICES")
    if cvd:
        ids = [x for x in cvd.split(",") if x.strip()]
        if local_rank < len(ids):
            return ids[local_rank]
    return str(local_rank)


def load_scene():
    import scenes
    return scenes.object_scene(1, n_views=20)


# ----------------------------------------------------------------------------- roofline bookkeeping
def algorithmic_per_sample(kw, precision):
    """Algorithmic work per ray-sample: bytes the method must
    move and FLOPs it must compute, per kernel stage."""
    L, F = kw["levels"], 2
    LF = L * F
    mlp_fwd = 2 * (64 * LF + 16 * 64 + 64 * 32 + 64 * 64 + 3 * 64)
    mlp_bwd = 2 * mlp_fwd
    gather = L * 8 * F * (2 if precision == 1 else 4)          # table reads
    scatter = L * 8 * F * 4                                      # fp32 gradient atomics
    return {"mlp_fwd_flop": mlp_fwd, "mlp_bwd_flop": mlp_bwd, "gather_bytes": gather, "scatter_bytes": scatter}


def load_measured_peaks():
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))), "measured"
    except Exception:
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0, "sm_max_mhz": 1965.0}, "fallback"


def ncu_traffic(kernel):
    """dram bytes per launch of `kernel` from the committed ncu --set full summary, or None."""
    try:
        d = json.load(open(os.path.join(ROOT, "profiles", "ncu_traffic.json")))
        return d.get(kernel)
    except Exception:
        return None


# measured ceiling of the fused kernel's request mix (tools/micro/tma_gather_bench.cu,
# profiles/r1_micro.md): random 16-B LDG.128 gathers + RED.v4.f32 scatters 1:1 over
# L2-resident tables, per SM and cycle
REQ_CEILING = 0.828


def request_roofline(kw, samples_per_launch, ms, sm_clk, n_sm):
    """L1 sector requests of the gathers + REDs per SM-cycle against the measured
    random-access ceiling; sectors per hit sample from the committed ncu capture of
    the same model (profiles/ncu_requests.json), else None."""
    try:
        entries = json.load(open(os.path.join(ROOT, "profiles", "ncu_requests.json")))["entries"]
    except Exception:
        return None
    mine = {k: v for k, v in kw.items() if not k.startswith("_")}
    d = next((e for e in entries if e["kw"] == mine), None)
    if d is None:
        return None
    req = d["sectors_per_hit_sample"] * samples_per_launch
    achieved = req / (ms * 1e-3 * sm_clk * n_sm)
    return {"bound": "l1_l2_random_requests", "achieved": achieved, "peak": REQ_CEILING,
            "unit": "sector requests / SM / cycle", "frac": achieved / REQ_CEILING,
            "source": f"{d['sectors_per_hit_sample']:.1f} sectors per hit sample ({d['profile']}); "
                      "ceiling tools/micro/tma_gather_bench.cu"}


def roofline(prof, kw, precision, samples_per_launch, n_objs):
    peaks, src = load_measured_peaks()
    work = algorithmic_per_sample(kw, precision)
    stages = {k: v for k, v in prof.items() if v["launches"] > 0 and k not in ("l2_flush",)}
    dom = max(stages, key=lambda k: stages[k]["ms"])
    st = stages[dom]
    ms = st["ms"] / st["launches"]
    params = None
    sm_clk = peaks.get("sm_max_mhz", 1965.0) * 1e6
    if dom in ("fused_mixed",):
        # fused tile kernel: bound by L2/HBM traffic of the gathers + atomics
        bytes_ = samples_per_launch * (work["gather_bytes"] + work["scatter_bytes"])
        achieved = bytes_ / (ms * 1e-3) / 1e9
        peak = peaks["hbm_gbs"]
        out = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s"}
        # sectors per hit sample captured on the same model (any number of objects)
        rq = request_roofline(kw, samples_per_launch, ms, sm_clk, 148)
        if rq:
            out["request_roofline"] = rq
    elif dom in ("fwd_fp32", "bwd_fp32"):
        flop = samples_per_launch * (work["mlp_fwd_flop"] if dom == "fwd_fp32" else work["mlp_bwd_flop"])
        achieved = flop / (ms * 1e-3) / 1e12
        peak = 148 * 128 * 2 * sm_clk / 1e12           # fp32 FMA lanes x 2 FLOP x max SM clock
        out = {"bound": "alu", "achieved": achieved, "peak": peak, "unit": "TFLOP/s"}
    elif dom == "adam":
        # dense upper bound: 4 B grad read for all + 28 B for updated params
        nparam = kw["_n_params"] * n_objs
        bytes_ = nparam * 32
        achieved = bytes_ / (ms * 1e-3) / 1e9
        out = {"bound": "hbm", "achieved": achieved, "peak": peaks["hbm_gbs"], "unit": "GB/s"}
    else:
        bytes_ = samples_per_launch * 24
        achieved = bytes_ / (ms * 1e-3) / 1e9
        out = {"bound": "hbm", "achieved": achieved, "peak": peaks["hbm_gbs"], "unit": "GB/s"}
    out["frac"] = out["achieved"] / out["peak"]
    out["kernel"] = dom
    out["ms_per_launch"] = ms
    out["peak_source"] = src
    out["traffic"] = ncu_traffic(dom)
    return out


# ----------------------------------------------------------------------------- inference (8(a) a10, a11)
def measure_inference(ctx, h, ob, frame, torch):
    """cfg4-style inference on one trained object: density on the 128^3 vertex
    lattice spanning the box (marching-cubes input, R21) with device buffers, and
    one 640x480 render (128 midpoints per ray, host outputs)."""
    a = [float(x) for x in ob.a]
    axes = [torch.linspace(-a[k], a[k], 128, device="cuda") for k in range(3)]
    P = torch.stack(torch.meshgrid(*axes, indexing="ij"), -1).reshape(-1, 3).float().contiguous()
    ctx.query_density(h, P)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = 5
    e0.record()
    for _ in range(reps):
        ctx.query_density(h, P)
    e1.record()
    torch.cuda.synchronize()
    q_ms = e0.elapsed_time(e1) / reps
    ctx.render(h, frame.T_wc, frame.K, 640, 480, 128)
    t0 = time.perf_counter()
    ctx.render(h, frame.T_wc, frame.K, 640, 480, 128)
    r_s = time.perf_counter() - t0
    peaks, src = load_measured_peaks()
    q_gbs = P.shape[0] * 16 * 8 * 4 / (q_ms * 1e-3) / 1e9   # 16 levels x 8 corners x 4 B (fp16 F=2) per point
    return {"query_density": {"points_per_s": P.shape[0] / (q_ms * 1e-3), "ms_per_lattice": q_ms,
                              "points": int(P.shape[0]), "what": "128^3 vertex lattice of the trained object, "
                              "device buffers, CUDA events (mixed path: fp16 tables + tcgen05 first layer)",
                              "roofline": {"bound": "hbm", "achieved": q_gbs, "peak": peaks["hbm_gbs"], "unit": "GB/s",
                                           "frac": q_gbs / peaks["hbm_gbs"], "peak_source": src,
                                           "note": "algorithmic gather bytes; the 3.4 MB table is L2-resident, so the "
                                                   "random-request rate, not HBM, binds it"}},
            "render": {"rays_per_s": 640 * 480 / r_s, "ms_per_frame": r_s * 1e3, "samples_per_ray": 128,
                       "what": "one 640x480 frame, host outputs, wall clock (mixed path: tensor-core forward of midpoint samples + compositing)"}}


# ----------------------------------------------------------------------------- CPU oracle
def oracle_run(scene, kw, rays, iters, obj_id=0):
    import numpy as np
    import oracle as O
    ocfg = O.ModelConfig(**{k: v for k, v in kw.items() if k in O.ModelConfig.__dataclass_fields__})
    ocfg.rays_per_iter = rays
    ob = scene.objects[0]
    st = O.ObjectState(ocfg, ob.t, ob.yaw, ob.a, obj_id, O.init_params(ocfg, 0))
    for fr in scene.frames:
        st.kfs.append(O.ingest_observation(fr.rgb, fr.mask, fr.T_wc, fr.K, ob.instance_id))
    O.train_iteration(st)                       # warm-up
    t0 = time.perf_counter()
    samples = 0
    for _ in range(iters):
        L, _, _ = O.train_iteration(st)
        samples += L["samples"]
    dt = time.perf_counter() - t0
    return samples, dt


def host_threads():
    try:
        from threadpoolctl import threadpool_info
        n = max((i.get("num_threads", 1) for i in threadpool_info()), default=1)
    except Exception:
        n = 1
    return max(1, n)


def cpu_baseline(scene, kw, rays=1024, iters=3):
    samples, dt = oracle_run(scene, kw, rays, iters)
    return {"value": samples / dt, "unit": "ray-samples/s", "cores": host_threads(), "kind": "oracle",
            "sample": f"{iters} oracle iterations of the cfg1 object at {rays} rays x {kw['samples_per_ray']} samples "
                      f"(numpy fp32-geometry/fp64; {samples} ray-samples in {dt:.1f} s)"}


# ----------------------------------------------------------------------------- reference arm
def run_reference(args):
    ws, rank, _ = dist_env()
    if rank != 0:
        return 0
    scene = load_scene()
    kw = workload_kwargs(args, 0)
    rays = 256
    for _ in range(args.warmup):
        oracle_run(scene, kw, rays, 1)
    samples, dt = oracle_run(scene, kw, rays, args.steps)
    v = samples / dt
    line = {"impl": "reference", "metric": "NeRF train ray-samples/s", "value": v, "unit": "ray-samples/s",
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup, "ms_per_step": dt / args.steps * 1e3,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded box-union-torus SDF object, 20 keyframes 640x480)",
            "config": {"workload": "cfg1 (1 object/rank; reference = CPU oracle, bounded sample)",
                       "rays_per_iter": rays, "samples_per_ray": kw["samples_per_ray"], "levels": 16, "log2_T": 16},
            "cpu_baseline": {"value": v, "unit": "ray-samples/s", "cores": host_threads(), "kind": "oracle",
                             "sample": f"{args.steps} oracle iterations at {rays} rays x 64 samples"},
            "e2e": {"value": v, "unit": "ray-samples/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


# ----------------------------------------------------------------------------- our arm
def run_ours(args):
    import numpy as np
    import torch

    ws, rank, local = dist_env()
    if args.gpus > 1 and ws != args.gpus:
        print(f"--gpus {args.gpus} needs torchrun with {args.gpus} ranks (WORLD_SIZE={ws})", file=sys.stderr)
        return 2
    torch.cuda.set_device(local)
    pg = None
    if ws > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        pg = dist
    from paper_2304_05735_b200 import romap as R

    ctx = R.Context(local)
    precision = 1 if args.precision == "mixed" else 0
    if args.precision == "auto":
        # the mixed (tensor-core) path when this build has it, else the fp32 GPU path
        try:
            ctx.destroy_object(ctx.create_object([0, 0, 0], 0.0, [1, 1, 1], R.model_config(**cfg1_kwargs(1)), 1))
            precision = 1
        except R.RomapError:
            precision = 0
    if args.network == "paper":
        precision = 1
    kw = workload_kwargs(args, precision)
    scene = load_scene()
    from paper_2304_05735_b200.shard import partition, reduce_throughput
    objs = []
    ob = scene.objects[0]
    n_total = args.objects or args.objects_per_gpu * ws
    mine = partition([kw["rays_per_iter"] * kw["samples_per_ray"]] * n_total, ws)[rank]   # LPT by cost (8(e))
    for gid in mine:
        h = ctx.create_object(ob.t, ob.yaw, ob.a, R.model_config(**kw), ob.instance_id, obj_id=gid)
        for fr in scene.frames[:args.keyframes]:
            ctx.add_observation(h, fr.rgb, fr.mask, fr.T_wc, fr.K)
        objs.append(h)
    info = ctx.object_info(objs[0])
    kw["_n_params"] = info["table_params"] + info["mlp_params"]

    # warm-up (untimed)
    ctx.train_step(objs, args.warmup)
    torch.cuda.synchronize()

    # timed region: exactly K iterations, L2 flushed before each by the library hook.
    # Only the flush (subtracted) and the dominant kernel (roofline) are bracketed
    # with CUDA events here; the full per-stage breakdown comes from a separate
    # short profiled pass after the timed region.
    ctx.set_l2_flush(FLUSH_BYTES)
    dominant = "fused_mixed" if precision == 1 else "bwd_fp32"
    ctx.profile_enable(True, stages=[dominant, "l2_flush"])
    sampler, spath = start_clock_sampler(visible_index(local))
    time.sleep(0.3)
    stream = torch.cuda.current_stream()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if pg:
        pg.barrier()
    torch.cuda.synchronize()
    ev0.record(stream)
    th0 = time.perf_counter()
    stats = ctx.train_step(objs, args.steps)
    host_ms = (time.perf_counter() - th0) * 1e3
    ev1.record(stream)
    torch.cuda.synchronize()
    if pg:
        pg.barrier()
    clocks = stop_clock_sampler(sampler, spath)
    prof = ctx.profile_read()
    # separate, untimed pass: every stage bracketed with events (breakdown only)
    ctx.profile_enable(True)
    n_brk = min(10, args.steps)
    ctx.train_step(objs, n_brk)
    prof_all = ctx.profile_read()
    ctx.profile_enable(False)
    ctx.set_l2_flush(0)
    total_ms = ev0.elapsed_time(ev1)
    flush_ms = prof.get("l2_flush", {}).get("ms", 0.0)
    step_ms = (total_ms - flush_ms) / args.steps
    samples = sum(s["samples"] for s in stats)
    launches = sum(v["launches"] for k, v in prof.items() if k != "l2_flush")

    # e2e: the paper's online unit through the public API with HOST buffers: one new
    # keyframe (640x480 rgb + mask from pinned host memory) -> add_observation ->
    # train_step(n_iters = e2e_iters) -> per-object stats read back to the host
    e2e_frames = scene.frames[args.keyframes:] or scene.frames
    pinned = []
    for fr in e2e_frames:
        rgb = torch.from_numpy(fr.rgb).pin_memory()
        mask = torch.from_numpy(fr.mask.astype(np.int16)).pin_memory()
        pinned.append((rgb, mask, fr))
    h2d = 0
    e2e_samples = 0
    if pg:
        pg.barrier()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for k in range(args.e2e_steps):
        rgb, mask, fr = pinned[k % len(pinned)]
        m_np = mask.numpy().view(np.uint16)
        for h in objs:
            ctx.add_observation(h, rgb.numpy(), m_np, fr.T_wc, fr.K)
        st = ctx.train_step(objs, args.e2e_iters)
        e2e_samples += sum(s["samples"] for s in st)
        ys, xs = np.nonzero(m_np == ob.instance_id)
        h2d += len(objs) * ((xs.max() - xs.min() + 1) * (ys.max() - ys.min() + 1) * 4 + 96 + 8)
    torch.cuda.synchronize()
    e2e_s = time.perf_counter() - t0
    if pg:
        pg.barrier()

    # reductions over ranks: max time, sum of samples (NCCL all_reduce, shard.reduce_throughput)
    t_max_ms, tot_samples, value = reduce_throughput(step_ms * args.steps, samples, pg, device="cuda")
    e2e_max_ms, tot_e2e, e2e_value = reduce_throughput(e2e_s * 1e3, e2e_samples, pg, device="cuda")

    infer = measure_inference(ctx, objs[0], ob, scene.frames[0], torch) if rank == 0 else None
    if infer is not None:
        # cfg4 (ii): render_scene of every object on this GPU from 10 poses (640x480,
        # <= 128 samples per segment, host outputs)
        poses = scene.frames[:10]
        ctx.render_scene(objs, poses[0].T_wc, poses[0].K, 640, 480, 128)
        t0 = time.perf_counter()
        for fr in poses:
            ctx.render_scene(objs, fr.T_wc, fr.K, 640, 480, 128)
        rs_s = (time.perf_counter() - t0) / len(poses)
        infer["render_scene"] = {"objects": len(objs), "poses": len(poses), "ms_per_frame": rs_s * 1e3,
                                 "rays_per_s": 640 * 480 / rs_s,
                                 "what": "romap_render_scene of all objects, 640x480, 128 samples per segment, "
                                         "host outputs, wall clock"}
    if rank == 0:
        rf = roofline(prof, kw, precision, samples / args.steps, len(objs))
        paper_sps = paper_baseline_samples_per_s(kw)
        if args.network == "paper":
            desc = (f"paper network (PAPER.md:222, R24): L=16 F=2 T=2^{kw['log2_T']} res 16->2048, "
                    f"{kw['hidden_layers']} hidden layer(s) of 64 on positions -> sigma, rgb, {kw['rays_per_iter']} rays x 32 "
                    f"stratified samples per object, Adam")
        else:
            desc = (f"L=16 F=2 T=2^{kw['log2_T']} res 16->512, density 32->64->16 + SH4 colour 32->64->64->3, "
                    f"{kw['rays_per_iter']} rays x 64 stratified samples per object, Adam")
        cpu = None if args.no_cpu_baseline else cpu_baseline(scene, kw)
        per_obj_ms = t_max_ms / args.steps / len(objs)
        line = {
            "metric": "NeRF train ray-samples/s", "value": value, "unit": "ray-samples/s", "n_gpus": ws,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": t_max_ms / args.steps,
            "higher_is_better": True, "scaling": "strong" if args.objects else "weak",
            "vs_baseline": (value / paper_sps) if paper_sps else None,
            "dtype": "f16-mma/f32" if precision == 1 else "f32",
            "data": "synthetic (seeded box-union-torus SDF object on a textured floor, 20 keyframes 640x480, 1 cm pose jitter)",
            "config": {"workload": (f"{'paper' if args.network == 'paper' else 'cfg1'} family: {n_total} object(s) "
                                    f"over {ws} GPU(s) (LPT by cost)" if args.objects
                                    else f"{'paper' if args.network == 'paper' else 'cfg1'}: {len(objs)} object(s) per GPU")
                                   + ", " + desc,
                       "objects_per_gpu": len(objs), "rays_per_iter": kw["rays_per_iter"],
                       "samples_per_ray": kw["samples_per_ray"], "keyframes": args.keyframes,
                       "precision": "mixed" if precision == 1 else "fp32",
                       "l2": f"flushed before every iteration ({FLUSH_BYTES >> 20} MiB write by romap_set_l2_flush), "
                             "flush time excluded via the library's CUDA events",
                       "parallelism": f"objects sharded over {ws} rank(s), NCCL only for the final max/sum"},
            "s_to_budget_per_object": BUDGET_SAMPLES / (value / max(1, ws * len(objs))),
            "ms_per_iteration_per_object": per_obj_ms,
            "paper_context": {"samples_per_s": PAPER_SAMPLES_PER_S, "ms_per_iteration": 0.706,
                              "note": ("RTX 4090, N=32, position-only 1x64 MLP (PAPER.md:222,307); "
                                       + ("this workload (vs_baseline = value / the paper's rate)" if paper_sps
                                          else "not this workload"))},
            "hit_samples_per_step": samples / args.steps,
            "stage_ms_per_step": {k: v["ms"] / n_brk for k, v in prof_all.items() if v["launches"] or v["ms"]},
            "stage_ms_note": f"separate {n_brk}-iteration pass with every stage bracketed by events (not the timed region)",
            "kernel_ms_per_step": sum(v["ms"] for k, v in prof_all.items() if k != "l2_flush") / n_brk,
            "timed_region": {"total_ms": total_ms, "l2_flush_ms_subtracted": flush_ms, "host_ms_in_call": host_ms,
                             "dominant_ms": prof.get(dominant, {}).get("ms")},
            "gpu_launches": launches,
            "roofline": rf,
            "cpu_baseline": cpu,
            "e2e": {"value": e2e_value, "unit": "ray-samples/s", "h2d_bytes_per_step": int(h2d / max(1, args.e2e_steps)),
                    "d2h_bytes_per_step": int(len(objs) * 40 + 4),
                    "step": f"add_observation(1 keyframe, host) + train_step({args.e2e_iters} iterations) + stats D2H"},
            "clocks": clocks,
            "inference": infer,
        }
        print(json.dumps(line), flush=True)
    ctx.close()
    if pg:
        pg.destroy_process_group()
    return 0


def run_table4(args):
    """The paper's Table 4 grid on one GPU: ms per training iteration
    of one object (4096 rays x 32, a1..a8 incl. Adam, L2 flushed before each iteration)
    next to the paper's RTX 4090 numbers."""
    import torch
    from paper_2304_05735_b200 import romap as R

    ctx = R.Context(0)
    scene = load_scene()
    ob = scene.objects[0]
    rows = []
    for (lt, hl), pms in sorted(PAPER_MS.items(), key=lambda x: (x[0][1], x[0][0])):
        kw = paper_kwargs(lt, hl)
        h = ctx.create_object(ob.t, ob.yaw, ob.a, R.model_config(**kw), ob.instance_id)
        for fr in scene.frames[:args.keyframes]:
            ctx.add_observation(h, fr.rgb, fr.mask, fr.T_wc, fr.K)
        ctx.train_step([h], args.warmup)
        ctx.set_l2_flush(FLUSH_BYTES)
        ctx.profile_enable(True, stages=["l2_flush"])
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        st = ctx.train_step([h], args.steps)
        e1.record()
        torch.cuda.synchronize()
        fl = ctx.profile_read()["l2_flush"]["ms"]
        ctx.profile_enable(False)
        ctx.set_l2_flush(0)
        ms = (e0.elapsed_time(e1) - fl) / args.steps
        rows.append({"log2_T": lt, "hidden_layers": hl, "ms_per_iteration": ms,
                     "ray_samples_per_s": st[0]["samples"] / (ms * 1e-3 * args.steps),
                     "paper_ms_rtx4090": pms, "speedup_vs_paper": pms / ms})
        ctx.destroy_object(h)
    ctx.close()
    print(json.dumps({"metric": "NeRF train ms per iteration (paper Table 4 grid)", "unit": "ms",
                      "higher_is_better": False, "steps": args.steps, "warmup": args.warmup,
                      "data": "synthetic cfg1-family object, 20 keyframes 640x480",
                      "l2": "flushed before every iteration, flush time excluded", "table4": rows}), flush=True)
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--precision", choices=["auto", "mixed", "fp32"], default="auto")
    ap.add_argument("--objects-per-gpu", type=int, default=1)
    ap.add_argument("--objects", type=int, default=0,
                    help="total objects over all ranks, LPT-partitioned (0: objects-per-gpu x ranks)")
    ap.add_argument("--keyframes", type=int, default=20)
    ap.add_argument("--rays-per-iter", type=int, default=0, help="rays per object and iteration (0: the config's)")
    ap.add_argument("--e2e-steps", type=int, default=8)
    ap.add_argument("--e2e-iters", type=int, default=50)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--network", choices=["baseline", "paper"], default="baseline",
                    help="baseline: BASELINE cfg1 (default, the headline); paper: PAPER.md:222 network (R24)")
    ap.add_argument("--hidden-layers", type=int, default=1, help="--network paper: hidden layers (Table 4: 1..3)")
    ap.add_argument("--log2-T", type=int, default=0, help="hash table size override (Table 4: 14..20)")
    ap.add_argument("--table4", action="store_true", help="run the paper's Table 4 sweep (PAPER.md:353-357)")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        return run_reference(args)
    if args.table4:
        return run_table4(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
