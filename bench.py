#!/usr/bin/env python
"""bench.py -- RO-MAP multi-object NeRF training throughput on B200.

Metric (BASELINE.json): NeRF train ray-samples/s and seconds-to-budget per object.
A step = one training iteration of every object on the rank: ray sampling ->
hash encode -> MLP -> volume render + loss -> backward -> Adam (SURVEY.md 8(a)
a1..a8), run through the C ABI (libromap.so).

Workloads (--workload; BASELINE.json configs, synthetic stand-ins of the paper's
640x480 sequences):
  cfg1  one object per rank: L=16, F=2, T=2^16, resolutions 16->512, density +
        SH colour MLP, 4096 rays x 64 stratified samples, 20 keyframes 640x480
        (the N=1 default: BASELINE's metric is quoted on it)
  cfg3  64 objects of the cfg1 family (seeded shapes, edges U(0.2, 1.5) m), 2048
        rays x 64 each, LPT-sharded over the ranks by cost, objects keep their
        global ids; strong scaling (the N>1 default)
  cfg2  8 objects of one room on one GPU, rays split by mask area (4096 x 8 in
        total), keyframes U{5..40} per object revealed in 6 batches, appended
        before iterations 0, 50, ..., 250 (300 iterations)
  cfg4  the 64 cfg3 objects trained 200 iterations, then density on a 128^3
        lattice per object and render_scene of all 64 (placed in a room with
        romap_set_box) from 10 poses
With --gpus N and no WORLD_SIZE in the environment the script launches itself
under torch.distributed.run with N ranks (one per GPU, NCCL; init logged with
NCCL_DEBUG=INFO / SUBSYS=INIT).  No data-path collective: one all_reduce of the
timings at the end.

Timing: W warm-up iterations, then exactly K iterations in ONE train_step call,
bracketed by barrier + cuda.synchronize on both sides and CUDA events; L2 is
flushed before every iteration by the library's measurement hook
(romap_set_l2_flush, 512 MiB) and the flush time -- timed by the library's own
events on its stream -- is subtracted.  Max over ranks.

--impl reference runs the CPU oracle (oracle/, the "reference arm" of this tier)
on a bounded sample of the same workload, on the host cores.  --dry-run runs the
launcher, the partition and the end-of-run reduction without a GPU (gloo; the
CPU test of the multi-rank path).
"""
from __future__ import annotations

import argparse
import json
import math
import os
import socket
import statistics
import subprocess
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

PAPER_SAMPLES_PER_S = 4096 * 32 / 0.706e-3     # PAPER.md:222,307 (RTX 4090; context only)
PAPER_ITERS_TO_BUDGET = 2833                    # ~2 s / 0.706 ms per iteration
FLUSH_BYTES = 512 << 20
CONFIG_ITERS = {"cfg1": 500, "cfg2": 300, "cfg3": 200, "cfg4": 200, "paper": 300}


def cfg1_kwargs(precision, rays=4096):
    return dict(levels=16, log2_T=16, base_res=16, finest_res=512.0, res_cap=0, samples_per_ray=64,
                rays_per_iter=rays, precision=precision, seed=1)


# the paper's own configuration (R24): T = 2^16, N_max = 2048,
# single hidden layer of 64 on positions only, 4096 rays x N = 32; Table 4 varies T and layers
PAPER_MS = {(16, 1): 0.706, (14, 1): 0.658, (18, 1): 0.921, (20, 1): 1.495, (16, 2): 0.862, (16, 3): 1.052}


def paper_kwargs(log2_T=16, hidden_layers=1):
    return dict(levels=16, log2_T=log2_T, base_res=16, finest_res=2048.0, res_cap=0, samples_per_ray=32,
                rays_per_iter=4096, precision=1, seed=1, network=1, hidden_layers=hidden_layers)


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


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def spawn_ranks(args):
    """--gpus N without a launcher: run this script under torch.distributed.run with
    N ranks on this node (rendezvous on 127.0.0.1), pass rank 0's JSON line through"""
    env = dict(os.environ)
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr=127.0.0.1", f"--master-port={_free_port()}", os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd, env=env)


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


def host_info():
    model = "unknown"
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                model = line.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    return {"cpu_model": model, "host_cores_available": len(os.sched_getaffinity(0))}


# ----------------------------------------------------------------------------- workloads
def cfg3_half_extents(gid):
    """cfg3 family member gid: edges U(0.2, 1.5) m per axis (BASELINE cfg2/3), seeded by the global id"""
    import numpy as np
    g = np.random.default_rng(3000 + gid)
    return (g.uniform(0.2, 1.5, size=3) / 2).astype(np.float32)


def objects_for_rank(workload, args, ws, rank, precision):
    """[(global id, SceneObject, [frames], rays)] of this rank, model kwargs, description"""
    import scenes
    from paper_2304_05735_b200.shard import partition
    if workload in ("cfg1", "paper"):
        kw = paper_kwargs(args.log2_T or 16, args.hidden_layers) if workload == "paper" else cfg1_kwargs(precision)
        if args.log2_T and workload == "cfg1":
            kw["log2_T"] = args.log2_T
        if args.rays_per_iter:
            kw["rays_per_iter"] = args.rays_per_iter
        n_total = args.objects or ws * args.objects_per_gpu
        mine = partition([kw["rays_per_iter"] * kw["samples_per_ray"]] * n_total, ws)[rank]
        sc = scenes.object_scene(1, n_views=20)
        ob = sc.objects[0]
        return [(gid, ob, sc.frames, kw["rays_per_iter"]) for gid in mine], kw, sc
    if workload in ("cfg3", "cfg4"):
        kw = cfg1_kwargs(precision, rays=args.rays_per_iter or 2048)
        n_total = args.objects or 64
        mine = partition([kw["rays_per_iter"] * kw["samples_per_ray"]] * n_total, ws)[rank]
        out = []
        for gid in mine:
            sc = scenes.object_scene(1000 + gid, n_views=20, half_extents=cfg3_half_extents(gid))
            out.append((gid, sc.objects[0], sc.frames, kw["rays_per_iter"]))
        return out, kw, None
    raise ValueError(workload)


def cfg2_plan(seed=2, n_objects=8, n_frames=200, rays_per_object=4096, batches=6):
    """BASELINE cfg2: 8 room objects; keyframes K_o ~ U{5..40} of the frames where the
    object covers >= 1 % of the image (evenly spaced along the trajectory), revealed
    in `batches` batches; R_total = 4096 x n split by total keyframe mask area (largest
    remainder, >= 128 per object, R9)"""
    import numpy as np
    import scenes
    sc = scenes.room_scene(seed, n_objects=n_objects, n_frames=n_frames)
    g = np.random.default_rng(seed + 100)
    plan = []
    for ob in sc.objects:
        vis = scenes.visible_frames(sc, ob.instance_id, min_frac=0.01) or scenes.visible_frames(sc, ob.instance_id)
        if not vis:
            continue
        k = min(len(vis), int(g.integers(5, 41)))
        pick = [vis[int(round(i))] for i in np.linspace(0, len(vis) - 1, k)]
        area = sum(int((sc.frames[i].mask == ob.instance_id).sum()) for i in pick)
        plan.append({"ob": ob, "frames": pick, "batches": [list(b) for b in np.array_split(np.asarray(pick), batches)],
                     "area": area})
    total = rays_per_object * len(plan)
    areas = np.array([p["area"] for p in plan], float)
    share = total * areas / areas.sum()
    rays = np.maximum(np.floor(share).astype(int), 128)
    rem = total - rays.sum()
    if rem > 0:
        rays[np.argsort(-(share - np.floor(share)))[:rem]] += 1
    for p, r in zip(plan, rays):
        p["rays"] = int(r)
    return sc, plan


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
    # the fused kernel's own inputs: the sample record (u, d_i) + delta written by
    # k_samples (20 B) and the ray record (84 B) shared by the ray's N samples
    inputs = 20 + 84.0 / kw["samples_per_ray"]
    return {"mlp_fwd_flop": mlp_fwd, "mlp_bwd_flop": mlp_bwd, "gather_bytes": gather, "scatter_bytes": scatter,
            "input_bytes": inputs}


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


# measured ceiling of the fused kernel's request mix (profiles/r1_micro.md): random
# 16-B LDG.128 gathers + RED.v4.f32 scatters 1:1 over L2-resident tables, per SM and cycle
REQ_CEILING = 0.828
_MODEL_KEYS = ("levels", "log2_T", "base_res", "finest_res", "res_cap", "samples_per_ray", "precision", "network",
               "hidden_layers")


def request_roofline(kw, samples_per_launch, ms, sm_clk, n_sm):
    """L1 sector requests of the gathers + REDs per SM-cycle against the measured
    random-access ceiling; sectors per hit sample from the committed ncu capture of
    the same model (profiles/ncu_requests.json; per sample, so any ray count), else None."""
    try:
        entries = json.load(open(os.path.join(ROOT, "profiles", "ncu_requests.json")))["entries"]
    except Exception:
        return None
    key = lambda d: tuple(d.get(k, {"network": 0, "hidden_layers": 1}.get(k)) for k in _MODEL_KEYS)
    d = next((e for e in entries if key(e["kw"]) == key(kw)), None)
    if d is None:
        return None
    req = d["sectors_per_hit_sample"] * samples_per_launch
    achieved = req / (ms * 1e-3 * sm_clk * n_sm)
    return {"bound": "l1_l2_random_requests", "achieved": achieved, "peak": REQ_CEILING,
            "unit": "sector requests / SM / cycle", "frac": achieved / REQ_CEILING,
            "source": f"{d['sectors_per_hit_sample']:.1f} sectors per hit sample ({d['profile']}); "
                      "ceiling profiles/r1_micro.md"}


def roofline(prof, kw, precision, samples_per_launch, n_objs):
    peaks, src = load_measured_peaks()
    work = algorithmic_per_sample(kw, precision)
    stages = {k: v for k, v in prof.items() if v["launches"] > 0 and v["ms"] > 0 and k not in ("l2_flush",)}
    dom = max(stages, key=lambda k: stages[k]["ms"])
    st = stages[dom]
    ms = st["ms"] / st["launches"]
    sm_clk = peaks.get("sm_max_mhz", 1965.0) * 1e6
    if dom in ("fused_mixed",):
        # algorithmic bytes of the hash gathers + gradient atomics + the per-sample
        # inputs the kernel reads
        bytes_ = samples_per_launch * (work["gather_bytes"] + work["scatter_bytes"] + work["input_bytes"])
        achieved = bytes_ / (ms * 1e-3) / 1e9
        out = {"bound": "hbm", "achieved": achieved, "peak": peaks["hbm_gbs"], "unit": "GB/s"}
        rq = request_roofline(kw, samples_per_launch, ms, sm_clk, 148)
        if rq:
            out["request_roofline"] = rq
    elif dom in ("fwd_fp32", "bwd_fp32"):
        flop = samples_per_launch * (work["mlp_fwd_flop"] if dom == "fwd_fp32" else work["mlp_bwd_flop"])
        achieved = flop / (ms * 1e-3) / 1e12
        peak = 148 * 128 * 2 * sm_clk / 1e12           # fp32 FMA lanes x 2 FLOP x max SM clock
        out = {"bound": "alu", "achieved": achieved, "peak": peak, "unit": "TFLOP/s"}
    elif dom == "adam":
        bytes_ = kw["_n_params"] * n_objs * 32
        achieved = bytes_ / (ms * 1e-3) / 1e9
        out = {"bound": "hbm", "achieved": achieved, "peak": peaks["hbm_gbs"], "unit": "GB/s"}
    else:
        bytes_ = samples_per_launch * 24
        achieved = bytes_ / (ms * 1e-3) / 1e9
        out = {"bound": "hbm", "achieved": achieved, "peak": peaks["hbm_gbs"], "unit": "GB/s"}
    out["frac"] = out["achieved"] / out["peak"]
    out["kernel"] = dom
    out["ms_per_launch"] = ms
    out["algorithmic_bytes_per_hit_sample"] = work["gather_bytes"] + work["scatter_bytes"] + (
        work["input_bytes"] if dom == "fused_mixed" else 0)
    out["hit_samples_per_launch"] = samples_per_launch
    out["peak_source"] = src
    out["traffic"] = ncu_traffic(dom)
    return out


# ----------------------------------------------------------------------------- inference (8(a) a10, a11; cfg4)
def room_layout(obs, spacing=0.25):
    """non-overlapping room positions for render_scene: boxes on a square grid of
    cells sized by the largest footprint (object frame centre -> world t, yaw kept)"""
    import numpy as np
    n = len(obs)
    side = int(math.ceil(math.sqrt(n)))
    cell = 2.0 * max(float(np.hypot(ob.a[0], ob.a[1])) for ob in obs) + spacing
    out = []
    for i, ob in enumerate(obs):
        gx, gy = i % side, i // side
        out.append(np.array([(gx - (side - 1) / 2) * cell, (gy - (side - 1) / 2) * cell, float(ob.a[2])], np.float32))
    return out, side * cell


def room_poses(extent, n=10, f=525.0):
    import numpy as np
    import scenes
    K = np.array([f, f, 320.0, 240.0], np.float32)
    out = []
    for i in range(n):
        az = 2 * math.pi * i / n
        r = 0.75 * extent + 1.0
        cam = (r * math.cos(az), r * math.sin(az), 0.45 * extent + 1.0)
        out.append((scenes.look_at(cam, (0.0, 0.0, 0.2)), K))
    return out


def measure_inference(ctx, hs, obs, poses, torch):
    """cfg4-style inference on trained objects: density on the 128^3 vertex lattice
    spanning each object's box (marching-cubes input, R21) with device buffers, one
    640x480 render of the first object, and render_scene of all objects from the poses."""
    peaks, src = load_measured_peaks()
    lattices = []
    for ob in obs:
        a = [float(x) for x in ob.a]
        axes = [torch.linspace(-a[k], a[k], 128, device="cuda") for k in range(3)]
        lattices.append(torch.stack(torch.meshgrid(*axes, indexing="ij"), -1).reshape(-1, 3).float().contiguous())
    for h, P in zip(hs, lattices):
        ctx.query_density(h, P)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for h, P in zip(hs, lattices):
        ctx.query_density(h, P)
    e1.record()
    torch.cuda.synchronize()
    q_ms = e0.elapsed_time(e1)
    npts = sum(P.shape[0] for P in lattices)
    q_gbs = npts * 16 * 8 * 4 / (q_ms * 1e-3) / 1e9   # 16 levels x 8 corners x 4 B (fp16 F=2) per point
    T0, K0 = poses[0]
    ctx.render(hs[0], T0, K0, 640, 480, 128)
    t0 = time.perf_counter()
    ctx.render(hs[0], T0, K0, 640, 480, 128)
    r_s = time.perf_counter() - t0
    ctx.render_scene(hs, T0, K0, 640, 480, 128)
    t0 = time.perf_counter()
    for T, K in poses:
        rgb, dep, opa = ctx.render_scene(hs, T, K, 640, 480, 128)
    rs_s = (time.perf_counter() - t0) / len(poses)
    # f2 mesh extraction at the paper's 64^3 (2.84 ms per object incl.
    # marching cubes): lattice + density + marching tetrahedra + triangles to the host
    nm = min(len(hs), 8)
    ctx.extract_mesh(hs[0], 64, 20.0)
    t0 = time.perf_counter()
    tris = [ctx.extract_mesh(h, 64, 20.0) for h in hs[:nm]]
    mesh_s = (time.perf_counter() - t0) / nm
    return {"mesh": {"objects": nm, "lattice": "65^3 vertices (64^3 cells)", "ms_per_object": mesh_s * 1e3,
                     "triangles_per_object": float(sum(len(t) for t in tris)) / nm, "paper_ms_per_object": 2.84,
                     "what": "romap_extract_mesh (k_lattice, density query, marching tetrahedra count / scan / emit), "
                             "world-frame triangles copied to the host, wall clock"},
            "query_density": {"objects": len(hs), "points": int(npts), "points_per_s": npts / (q_ms * 1e-3),
                              "ms_per_object_lattice": q_ms / len(hs),
                              "what": "128^3 vertex lattice per object box, device buffers, CUDA events (mixed path: "
                                      "fp16 tables + tcgen05 first layer)",
                              "roofline": {"bound": "hbm", "achieved": q_gbs, "peak": peaks["hbm_gbs"], "unit": "GB/s",
                                           "frac": q_gbs / peaks["hbm_gbs"], "peak_source": src,
                                           "note": "algorithmic gather bytes; each 3.4 MB table is L2-resident, so the "
                                                   "random-request rate, not HBM, binds it"}},
            "render": {"rays_per_s": 640 * 480 / r_s, "ms_per_frame": r_s * 1e3, "samples_per_ray": 128,
                       "what": "one 640x480 frame of one object, host outputs, wall clock"},
            "render_scene": {"objects": len(hs), "poses": len(poses), "ms_per_frame": rs_s * 1e3,
                             "rays_per_s": 640 * 480 / rs_s, "hit_pixels_last_pose": int((opa > 0).sum()),
                             "what": "romap_render_scene of all objects, 640x480, <= 128 samples per segment, "
                                     "host outputs, wall clock"}}


# ----------------------------------------------------------------------------- CPU oracle
def oracle_run(ob, frames, kw, rays, iters, obj_id=0):
    import oracle as O
    from threadpoolctl import threadpool_limits
    ocfg = O.ModelConfig(**{k: v for k, v in kw.items() if k in O.ModelConfig.__dataclass_fields__})
    ocfg.rays_per_iter = rays
    st = O.ObjectState(ocfg, ob.t, ob.yaw, ob.a, obj_id, O.init_params(ocfg, 0))
    for fr in frames:
        st.kfs.append(O.ingest_observation(fr.rgb, fr.mask, fr.T_wc, fr.K, ob.instance_id))
    with threadpool_limits(1):                   # the plain oracle, one core (BLAS pinned to 1 thread)
        O.train_iteration(st)                    # warm-up
        t0 = time.perf_counter()
        samples = 0
        for _ in range(iters):
            L, _, _ = O.train_iteration(st)
            samples += L["samples"]
        dt = time.perf_counter() - t0
    return samples, dt


def cpu_baseline(ob, frames, kw, rays=1024, iters=8):
    samples, dt = oracle_run(ob, frames, kw, rays, iters)
    return dict({"value": samples / dt, "unit": "ray-samples/s", "cores": 1, "kind": "oracle",
                 "sample": f"{iters} oracle iterations of one object of this workload at {rays} rays x "
                           f"{kw['samples_per_ray']} samples (numpy, fp32 geometry / fp64 arithmetic, BLAS limited "
                           f"to 1 thread; {samples} ray-samples in {dt:.1f} s)"}, **host_info())


# ----------------------------------------------------------------------------- reference arm
def run_reference(args):
    ws, rank, _ = dist_env()
    if rank != 0:
        return 0
    import scenes
    workload = resolve_workload(args, args.gpus)
    kw = cfg1_kwargs(0, rays=2048 if workload in ("cfg3", "cfg4") else 4096)
    if workload == "paper":
        kw = paper_kwargs(args.log2_T or 16, args.hidden_layers)
    if workload in ("cfg3", "cfg4"):
        sc = scenes.object_scene(1000, n_views=20, half_extents=cfg3_half_extents(0))
    else:
        sc = scenes.object_scene(1, n_views=20)
    ob = sc.objects[0]
    rays = 256
    for _ in range(args.warmup):
        oracle_run(ob, sc.frames, kw, rays, 1)
    samples, dt = oracle_run(ob, sc.frames, kw, rays, args.steps)
    v = samples / dt
    line = {"impl": "reference", "metric": "NeRF train ray-samples/s", "value": v, "unit": "ray-samples/s",
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup, "ms_per_step": dt / args.steps * 1e3,
            "higher_is_better": True, "scaling": "strong" if workload in ("cfg3", "cfg4") else "weak",
            "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded box-union-torus SDF object, 20 keyframes 640x480)",
            "config": {"workload": f"{workload} (reference = the CPU oracle on one object, bounded sample)",
                       "rays_per_iter": rays, "samples_per_ray": kw["samples_per_ray"], "levels": kw["levels"],
                       "log2_T": kw["log2_T"]},
            "cpu_baseline": dict({"value": v, "unit": "ray-samples/s", "cores": 1, "kind": "oracle",
                                  "sample": f"{args.steps} oracle iterations at {rays} rays x {kw['samples_per_ray']} "
                                            "samples, BLAS limited to 1 thread"}, **host_info()),
            "e2e": {"value": v, "unit": "ray-samples/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


# ----------------------------------------------------------------------------- dry run (CPU, gloo)
def run_dry(args):
    """the multi-rank path without a GPU: launcher, LPT partition of the workload's
    objects, end-of-run reduction (gloo), JSON line; no kernels, no data"""
    import torch
    import torch.distributed as dist
    from paper_2304_05735_b200.shard import partition, reduce_throughput
    ws, rank, _ = dist_env()
    if ws > 1:
        dist.init_process_group("gloo")
    workload = resolve_workload(args, ws)
    rays = args.rays_per_iter or (2048 if workload in ("cfg3", "cfg4") else 4096)
    n_total = args.objects or (64 if workload in ("cfg3", "cfg4") else ws * args.objects_per_gpu)
    mine = partition([rays * 64] * n_total, ws)[rank]
    samples = len(mine) * rays * 64 * args.steps
    elapsed_ms = 1.0 + rank                       # stand-in per-rank device times
    pg = dist if ws > 1 else None
    t_max, tot, value = reduce_throughput(elapsed_ms, samples, pg)
    objs = [None] * ws
    if ws > 1:
        dist.all_gather_object(objs, mine)
    else:
        objs = [mine]
    if rank == 0:
        print(json.dumps({"metric": "NeRF train ray-samples/s", "value": value, "unit": "ray-samples/s",
                          "n_gpus": ws, "steps": args.steps, "warmup": args.warmup, "dry_run": True,
                          "config": {"workload": workload, "objects": n_total, "rays_per_iter": rays},
                          "partition": objs, "max_ms": t_max, "total_samples": tot}), flush=True)
    if ws > 1:
        dist.barrier()
        dist.destroy_process_group()
    return 0


def resolve_workload(args, ws):
    if args.network == "paper":
        return "paper"
    if args.workload != "auto":
        return args.workload
    return "cfg3" if ws > 1 else "cfg1"


# ----------------------------------------------------------------------------- our arm
def timed_train(ctx, hs, steps, precision, pg, torch, local, flush=True):
    """exactly `steps` iterations of all objects in ONE train_step call (device-timed;
    flush: L2 flushed before each iteration, flush time subtracted; else the working
    set of the objects on the GPU is larger than L2); returns stats, timing"""
    ctx.set_l2_flush(FLUSH_BYTES if flush else 0)
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
    stats = ctx.train_step(hs, steps)
    host_ms = (time.perf_counter() - th0) * 1e3
    ev1.record(stream)
    torch.cuda.synchronize()
    if pg:
        pg.barrier()
    clocks = stop_clock_sampler(sampler, spath)
    prof = ctx.profile_read()
    # separate, untimed pass: every stage bracketed with events (breakdown only)
    ctx.profile_enable(True)
    n_brk = min(10, steps)
    ctx.train_step(hs, n_brk)
    prof_all = ctx.profile_read()
    ctx.profile_enable(False)
    ctx.set_l2_flush(0)
    total_ms = ev0.elapsed_time(ev1)
    flush_ms = prof.get("l2_flush", {}).get("ms", 0.0)
    return {"stats": stats, "total_ms": total_ms, "flush_ms": flush_ms, "step_ms": (total_ms - flush_ms) / steps,
            "host_ms": host_ms, "prof": prof, "prof_all": prof_all, "n_brk": n_brk, "clocks": clocks,
            "dominant": dominant}


def run_ours(args):
    import numpy as np
    import torch

    ws, rank, local = dist_env()
    # ROMAP_BENCH_SHARE_GPU=1: every rank on cuda:0 with a gloo reduction -- a check of
    # the multi-rank launcher on a one-GPU box (ranks never wait on each other's
    # kernels; not a measurement of scaling)
    share = os.environ.get("ROMAP_BENCH_SHARE_GPU") == "1"
    if share:
        local = 0
    torch.cuda.set_device(local)
    pg = None
    red_dev = "cpu" if share else "cuda"
    if ws > 1:
        import torch.distributed as dist
        if share:
            dist.init_process_group("gloo")
        else:
            # the communicator's rank / device map in the log (stderr: stdout carries the JSON line)
            os.environ.setdefault("NCCL_DEBUG", "INFO")
            os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
            os.environ.setdefault("NCCL_DEBUG_FILE", "/dev/stderr")
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        pg = dist
    from paper_2304_05735_b200 import romap as R
    from paper_2304_05735_b200.shard import reduce_throughput

    ctx = R.Context(local)
    precision = 0 if args.precision == "fp32" else 1
    workload = resolve_workload(args, ws)
    if workload == "cfg2":
        return run_cfg2(args, ctx, R, torch, precision)
    if workload == "online":
        return run_online(args, ctx, R, torch, precision)
    if workload == "paper":
        precision = 1
    items, kw, _ = objects_for_rank(workload, args, ws, rank, precision)
    hs, obs = [], []
    for gid, ob, frames, rays in items:
        h = ctx.create_object(ob.t, ob.yaw, ob.a, R.model_config(**kw), ob.instance_id, obj_id=gid)
        for fr in frames[:args.keyframes]:
            ctx.add_observation(h, fr.rgb, fr.mask, fr.T_wc, fr.K)
        hs.append(h)
        obs.append((ob, frames))
    info = ctx.object_info(hs[0])
    kw["_n_params"] = info["table_params"] + info["mlp_params"]

    ctx.train_step(hs, args.warmup)                   # warm-up (untimed)
    torch.cuda.synchronize()
    # L2 rule: flushed between iterations at every N (also where the rank's working set
    # alone exceeds L2, so per-N values stay comparable for the scaling curve)
    flush = True
    tr = timed_train(ctx, hs, args.steps, precision, pg, torch, local, flush)
    samples = sum(s["samples"] for s in tr["stats"])
    launches = sum(v["launches"] for k, v in tr["prof"].items() if k not in ("l2_flush", "graph_replay"))

    # e2e through the public API with HOST buffers: one new keyframe per object
    # (640x480 rgb + mask from pinned host memory) -> add_observation -> train_step(e2e_iters)
    # -> per-object stats read back to the host
    pinned = []
    for ob, frames in obs:
        fr = frames[-1]
        # bytes the library copies host -> device for this keyframe (the in-box crop as
        # uchar4 + its descriptor and prefix entry), counted here, outside the timed region
        ys, xs = np.nonzero(fr.mask == ob.instance_id)
        kf_bytes = int((xs.max() - xs.min() + 1) * (ys.max() - ys.min() + 1) * 4 + 96 + 8)
        pinned.append((torch.from_numpy(fr.rgb).pin_memory(), torch.from_numpy(fr.mask.astype(np.int16)).pin_memory(),
                       fr, kf_bytes))
    h2d, e2e_samples = 0, 0
    if pg:
        pg.barrier()
    torch.cuda.synchronize()
    # device-timed (CUDA events on torch's stream; the library's blocking stream is
    # ordered with it), so the host work between the records (ingest, enqueue, the
    # statistics read) is inside the interval
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    t0 = time.perf_counter()
    for _ in range(args.e2e_steps):
        for h, (rgb, mask, fr, kf_bytes) in zip(hs, pinned):
            ctx.add_observation(h, rgb.numpy(), mask.numpy().view(np.uint16), fr.T_wc, fr.K)
            h2d += kf_bytes
        st = ctx.train_step(hs, args.e2e_iters)
        e2e_samples += sum(s["samples"] for s in st)
    e1.record()
    torch.cuda.synchronize()
    e2e_wall_s = time.perf_counter() - t0
    e2e_s = e0.elapsed_time(e1) * 1e-3
    if pg:
        pg.barrier()

    # reductions over ranks: max time, sum of samples (NCCL all_reduce, shard.reduce_throughput)
    own_ms = tr["step_ms"] * args.steps
    t_max_ms, tot_samples, value = reduce_throughput(own_ms, samples, pg, device=red_dev)
    e2e_max_ms, tot_e2e, e2e_value = reduce_throughput(e2e_s * 1e3, e2e_samples, pg, device=red_dev)
    per_gpu = [samples / (own_ms * 1e-3)]
    devices = [torch.cuda.get_device_name(local)]
    if pg:
        g = [None] * ws
        pg.all_gather_object(g, (samples / (own_ms * 1e-3), torch.cuda.get_device_name(local), local))
        per_gpu = [x[0] for x in g]
        devices = [f"rank {r}: cuda:{x[2]} {x[1]}" for r, x in enumerate(g)]

    infer = None
    if rank == 0 and not args.no_inference:
        if workload == "cfg4":
            # the trained objects placed in one room (romap_set_box keeps the learned field, R27)
            ts, extent = room_layout([ob for ob, _ in obs])
            for h, (ob, _), t in zip(hs, obs, ts):
                ctx.set_box(h, t, ob.yaw, ob.a)
            poses = room_poses(extent)
        else:
            poses = [(fr.T_wc, fr.K) for fr in obs[0][1][:10]]
        infer = measure_inference(ctx, hs, [ob for ob, _ in obs], poses, torch)
    if rank == 0:
        rf = roofline(tr["prof"], kw, precision, samples / args.steps, len(hs))
        paper_sps = paper_baseline_samples_per_s(kw)
        if workload == "paper":
            desc = (f"paper network (PAPER.md:222, R24): L=16 F=2 T=2^{kw['log2_T']} res 16->2048, "
                    f"{kw['hidden_layers']} hidden layer(s) of 64 on positions -> sigma, rgb, {kw['rays_per_iter']} "
                    f"rays x 32 stratified samples per object, Adam")
        else:
            desc = (f"L=16 F=2 T=2^{kw['log2_T']} res 16->512, density 32->64->16 + SH4 colour 32->64->64->3, "
                    f"{kw['rays_per_iter']} rays x 64 stratified samples per object, Adam")
        objs_total = args.objects or (64 if workload in ("cfg3", "cfg4") else ws * args.objects_per_gpu)
        # the oracle's CPU baseline: rank 0 at N = 1 only (the contract; a multi-GPU run stays short)
        cpu = None if (args.no_cpu_baseline or ws > 1) else cpu_baseline(obs[0][0], obs[0][1], kw)
        t_iter_obj_ms = (t_max_ms / args.steps) / len(hs)
        strong = workload in ("cfg3", "cfg4") or bool(args.objects)
        line = {
            "metric": "NeRF train ray-samples/s", "value": value, "unit": "ray-samples/s", "n_gpus": ws,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": t_max_ms / args.steps,
            "higher_is_better": True, "scaling": "strong" if strong else "weak",
            "vs_baseline": (value / paper_sps) if paper_sps else None,
            "dtype": "f16-mma/f32" if precision == 1 else "f32",
            "data": ("synthetic: seeded box-union-torus SDF objects of the cfg1 family on a textured floor, 20 "
                     "keyframes 640x480 each, 1 cm pose jitter (stand-in for the paper's sequences, DESIGN.md 5)"),
            "config": {"workload": f"{workload}: {objs_total} object(s) over {ws} GPU(s), {len(hs)} on rank 0 "
                                   f"(LPT by cost, global ids kept), " + desc,
                       "objects_total": objs_total, "objects_rank0": len(hs), "rays_per_iter": kw["rays_per_iter"],
                       "samples_per_ray": kw["samples_per_ray"], "keyframes": args.keyframes,
                       "precision": "mixed" if precision == 1 else "fp32",
                       "l2": f"flushed before every iteration ({FLUSH_BYTES >> 20} MiB write by romap_set_l2_flush), "
                             "flush time excluded via the library's CUDA events",
                       "parallelism": f"objects sharded over {ws} rank(s), {'gloo (shared-GPU launcher check)' if share else 'NCCL'} "
                                      "only for the final max/sum"},
            "per_gpu_value": per_gpu,
            "ranks": devices,
            "s_to_budget_per_object": {
                "config_iterations": CONFIG_ITERS[workload],
                "s_config": t_iter_obj_ms * CONFIG_ITERS[workload] / 1e3,
                "s_paper_budget": t_iter_obj_ms * PAPER_ITERS_TO_BUDGET / 1e3,
                "paper_s": 2.0,
                "note": "SURVEY 8(d): (i) the config's own iteration count, (ii) the paper's ~2 s = 2833 iterations "
                        "of 0.706 ms (PAPER.md:307,320); GPU time per iteration / objects on the GPU"},
            "ms_per_iteration_per_object": t_iter_obj_ms,
            "paper_context": {"samples_per_s": PAPER_SAMPLES_PER_S, "ms_per_iteration": 0.706,
                              "note": ("RTX 4090, N=32, position-only 1x64 MLP (PAPER.md:222,307); "
                                       + ("this workload (vs_baseline = value / the paper's rate)" if paper_sps
                                          else "not this workload"))},
            "hit_samples_per_step": samples / args.steps,
            "stage_ms_per_step": {k: v["ms"] / tr["n_brk"] for k, v in tr["prof_all"].items() if v["ms"]},
            "stage_ms_note": f"separate {tr['n_brk']}-iteration pass with every stage bracketed by events",
            "kernel_ms_per_step": sum(v["ms"] for k, v in tr["prof_all"].items() if k != "l2_flush") / tr["n_brk"],
            "timed_region": {"total_ms": tr["total_ms"], "l2_flush_ms_subtracted": tr["flush_ms"],
                             "host_ms_in_call": tr["host_ms"], "dominant_ms": tr["prof"].get(tr["dominant"], {}).get("ms")},
            "gpu_launches": launches,
            "roofline": rf,
            "cpu_baseline": cpu,
            "e2e": {"value": e2e_value, "unit": "ray-samples/s", "h2d_bytes_per_step": int(h2d / max(1, args.e2e_steps)),
                    "d2h_bytes_per_step": int(len(hs) * 72 + 4),
                    "step": f"add_observation(1 keyframe per object, host) + train_step({args.e2e_iters} iterations, "
                            "graph replay) + per-object stats D2H",
                    "timing": "CUDA events around the e2e steps (max over ranks)", "wall_s_rank0": e2e_wall_s},
            "clocks": tr["clocks"],
            "inference": infer,
        }
        print(json.dumps(line), flush=True)
    ctx.close()
    if pg:
        pg.destroy_process_group()
    return 0


def run_cfg2(args, ctx, R, torch, precision):
    """BASELINE cfg2 on one GPU: 8 room objects batched in one launch with rays split by
    mask area; keyframes appended in 6 batches before iterations 0, 50, ..., 250; the
    whole schedule (appends included) is the timed region (CUDA events)."""
    import numpy as np
    sc, plan = cfg2_plan()
    kw = cfg1_kwargs(precision)

    def setup():
        hs = []
        for k, p in enumerate(plan):
            ob = p["ob"]
            h = ctx.create_object(ob.t, ob.yaw, ob.a, R.model_config(**dict(kw, rays_per_iter=p["rays"])),
                                  ob.instance_id, obj_id=k)
            hs.append(h)
        return hs

    def run(hs, iters, timed):
        samples, done, b = 0, 0, 0
        append_s = 0.0
        while done < iters:
            if b < 6 and done == 50 * b:
                t0 = time.perf_counter()
                for h, p in zip(hs, plan):
                    for fi in p["batches"][b]:
                        fr = sc.frames[fi]
                        ctx.add_observation(h, fr.rgb, fr.mask, fr.T_wc, fr.K)
                append_s += time.perf_counter() - t0
                b += 1
            n = min(iters - done, 50 * b - done if b < 6 else iters - done)
            st = ctx.train_step(hs, n)
            samples += sum(s["samples"] for s in st)
            done += n
        return samples, append_s

    hs = setup()
    run(hs, args.warmup, False)                      # warm-up objects (discarded)
    for h in hs:
        ctx.destroy_object(h)
    hs = setup()
    # the workload is the whole 300-iteration schedule (6 append batches), whatever --steps says
    steps = max(args.steps, CONFIG_ITERS["cfg2"])
    sampler, spath = start_clock_sampler(visible_index(0))
    time.sleep(0.3)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    p0 = ctx.profile_read()                           # launch counters are always kept
    torch.cuda.synchronize()
    e0.record()
    samples, append_s = run(hs, steps, True)
    e1.record()
    torch.cuda.synchronize()
    clocks = stop_clock_sampler(sampler, spath)
    p1 = ctx.profile_read()
    launches = sum(p1[k]["launches"] - p0[k]["launches"] for k in p1 if k not in ("l2_flush", "graph_replay"))
    ms = e0.elapsed_time(e1)
    value = samples / (ms * 1e-3)
    t_iter_obj_ms = ms / steps / len(hs)
    print(json.dumps({
        "metric": "NeRF train ray-samples/s", "value": value, "unit": "ray-samples/s", "n_gpus": 1,
        "steps": steps, "warmup": args.warmup, "ms_per_step": ms / steps, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f16-mma/f32" if precision == 1 else "f32",
        "data": "synthetic room (seed 2): 8 cfg1-family objects, edges U(0.2, 1.5) m, 200-frame 640x480 trajectory",
        "config": {"workload": "cfg2: 8 objects batched in one launch, rays split by keyframe mask area "
                               "(4096 x 8 total, >= 128 each), keyframes U{5..40} per object appended in 6 batches "
                               "before iterations 0, 50, ..., 250", "rays": [p["rays"] for p in plan],
                   "keyframes": [len(p["frames"]) for p in plan],
                   "l2": "not flushed (appends between chunks; the objects' tables live in L2 across iterations)"},
        "timed_region": {"total_ms": ms, "host_append_s": append_s, "includes": "add_observation of every batch"},
        "s_to_budget_per_object": {"config_iterations": 300, "s_config": t_iter_obj_ms * 300 / 1e3,
                                   "s_paper_budget": t_iter_obj_ms * PAPER_ITERS_TO_BUDGET / 1e3, "paper_s": 2.0},
        "ms_per_iteration_per_object": t_iter_obj_ms,
        "clocks": clocks, "cpu_baseline": None,
        "e2e": None, "e2e_note": "the timed region is itself end to end: host keyframe appends (add_observation from "
                                 "host buffers) and per-call statistics read-backs are inside it",
        "gpu_launches": launches}), flush=True)
    ctx.close()
    return 0


def run_online(args, ctx, R, torch, precision):
    """SURVEY f3 measured: the paper's online schedule on the cfg2 room.  The frames of
    the 200-frame trajectory arrive at --online-hz (the paper's SLAM rate, 25 Hz,
    PAPER.md:7,305); every object visible in a frame is offered to the asynchronous
    trainer (romap_async_offer: Eq. 5 gate at 25 deg, +300 iterations per accepted
    keyframe); after the last frame the worker finishes every
    pending budget.  Reports the producer's offer latency (it must never block), the
    keyframes accepted, and the iterations and drawn ray-samples per second of the
    trainer over the whole run."""
    import numpy as np
    sc, plan = cfg2_plan()
    kw = cfg1_kwargs(precision)
    hs = {}
    for k, p in enumerate(plan):
        ob = p["ob"]
        hs[ob.instance_id] = (ctx.create_object(ob.t, ob.yaw, ob.a, R.model_config(**dict(kw, rays_per_iter=p["rays"])),
                                                ob.instance_id, obj_id=k), p["rays"])
    period = 1.0 / args.online_hz if args.online_hz > 0 else 0.0
    ctx.async_start(chunk=50, alpha_deg=25.0, iters_per_update=300, queue_cap=256)
    lat = []
    t_start = time.perf_counter()
    for i, fr in enumerate(sc.frames):
        ids = [iid for iid in np.unique(fr.mask) if iid in hs]
        for iid in ids:
            t0 = time.perf_counter()
            ctx.async_offer(hs[iid][0], fr.rgb, fr.mask, fr.T_wc, fr.K)
            lat.append(time.perf_counter() - t0)
        if period:
            time.sleep(max(0.0, t_start + (i + 1) * period - time.perf_counter()))
    t_frames = time.perf_counter() - t_start
    st = ctx.async_stop(finish_pending=True)
    torch.cuda.synchronize()
    t_all = time.perf_counter() - t_start
    steps = {iid: int(ctx.get_params(h, R.BLOCK_STEP)[0]) for iid, (h, _) in hs.items()}
    drawn = sum(steps[iid] * rays * kw["samples_per_ray"] for iid, (_, rays) in hs.items())
    lat_ms = sorted(x * 1e3 for x in lat)
    print(json.dumps({
        "metric": "NeRF train ray-samples/s (online schedule)", "value": drawn / t_all, "unit": "drawn ray-samples/s",
        "n_gpus": 1, "higher_is_better": True, "dtype": "f16-mma/f32" if precision == 1 else "f32",
        "data": "synthetic room (seed 2): 8 cfg1-family objects, 200-frame 640x480 trajectory",
        "config": {"workload": f"online (SURVEY f3): frames at {args.online_hz} Hz, Eq. 5 gate 25 deg, 300 iterations "
                               "per accepted keyframe, async trainer (chunks of 50), rays split by mask area",
                   "rays": [r for _, r in hs.values()]},
        "producer": {"offers": len(lat), "offer_ms_median": lat_ms[len(lat_ms) // 2], "offer_ms_max": lat_ms[-1],
                     "frames_s": t_frames, "note": "a queue push; the producer never waits on the GPU"},
        "trainer": {"accepted_keyframes": st["accepted"], "rejected": st["rejected"], "dropped": st["dropped"],
                    "iterations_per_object": steps, "wall_s": t_all,
                    "s_after_last_frame": t_all - t_frames,
                    "note": "value = drawn ray-samples (steps x rays x N, misses included) / wall time of the run"}}),
          flush=True)
    ctx.close()
    return 0


def run_table4(args):
    """The paper's Table 4 grid on one GPU: ms per training iteration
    of one object (4096 rays x 32, a1..a8 incl. Adam, L2 flushed before each iteration)
    next to the paper's RTX 4090 numbers."""
    import torch
    import scenes
    from paper_2304_05735_b200 import romap as R

    ctx = R.Context(0)
    scene = scenes.object_scene(1, n_views=20)
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
    ap.add_argument("--online-hz", type=float, default=25.0, help="--workload online: frame rate of the producer")
    ap.add_argument("--workload", choices=["auto", "cfg1", "cfg2", "cfg3", "cfg4", "online"], default="auto",
                    help="auto: cfg1 at N=1 (BASELINE metric config), cfg3 (64 objects sharded) at N>1")
    ap.add_argument("--precision", choices=["auto", "mixed", "fp32"], default="auto")
    ap.add_argument("--objects-per-gpu", type=int, default=1, help="cfg1: objects per rank (weak scaling)")
    ap.add_argument("--objects", type=int, default=0, help="total objects over all ranks (cfg3 default 64)")
    ap.add_argument("--keyframes", type=int, default=20)
    ap.add_argument("--rays-per-iter", type=int, default=0, help="rays per object and iteration (0: the config's)")
    ap.add_argument("--e2e-steps", type=int, default=4)
    ap.add_argument("--e2e-iters", type=int, default=50)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-inference", action="store_true")
    ap.add_argument("--dry-run", action="store_true", help="launcher + partition + reduction only (CPU, gloo)")
    ap.add_argument("--network", choices=["baseline", "paper"], default="baseline",
                    help="baseline: BASELINE cfg1 (default, the headline); paper: PAPER.md:222 network (R24)")
    ap.add_argument("--hidden-layers", type=int, default=1, help="--network paper: hidden layers (Table 4: 1..3)")
    ap.add_argument("--log2-T", type=int, default=0, help="hash table size override (Table 4: 14..20)")
    ap.add_argument("--table4", action="store_true", help="run the paper's Table 4 sweep (PAPER.md:353-357)")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        return spawn_ranks(args)
    if args.impl == "reference":
        return run_reference(args)
    if args.dry_run:
        return run_dry(args)
    if args.table4:
        return run_table4(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
