"""Summarise an ncu launch list (csv) and an ncu --set full report into
profiles/<tag>_*.md / .json, and update profiles/ncu_traffic.json (dram bytes
per launch per stage) that bench.py reads for roofline.traffic."""
import collections
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
STAGE = {"k_raygen_samples": "raygen", "k_raygen": "raygen", "k_fwd_fp32": "fwd_fp32", "k_render_loss": "render_loss", "k_bwd_fp32": "bwd_fp32",
         "k_fused_mixed": "fused_mixed", "k_adam": "adam", "k_step_inc": "step_inc", "k_zero_grads": "zero_grads"}
METRICS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_bytes.sum",
           "sm__throughput.avg.pct_of_peak_sustained_elapsed", "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed",
           "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
           "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
           "sm__inst_executed_pipe_tensor.avg.pct_of_peak_sustained_active",
           "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
           "launch__grid_size", "launch__block_size", "smsp__inst_executed.sum",
           "l1tex__t_sector_hit_rate.pct", "lts__t_sector_hit_rate.pct",
           # request-rate roofline of the hash-grid gathers / scatters
           "l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum", "l1tex__t_sectors_pipe_lsu_mem_global_op_red.sum",
           "l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed",
           "lts__t_tag_requests.avg.pct_of_peak_sustained_elapsed",
           "lts__t_requests_srcunit_ltcfabric.sum", "sm__issue_active.avg.pct_of_peak_sustained_elapsed"]


def norm(name):
    """'void k_fused_mixed<16>(CfgDev, ...)' -> 'k_fused_mixed'"""
    n = name.split("(")[0].strip()
    if n.startswith("void "):
        n = n[5:]
    return n.split("<")[0].strip()


def launches(path):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
    hdr = rows[hi]
    ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    agg = collections.defaultdict(list)
    unit = None
    for r in rows[hi + 1:]:
        agg[norm(r[ki])].append(float(r[vi].replace(",", "")))
        unit = r[ui]
    scale = {"ns": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3, "nsecond": 1e-3}.get(unit, 1e-3)
    tot = sum(sum(v) for v in agg.values())
    return {k: {"n": len(v), "mean_us": sum(v) / len(v) * scale, "share": sum(v) / tot} for k, v in agg.items()}


def full(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        d = {"kernel": norm(r[hdr.index("Kernel Name")])}
        for m in METRICS:
            if m in hdr:
                d[m] = r[hdr.index(m)] + " " + units[hdr.index(m)]
        res.append(d)
    return res


def to_bytes(s):
    v, u = s.split()
    v = float(v.replace(",", ""))
    return v * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u, 1)


def main(tag, launch_csv, rep, hit_samples=None):
    os.makedirs(os.path.join(ROOT, "profiles"), exist_ok=True)
    L = launches(launch_csv) if launch_csv and os.path.exists(launch_csv) else {}
    F = full(rep) if rep and os.path.exists(rep) else []
    md = [f"# ncu summary {tag}", "", "## launch list (ncu --metrics gpu__time_duration.sum, cold-cache, serialised)", "",
          "| kernel | launches | mean us | share |", "|---|---|---|---|"]
    for k, v in sorted(L.items(), key=lambda x: -x[1]["share"]):
        md.append(f"| {k} | {v['n']} | {v['mean_us']:.1f} | {v['share']:.3f} |")
    md += ["", "## ncu --set full (per captured launch)", ""]
    traffic_path = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    traffic = json.load(open(traffic_path)) if os.path.exists(traffic_path) else {}
    for d in F:
        md.append(f"### {d['kernel']}")
        for m in METRICS:
            if m in d:
                md.append(f"- {m}: {d[m]}")
        md.append("")
        if "dram__bytes_read.sum" in d and d["kernel"] in STAGE:
            traffic[STAGE[d["kernel"]]] = to_bytes(d["dram__bytes_read.sum"]) + to_bytes(d["dram__bytes_write.sum"])
    # L1 sector requests (gathers + REDs) per hit ray-sample of the fused kernel:
    # bench.py's request roofline
    fm = [d for d in F if d["kernel"] == "k_fused_mixed" and "l1tex__t_sectors_pipe_lsu_mem_global_op_red.sum" in d]
    if fm and hit_samples:
        sec = [float(d["l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum"].split()[0]) +
               float(d["l1tex__t_sectors_pipe_lsu_mem_global_op_red.sum"].split()[0]) for d in fm]
        req = {"kernel": "k_fused_mixed", "profile": f"profiles/{tag}_ncu.json",
               "sectors_per_launch": sum(sec) / len(sec), "hit_samples_per_launch": float(hit_samples),
               "sectors_per_hit_sample": sum(sec) / len(sec) / float(hit_samples)}
        # (cfg1 entry of profiles/ncu_requests.json; other workloads are added by hand)
        path = os.path.join(ROOT, "profiles", "ncu_requests.json")
        try:
            allreq = json.load(open(path))
        except Exception:
            allreq = {"entries": []}
        req["workload"] = "cfg1"
        req["kw"] = {"levels": 16, "log2_T": 16, "base_res": 16, "finest_res": 512.0, "res_cap": 0,
                     "samples_per_ray": 64, "rays_per_iter": 4096, "precision": 1, "seed": 1}
        allreq["entries"] = [e for e in allreq.get("entries", []) if e.get("workload") != "cfg1"] + [req]
        json.dump(allreq, open(path, "w"), indent=1)
        md += ["## request rate", "", f"- L1 sector requests (global ld + red) per hit ray-sample: "
               f"{req['sectors_per_hit_sample']:.1f}", ""]
    open(os.path.join(ROOT, "profiles", f"{tag}_ncu.md"), "w").write("\n".join(md) + "\n")
    json.dump({"launches": L, "full": F}, open(os.path.join(ROOT, "profiles", f"{tag}_ncu.json"), "w"), indent=1)
    json.dump(traffic, open(traffic_path, "w"), indent=1)
    print("\n".join(md))


if __name__ == "__main__":
    # usage: ncu_summary.py <tag> [launch csv] [ncu-rep] [hit ray-samples per launch of the captured run]
    main(sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else None, sys.argv[3] if len(sys.argv) > 3 else None,
         sys.argv[4] if len(sys.argv) > 4 else None)
