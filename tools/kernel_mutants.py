"""Mutation testing of the CUDA path: does `pytest -m gpu` catch a plausible bug in
the kernels?  Each mutant below is one wrong operand / index / sign / dropped term
in a kernel source (the measured fused kernel, raygen, Adam, the shared hash
helpers).  `build` compiles every mutant here (nvcc cross-compiles; only the
objects that include the mutated file are rebuilt -- both builds of the fused
kernel, every object for a header -- the rest are the tree's own objects) into
paper_2304_05735_b200/mutants/libromap_<k>.so; `run` (on the GPU box) runs the
whole GPU suite against each library via ROMAP_LIB and lists the tests that
failed (a mutant is killed when at least one does).  Results: profiles/r2_kernel_mutants.txt, DESIGN.md section 4.

    python tools/kernel_mutants.py build [k0]   # here (CPU), after `make` in csrc/ (mutants k0..)
    python tools/kernel_mutants.py run [k0]     # on the GPU box
"""
import concurrent.futures
import os
import shutil
import subprocess
import sys
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CSRC = os.path.join(ROOT, "paper_2304_05735_b200", "csrc")
OUT = os.path.join(ROOT, "paper_2304_05735_b200", "mutants")
NVCC = "/usr/local/cuda/bin/nvcc"
FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC",
         "-Xcompiler", "-fvisibility=hidden", "--expt-relaxed-constexpr"]
OBJS = ["romap_api.o", "k_sample.o", "k_fp32.o", "k_adam.o", "k_fused_mixed.o", "k_infer_mixed.o", "k_mesh.o",
        "k_selftest.o", "k_det.o", "k_scene.o", "k_fused_mixed_det.o"]

FUSED = ["k_fused_mixed.o", "k_fused_mixed_det.o"]      # both builds of the fused kernel carry the bug
ALL = OBJS                                              # a header bug reaches every object that includes it

# (name, mutated file, old text (must occur once), new text, objects to rebuild)
MUTANTS = [
    ("scatter x-weight swapped", "k_fused_mixed.cu", "v[4 * p] = wa * g0;", "v[4 * p] = wb * g0;", FUSED),
    ("gather x lerp reversed", "k_fused_mixed.cu",
     "vx32[p] = make_float2(a.x + cl[q].f[0] * (c.x - a.x)", "vx32[p] = make_float2(c.x + cl[q].f[0] * (a.x - c.x)",
     FUSED),
    ("RED pair slots swapped", "k_fused_mixed.cu", "const float4 w4 = a_lo ? make_float4",
     "const float4 w4 = !a_lo ? make_float4", FUSED),
    ("coarse merge: every lane issues", "k_fused_mixed.cu", "issue = as_ && ((lane - run0) & wmask) == 0;",
     "issue = as_;", FUSED),
    ("loss scale not divided out", "k_fused_mixed.cu", "const float g0 = as_ ? g[2 * q] * inv_scale : 0.f",
     "const float g0 = as_ ? g[2 * q] : 0.f", FUSED),
    ("background term dropped", "k_fused_mixed.cu", "e[k] = sums[k] + TN * bgc[k] - (cls", "e[k] = sums[k] - (cls",
     FUSED),
    ("density-loss gradient on object rays", "k_fused_mixed.cu",
     "(cls == CLS_BG ? cfg.lambda_density * invB : 0.f);", "(cls == CLS_OBJ ? cfg.lambda_density * invB : 0.f);",
     FUSED),
    ("render transmittance inclusive", "k_fused_mixed.cu",
     "float Tl = __shfl_up_sync(0xffffffffu, incl, 1, sw);\n    if (sl == 0) Tl = 1.f;", "float Tl = incl;",
     FUSED),
    ("sigmoid derivative dropped", "k_fused_mixed.cu",
     "for (int k = 0; k < 3; ++k) v[k] = dcol[k] * c[k] * (1.f - c[k]) * scale;",
     "for (int k = 0; k < 3; ++k) v[k] = dcol[k] * c[k] * scale;", FUSED),
    ("ReLU mask dropped in the backward epilogue", "k_fused_mixed.cu",
     "q[k] = __hmul2(__floats2half2_rn(v[8 * c + 2 * k], v[8 * c + 2 * k + 1]), __hgt2(a[k], z));",
     "q[k] = __floats2half2_rn(v[8 * c + 2 * k], v[8 * c + 2 * k + 1]);", FUSED),
    ("hash primes y/z swapped", "hash_fp16.cuh",
     "(int)(dense ? n1 : 2654435761u), (int)(dense ? n1 * n1 : 805459861u)",
     "(int)(dense ? n1 : 805459861u), (int)(dense ? n1 * n1 : 2654435761u)", ALL),
    ("dense x-neighbour = base corner", "hash_fp16.cuh", "e[2 * k + 1] = x1 + yz[k];",
     "e[2 * k + 1] = x0 + yz[k];", ALL),
    ("Adam bias correction dropped", "k_adam.cu", "p[j] = p[j] - lr * (mj * ibc1) / (sqrtf(vj * ibc2) + eps);",
     "p[j] = p[j] - lr * mj / (sqrtf(vj) + eps);", ["k_adam.o"]),
    ("Adam sparse test on the MLP too", "k_adam.cu", "if (i0 + j < n_table && gj == 0.f) continue;",
     "if (gj == 0.f) continue;", ["k_adam.o"]),
    ("raygen background stream + 1", "k_sample.cu", "rr.bg[k] = u32_unit(rng_u32(pre, r, 1 + k));",
     "rr.bg[k] = u32_unit(rng_u32(pre, r, 2 + k));", ["k_sample.o"]),
    ("raygen pixel centre dropped", "romap_internal.cuh", "float pxf = __fadd_rn((float)px, 0.5f);",
     "float pxf = (float)px;", ALL),
    # the other rows: slab, fp32 path, inference, scene compositing, mesh, deterministic reductions
    ("slab t_near not clamped at 0", "romap_internal.cuh", "    tn = 0.0f;\n", "    tn = -3.0e38f;\n", ALL),
    ("fp32 backward: ReLU mask of g1 dropped", "k_fp32.cu", "dg1[k] = v64[k] > 0.f ? acc : 0.f;", "dg1[k] = acc;",
     ["k_fp32.o"]),
    ("density query: outside-box zero dropped", "k_infer_mixed.cu",
     "if (valid) out[p] = inside ? density_act(raw0, cfg.density_act) : 0.f;",
     "if (valid) out[p] = density_act(raw0, cfg.density_act);", ["k_infer_mixed.o"]),
    ("mixed render: midpoints at 1/4 of the stratum", "k_infer_mixed.cu", "dist = sample_dist(rr.tn, Dl, i, 0.5f);",
     "dist = sample_dist(rr.tn, Dl, i, 0.25f);", ["k_infer_mixed.o"]),
    ("render_scene: transmittance not carried", "k_scene.cu", "T *= 1.0f - segA[best];", "T *= 1.0f;",
     ["k_scene.o"]),
    ("marching tetrahedra: edge weight reversed", "k_mesh.cu", "const float w = (iso - sa) / (sb - sa);",
     "const float w = (sb - iso) / (sb - sa);", ["k_mesh.o"]),
    ("deterministic mode: first record of a run skipped", "k_det.cu",
     "for (long long j = i; j < n && key[j] == k; ++j) {", "for (long long j = i + 1; j < n && key[j] == k; ++j) {",
     ["k_det.o"]),
    ("deterministic mode: first tile's dW skipped", "k_det.cu", "for (long long t = t0; t < t1; ++t) s +=",
     "for (long long t = t0 + 1; t < t1; ++t) s +=", ["k_det.o"]),
]


def _build_one(k):
    name, fname, old, new, objs = MUTANTS[k]
    tmp = tempfile.mkdtemp(prefix=f"km{k:02d}_")
    try:
        src = os.path.join(tmp, "paper_2304_05735_b200", "csrc")
        shutil.copytree(CSRC, src, ignore=shutil.ignore_patterns("*.log", "kfm_*"))
        os.makedirs(os.path.join(tmp, "include"))
        shutil.copy(os.path.join(ROOT, "include", "romap.h"), os.path.join(tmp, "include"))
        path = os.path.join(src, fname)
        text = open(path).read()
        if text.count(old) != 1:
            return k, f"pattern count {text.count(old)}"
        open(path, "w").write(text.replace(old, new))
        for o in objs:
            det = o == "k_fused_mixed_det.o"                   # -DROMAP_DET build of k_fused_mixed.cu
            cu = "k_fused_mixed.cu" if det else o[:-2] + ".cu"
            extra = ["-DROMAP_DET"] if det else []
            r = subprocess.run([NVCC] + FLAGS + extra + ["-c", cu, "-o", o], cwd=src, capture_output=True, text=True)
            if r.returncode:
                return k, "compile failed: " + r.stderr[-500:]
        os.makedirs(OUT, exist_ok=True)
        lib = os.path.join(OUT, f"libromap_{k:02d}.so")
        r = subprocess.run([NVCC, "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-o", lib] + OBJS +
                           ["-Xcompiler", "-fvisibility=hidden"], cwd=src, capture_output=True, text=True)
        return k, "ok" if r.returncode == 0 else "link failed: " + r.stderr[-500:]
    finally:
        shutil.rmtree(tmp, ignore_errors=True)


def build(start=0):
    missing = [o for o in OBJS if not os.path.exists(os.path.join(CSRC, o))]
    if missing:
        sys.exit(f"build the tree first (make in {CSRC}); missing {missing}")
    with concurrent.futures.ThreadPoolExecutor(max(1, min(8, os.cpu_count() or 1))) as ex:
        for k, status in ex.map(_build_one, range(start, len(MUTANTS))):
            print(f"{k:02d} {MUTANTS[k][0]}: {status}", flush=True)


def run(start=0):
    print("mutant | GPU tests failed (of the whole suite) | rc, pytest summary", flush=True)
    for k, m in enumerate(MUTANTS):
        if k < start:
            continue
        lib = os.path.join(OUT, f"libromap_{k:02d}.so")
        env = dict(os.environ, ROMAP_LIB=lib)
        r = subprocess.run(["timeout", "900", sys.executable, "-m", "pytest", "tests", "-m", "gpu", "-q", "-rfE",
                            "-p", "no:cacheprovider"], cwd=ROOT, env=env, capture_output=True, text=True)
        failed = sorted({ln.split(" ")[1].split("::")[-1].split("[")[0] for ln in r.stdout.splitlines()
                         if ln.startswith(("FAILED ", "ERROR "))})
        tail = r.stdout.strip().splitlines()[-1] if r.stdout.strip() else r.stderr[-200:]
        verdict = f"{len(failed)} failing: " + ", ".join(failed) if failed else (
            "SURVIVED" if r.returncode == 0 else f"rc {r.returncode}")
        print(f"{k:02d} {m[0]} | {verdict} | {r.returncode} ({tail})", flush=True)


if __name__ == "__main__":
    {"build": build, "run": run}[sys.argv[1]](int(sys.argv[2]) if len(sys.argv) > 2 else 0)
