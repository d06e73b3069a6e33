#!/bin/bash
# run mixed-path parity + a short bench for the default build and every libromap_<v>.so variant given
mkdir -p gpurun_out
for v in base "$@"; do
  if [ "$v" = base ]; then export ROMAP_LIB=; else export ROMAP_LIB=$PWD/paper_2304_05735_b200/libromap_$v.so; fi
  timeout 300 python -m pytest tests/test_gpu_parity_mixed.py -q -x -p no:cacheprovider > gpurun_out/var_$v.log 2>&1
  rc=$?
  timeout 300 python bench.py --no-cpu-baseline --no-inference --steps 30 --e2e-steps 1 > gpurun_out/var_$v.json 2>/dev/null
  # L1 sector requests of the fused kernel (gathers, REDs) for the variant
  timeout 600 ncu --metrics gpu__time_duration.sum,l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum,l1tex__t_sectors_pipe_lsu_mem_global_op_red.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum,l1tex__data_pipe_lsu_wavefronts.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared_op_misc.sum \
    --clock-control none -k regex:k_fused_mixed -s 3 -c 2 --csv --log-file gpurun_out/var_${v}_ncu.csv \
    python bench.py --no-cpu-baseline --no-inference --steps 5 --warmup 3 --e2e-steps 1 > /dev/null 2>&1
  python - "$v" "$rc" <<'PY'
import json, sys
v, rc = sys.argv[1], sys.argv[2]
try:
    d = json.loads(open(f"gpurun_out/var_{v}.json").read().strip().splitlines()[-1])
    import csv
    sec = {}
    try:
        rows = [r for r in csv.reader(open(f"gpurun_out/var_{v}_ncu.csv")) if len(r) > 14 and r[0].isdigit()]
        for r in rows:
            sec.setdefault(r[12], []).append(float(r[14].replace(",", "")))
    except Exception:
        pass
    hs = d["hit_samples_per_step"]
    ld = sum(sec.get("l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum", [0])) / max(1, len(sec.get("l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum", [0])))
    rd = sum(sec.get("l1tex__t_sectors_pipe_lsu_mem_global_op_red.sum", [0])) / max(1, len(sec.get("l1tex__t_sectors_pipe_lsu_mem_global_op_red.sum", [0])))
    avg = lambda k: sum(sec.get(k, [0])) / max(1, len(sec.get(k, [0])))
    shw, allw = avg("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum"), avg("l1tex__data_pipe_lsu_wavefronts.sum")
    print(f"{v:10s} parity_rc={rc} value {d['value']:.4e} fused {d['roofline']['ms_per_launch']*1e3:.1f} us  "
          f"step {d['ms_per_step']*1e3:.1f} us  ld/sample {ld / hs:.1f} red/sample {rd / hs:.1f}  "
          f"LSU wavefronts/sample {allw / hs:.1f} (shared {shw / hs:.1f}, misc "
          f"{avg('l1tex__data_pipe_lsu_wavefronts_mem_shared_op_misc.sum') / hs:.1f})")
except Exception as e:
    print(v, "failed", rc, e)
PY
done
