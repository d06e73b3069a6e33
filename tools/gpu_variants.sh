#!/bin/bash
# run mixed-path parity + a short bench for the default build and every libromap_<v>.so variant given
mkdir -p gpurun_out
for v in base "$@"; do
  if [ "$v" = base ]; then export ROMAP_LIB=; else export ROMAP_LIB=$PWD/paper_2304_05735_b200/libromap_$v.so; fi
  timeout 300 python -m pytest tests/test_gpu_parity_mixed.py -q -x -p no:cacheprovider > gpurun_out/var_$v.log 2>&1
  rc=$?
  timeout 300 python bench.py --no-cpu-baseline --steps 30 --e2e-steps 1 > gpurun_out/var_$v.json 2>/dev/null
  python - "$v" "$rc" <<'PY'
import json, sys
v, rc = sys.argv[1], sys.argv[2]
try:
    d = json.loads(open(f"gpurun_out/var_{v}.json").read().strip().splitlines()[-1])
    print(f"{v:10s} parity_rc={rc} value {d['value']:.4e} fused {d['stage_ms_per_step']['fused_mixed']*1e3:.1f} us  step {d['ms_per_step']*1e3:.1f} us")
except Exception as e:
    print(v, "failed", rc, e)
PY
done
