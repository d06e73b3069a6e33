#!/bin/bash
# refresh the measured results quoted in README / BASELINE.md / DESIGN.md (one gpurun call)
TAG=${1:-r}
mkdir -p gpurun_out
timeout 300 python bench.py --no-cpu-baseline > gpurun_out/res_${TAG}_cfg1.json 2> gpurun_out/res_${TAG}_cfg1.err; echo "cfg1 rc=$?"
timeout 300 python bench.py --no-cpu-baseline --network paper > gpurun_out/res_${TAG}_paper.json 2> gpurun_out/res_${TAG}_paper.err; echo "paper rc=$?"
timeout 300 python bench.py --no-cpu-baseline --objects-per-gpu 8 --steps 20 --warmup 5 > gpurun_out/res_${TAG}_obj8.json 2> gpurun_out/res_${TAG}_obj8.err; echo "obj8 rc=$?"
timeout 400 python bench.py --no-cpu-baseline --objects-per-gpu 32 --steps 10 --warmup 3 > gpurun_out/res_${TAG}_obj32.json 2> gpurun_out/res_${TAG}_obj32.err; echo "obj32 rc=$?"
timeout 900 python bench.py --no-cpu-baseline --table4 > gpurun_out/res_${TAG}_table4.json 2> gpurun_out/res_${TAG}_table4.err; echo "table4 rc=$?"
python - "$TAG" <<'PY'
import json, sys
t = sys.argv[1]
for k in ("cfg1", "paper", "obj8", "obj32"):
    try:
        d = json.loads(open(f"gpurun_out/res_{t}_{k}.json").read().strip().splitlines()[-1])
        rr = d.get("roofline", {})
        print(k, f"value {d['value']:.4e} ms/step {d['ms_per_step']*1e3:.1f} us vs_baseline {d.get('vs_baseline')} frac {rr.get('frac')} req {rr.get('request_roofline', {}).get('frac')}")
    except Exception as e:
        print(k, "failed", e)
PY
