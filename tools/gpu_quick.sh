#!/bin/bash
# quick GPU iteration: mixed parity + bench (no ncu)
TAG=${1:-q}
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_tensorcore.py tests/test_gpu_parity_mixed.py -q -p no:cacheprovider -x > gpurun_out/pytest_$TAG.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_$TAG.log
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; echo "bench rc=$?"
python - <<PY
import json
try:
    d=json.loads(open("gpurun_out/bench_$TAG.json").read().strip().splitlines()[-1])
    print("value %.3e ms/step %.4f" % (d["value"], d["ms_per_step"]), {k: round(v,4) for k,v in d["stage_ms_per_step"].items()}, "e2e %.3e" % d["e2e"]["value"], d["clocks"])
except Exception as e:
    print("bench parse failed", e); print(open("gpurun_out/bench_$TAG.err").read()[-2000:])
PY
