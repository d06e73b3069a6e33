#!/bin/bash
# quick GPU iteration: all GPU tests + bench (no ncu); every step under its own timeout
TAG=${1:-q}
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -x > gpurun_out/pytest_$TAG.log 2>&1; echo "pytest rc=$?"; tail -5 gpurun_out/pytest_$TAG.log
timeout 300 python bench.py --no-cpu-baseline > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; echo "bench rc=$?"
python - <<PY
import json
try:
    d=json.loads(open("gpurun_out/bench_$TAG.json").read().strip().splitlines()[-1])
    print("value %.3e ms/step %.4f" % (d["value"], d["ms_per_step"]), {k: round(v,4) for k,v in d["stage_ms_per_step"].items()}, "e2e %.3e" % d["e2e"]["value"], d["roofline"]["frac"], d["clocks"])
except Exception as e:
    print("bench parse failed", e); print(open("gpurun_out/bench_$TAG.err").read()[-3000:])
PY
