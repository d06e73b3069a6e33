#!/bin/bash
# end-of-round evidence in one gpurun call: GPU suite, smoke, default bench,
# the bench's kernel launch list under ncu, one --set full capture of the fused kernel
TAG=${1:-r2f}
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/${TAG}_gputest.log 2>&1; echo "gpu tests rc=$?"; tail -1 gpurun_out/${TAG}_gputest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/${TAG}_smoke.log 2>&1; echo "smoke rc=$?"
timeout 600 python bench.py > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err; echo "bench rc=$?"
CMD="python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-inference --e2e-steps 1"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"^k_" -c 400 --csv \
  --log-file gpurun_out/${TAG}_launches.csv $CMD > gpurun_out/${TAG}_ncu_list.log 2>&1; echo "ncu list rc=$?"
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_fused_mixed -s 2 -c 1 \
  -o gpurun_out/prof_${TAG} -f $CMD > gpurun_out/${TAG}_ncu_full.log 2>&1; echo "ncu full rc=$?"
