#!/bin/bash
# ncu --set full of the fused kernel on the paper's workload (--network paper)
TAG=${1:-p}
mkdir -p gpurun_out
CMD="python bench.py --network paper --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 1"
$CMD > gpurun_out/plainp_$TAG.json 2>&1 && \
ncu --set full --clock-control none -k regex:k_fused_mixed -s 2 -c 1 -o gpurun_out/profp_$TAG -f $CMD > gpurun_out/ncup_$TAG.log 2>&1; echo "ncu rc=$?"
