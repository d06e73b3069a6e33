#!/bin/bash
# ncu --set full of the top kernel after a clean plain run of the same command
TAG=${1:-n}
KRE=${2:-k_fused_mixed}
mkdir -p gpurun_out
CMD="python bench.py --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 1"
$CMD > gpurun_out/plain_$TAG.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"$KRE" -s 2 -c 1 -o gpurun_out/prof_$TAG -f $CMD > gpurun_out/ncu_full_$TAG.log 2>&1; echo "ncu full rc=$?"
tail -3 gpurun_out/ncu_full_$TAG.log
