#!/bin/bash
# quick GPU check + phase timing of the fused kernel (rebuilds k_fused_mixed with -DROMAP_FUSED_PROF on the box)
TAG=${1:-p}
bash tools/gpu_quick.sh $TAG
cd paper_2304_05735_b200/csrc && touch k_fused_mixed.cu && make EXTRA=-DROMAP_FUSED_PROF > /dev/null 2>&1 && cd ../.. && \
  timeout 300 python tools/fused_prof.py
