#!/bin/bash
# build an experiment variant of the fused kernel: libromap_<name>.so with extra -D flags
# usage: bash tools/build_variant.sh <name> "<nvcc flags>" [k_fused_mixed source, default the tree's]
set -e
cd "$(dirname "$0")/../paper_2304_05735_b200/csrc"
NVCC=/usr/local/cuda/bin/nvcc
ARCH="-gencode arch=compute_100a,code=sm_100a"
$NVCC $ARCH $2 -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Xcompiler -fvisibility=hidden -Xptxas -v \
  --expt-relaxed-constexpr -I. -c ${3:-k_fused_mixed.cu} -o kfm_$1.o 2> kfm_$1.ptxas.log || (cat kfm_$1.ptxas.log; false)
$NVCC $ARCH -shared -o ../libromap_$1.so romap_api.o k_sample.o k_fp32.o k_adam.o kfm_$1.o k_infer_mixed.o k_mesh.o k_selftest.o \
  k_det.o k_scene.o k_fused_mixed_det.o -Xcompiler -fvisibility=hidden
grep -A2 "k_fused_mixedILi16" kfm_$1.ptxas.log | grep -E "registers|spill" | tr '\n' ' '; echo " <- $1"
