#!/bin/bash
# Build a variant of the product library with extra -D flags into
# paper_1902_04995_b200/lib/variants/<name>.so (A/B timing via LP2D_B200_LIB).
set -e
cd "$(dirname "$0")/../paper_1902_04995_b200/csrc"
name=$1; shift
mkdir -p ../lib/variants ../build/variants
NV=/usr/local/cuda/bin/nvcc
$NV -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo --fmad=false -std=c++17 -Xcompiler -fPIC \
  -Xptxas -v "$@" -c -o ../build/variants/$name.o lp2d_capi.cu 2> ../build/variants/$name.ptxas.log
$NV -gencode arch=compute_100a,code=sm_100a -shared -o ../lib/variants/$name.so ../build/variants/$name.o ../build/lp2d_generate.o -lpthread
grep -A2 "k_solve_fxItLi$LP2D_NS" ../build/variants/$name.ptxas.log | grep -E "spill|Used" | head -4 || true
