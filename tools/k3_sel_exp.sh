#!/bin/bash
# Timing-experiment variants of libspl.so for the fused select (results are
# WRONG by design): K3_SEL_EXP=1 no index stores, 2 = stop after the counts.
# Use: SPL_LIB=build/exp/libspl_sel1.so SPL_K3_TRACE=1 python bench.py ...
set -e
cd "$(dirname "$0")/.."
F="-gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC --expt-relaxed-constexpr -Iinclude"
for e in 1 2; do
  d=build/exp/sel$e; mkdir -p $d
  cp build/obj/*.o $d/
  nvcc $F -DK3_SEL_EXP=$e -c paper_2508_19740_b200/csrc/hamming_topk.cu -o $d/hamming_topk.o
  nvcc -gencode arch=compute_100a,code=sm_100a -shared -o build/exp/libspl_sel$e.so $d/*.o -Xlinker --version-script=paper_2508_19740_b200/csrc/exports.map
done
