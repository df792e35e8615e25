#!/bin/bash
# Builds timing-experiment variants of libspl.so (results are WRONG by design):
#   K3_EXP=1 no histogram updates, 2 = also no popcount.
# Use: SPL_LIB=build/exp/libspl_exp1.so SPL_K3_TRACE=1 python bench.py ...
set -e
cd "$(dirname "$0")/.."
mkdir -p build/exp
for e in 1 2; do
  d=build/exp/obj$e; mkdir -p $d
  F="-gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC --expt-relaxed-constexpr -Iinclude"
  objs=""
  for f in capi hamming_topk encode_exact encode_tc sparse_attend bitcodes_misc; do
    x=""; [ $f = encode_exact ] && x="-fmad=false -prec-div=true -prec-sqrt=true -ftz=false"
    [ $f = hamming_topk ] && x="-DK3_EXP=$e"
    nvcc $F $x -c paper_2508_19740_b200/csrc/$f.cu -o $d/$f.o &
    objs="$objs $d/$f.o"
  done
  wait
  nvcc -gencode arch=compute_100a,code=sm_100a -shared -o build/exp/libspl_exp$e.so $objs -Xlinker --version-script=paper_2508_19740_b200/csrc/exports.map
done
