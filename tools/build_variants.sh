#!/bin/bash
# Build libmpgpu variants with different compile-time knobs for A/B timing on the box.
# usage: [ONLY="gemm lu"] tools/build_variants.sh NAME "-DKNOB=VAL ..." [NAME2 "FLAGS2" ...]
set -e
cd "$(dirname "$0")/.."
OUT=paper_1410_1599_b200/_variants
mkdir -p $OUT
NVCC="/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 --expt-relaxed-constexpr -Xcompiler -fPIC -Iinclude"
while [ $# -gt 0 ]; do
  name=$1; flags=$2; shift 2
  d=$OUT/$name; mkdir -p $d
  ALL="gemm gemm_tc metrics elementwise elementwise_fused8 elementwise_fused16 elementwise_fused32 lu capi group gemm_wide metrics_wide elementwise_wide64 elementwise_wide128 elementwise_wide256 elementwise_wide288 lu_wide64 lu_wide128 lu_wide256 lu_wide288"
  for s in $ALL; do
    if [ -n "$ONLY" ] && ! [[ " $ONLY " == *" $s "* ]]; then
      cp paper_1410_1599_b200/_build/$s.cu.o $d/$s.o  # ONLY="gemm ...": reuse the main build's other objects
    else
      $NVCC $flags -c paper_1410_1599_b200/csrc/$s.cu -o $d/$s.o &
    fi
  done
  wait
  $NVCC -shared -o $d/libmpgpu.so $d/*.o -cudart static
  rm -f $d/*.o  # only the .so travels to the GPU box
  echo built $d/libmpgpu.so
done
