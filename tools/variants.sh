#!/bin/bash
# Builds variants of libspnnz_gpu.so with extra nvcc defines, for A/B timing:
#   tools/variants.sh NAME "-DFOO=1" [NAME2 "-DBAR=2" ...]
# -> build/var_NAME/libspnnz_gpu.so ; run with SPNNZ_GPU_LIB=build/var_NAME/libspnnz_gpu.so
set -e
cd "$(dirname "$0")/.."
NVCC=${NVCC:-/usr/local/cuda/bin/nvcc}
FLAGS="-gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -fmad=false -Xcompiler -fPIC,-ffp-contract=off -Iinclude -Ipaper_2207_13848_b200/csrc"
while [ $# -ge 2 ]; do
  name=$1; defs=$2; shift 2
  out=build/var_$name; mkdir -p $out
  objs=""
  for f in flop sample_predict symbolic heavy; do
    $NVCC $FLAGS $defs -c -o $out/$f.o paper_2207_13848_b200/csrc/$f.cu &
    objs="$objs $out/$f.o"
  done
  $NVCC $FLAGS $defs -c -o $out/capi.o paper_2207_13848_b200/csrc/capi.cpp &
  wait
  $NVCC -gencode arch=compute_100a,code=sm_100a -shared -o $out/libspnnz_gpu.so $objs $out/capi.o -ldl
  echo "built $out/libspnnz_gpu.so"
done
