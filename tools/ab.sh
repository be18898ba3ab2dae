#!/bin/bash
# A/B: quick bench of config $1 for the in-tree build and each variant name
# given: tools/ab.sh 5 g1 g2 ...  -> gpurun_out/ab_<cfg>_<name>.log
cfg=$1; shift
mkdir -p gpurun_out
python bench.py --config $cfg --no-e2e --no-cpu-baseline --no-accuracy > gpurun_out/ab_${cfg}_base.log 2>&1
for v in "$@"; do
  SPNNZ_GPU_LIB=build/var_$v/libspnnz_gpu.so python bench.py --config $cfg --no-e2e --no-cpu-baseline --no-accuracy > gpurun_out/ab_${cfg}_$v.log 2>&1
done
