#!/bin/bash
# per-kernel launch list (ncu, one metric) of one predictor pass for the
# in-tree build ("base") and each variant: tools/qlaunch.sh <cfg> base v1 v2
# -> gpurun_out/launches_cfg<cfg>_<v>.csv
mkdir -p gpurun_out
cfg=$1; shift
for v in "$@"; do
  lib=""; [ "$v" != base ] && lib=build/var_$v/libspnnz_gpu.so
  SPNNZ_GPU_LIB=$lib ncu --metrics gpu__time_duration.sum --clock-control none --csv \
      --log-file gpurun_out/launches_cfg${cfg}_$v.csv \
      python bench.py --config $cfg --profile-steps 1 > gpurun_out/ncu_cfg${cfg}_$v.log 2>&1
done
