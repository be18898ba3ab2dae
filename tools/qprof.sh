#!/bin/bash
# per-kernel launch list of one predictor pass per config (ncu, one metric)
# usage: tools/qprof.sh "5 2"   -> gpurun_out/launches_cfg<c>.csv
mkdir -p gpurun_out
for c in ${1:-5}; do
  ncu --metrics gpu__time_duration.sum --clock-control none --csv \
      --log-file gpurun_out/launches_cfg$c.csv \
      python bench.py --config $c --profile-steps 1 > gpurun_out/ncu_cfg$c.log 2>&1
done
