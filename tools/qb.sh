#!/bin/bash
# quick per-config bench (no e2e / cpu baseline / accuracy) into gpurun_out/
# usage: tools/qb.sh "5 2 3 4"
mkdir -p gpurun_out
for c in ${1:-5 2 3 4}; do
  python bench.py --config $c --no-e2e --no-cpu-baseline --no-accuracy > gpurun_out/bench_cfg$c.log 2>&1
done
