#!/bin/bash
# ncu --set full of the kernels matching a regex, one predictor pass
# usage: tools/qfull.sh <config> <kernel-regex> <out-name> [count]
mkdir -p gpurun_out
ncu --set full --clock-control none --import-source on -k "regex:$2" -c ${4:-3} \
    -o gpurun_out/$3 -f python bench.py --config $1 --profile-steps 1 > gpurun_out/$3.log 2>&1
