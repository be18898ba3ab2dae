python -m pytest tests -m gpu -x -q -k "flop or config_vs or fuzz" > gpurun_out/t23.log 2>&1; echo rc=$? >> gpurun_out/t23.log
B="python bench.py --no-e2e --no-cpu-baseline --no-accuracy"
for c in 5 2 3; do $B --config $c > gpurun_out/c23_$c.log 2>&1; done
SPNNZ_FLOP_NOL1=0 $B --config 5 > gpurun_out/c23_5l1.log 2>&1
$B --config 5 > gpurun_out/c23_5b.log 2>&1
