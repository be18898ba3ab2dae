python -m pytest tests -m gpu -x -q -k "flop or config_vs" > gpurun_out/t24.log 2>&1; echo rc=$? >> gpurun_out/t24.log
B="python bench.py --no-e2e --no-cpu-baseline --no-accuracy"
for c in 5 2; do $B --config $c > gpurun_out/c24_$c.log 2>&1; done
SPNNZ_FLOP_NOL1=0 $B --config 5 > gpurun_out/c24_5l1.log 2>&1
$B --config 5 > gpurun_out/c24_5b.log 2>&1
