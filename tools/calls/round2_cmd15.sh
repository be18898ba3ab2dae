python -m pytest tests -m gpu -x -q -k "flop" > gpurun_out/t15.log 2>&1; echo rc=$? >> gpurun_out/t15.log
B="python bench.py --no-e2e --no-cpu-baseline --no-accuracy"
$B --config 4 > gpurun_out/c15_4.log 2>&1
$B --config 3 > gpurun_out/c15_3.log 2>&1
SPNNZ_FLOP_RB=1 $B --config 3 > gpurun_out/c15_3rb.log 2>&1
$B --config 1 > gpurun_out/c15_1.log 2>&1
