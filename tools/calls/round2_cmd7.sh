python -m pytest tests -m gpu -x -q -k "flop or fused or config" > gpurun_out/t7.log 2>&1; echo rc=$? >> gpurun_out/t7.log
B="python bench.py --no-e2e --no-cpu-baseline --no-accuracy"
$B --config 3 > gpurun_out/c7_3rb.log 2>&1
SPNNZ_FLOP_RB=0 $B --config 3 > gpurun_out/c7_3rows.log 2>&1
$B --config 4 > gpurun_out/c7_4rb.log 2>&1
SPNNZ_FLOP_RB=0 $B --config 4 > gpurun_out/c7_4tiles.log 2>&1
$B --config 1 > gpurun_out/c7_1.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/l7_cfg3.csv python bench.py --config 3 --profile-steps 1 > /dev/null 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/l7_cfg4.csv python bench.py --config 4 --profile-steps 1 > /dev/null 2>&1
