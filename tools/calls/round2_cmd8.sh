python -m pytest tests -m gpu -x -q -k "flop or fused or config1 or pipeline or with_plan" > gpurun_out/t8.log 2>&1; echo rc=$? >> gpurun_out/t8.log
B="python bench.py --no-e2e --no-cpu-baseline --no-accuracy"
$B --config 4 > gpurun_out/c8_4rb.log 2>&1
SPNNZ_FLOP_RB=0 $B --config 4 > gpurun_out/c8_4tiles.log 2>&1
$B --config 3 > gpurun_out/c8_3rb.log 2>&1
SPNNZ_FLOP_RB=0 $B --config 3 > gpurun_out/c8_3rows.log 2>&1
$B --config 1 > gpurun_out/c8_1.log 2>&1
$B --config 2 > gpurun_out/c8_2.log 2>&1
$B --config 5 > gpurun_out/c8_5.log 2>&1
ncu --set full --clock-control none --import-source on -k "regex:k_flop_rb" -c 1 -o gpurun_out/prof8_cfg4rb -f python bench.py --config 4 --profile-steps 1 > gpurun_out/prof8_cfg4rb.log 2>&1
ncu --set full --clock-control none --import-source on -k "regex:k_flop_rb" -c 1 -o gpurun_out/prof8_cfg3rb -f python bench.py --config 3 --profile-steps 1 > gpurun_out/prof8_cfg3rb.log 2>&1
