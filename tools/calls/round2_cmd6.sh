python -m pytest tests -m gpu -x -q -k "flop or fused or config" > gpurun_out/t6.log 2>&1; echo rc=$? >> gpurun_out/t6.log
B="python bench.py --no-e2e --no-cpu-baseline --no-accuracy"
$B --config 3 > gpurun_out/c6_3rows.log 2>&1
SPNNZ_FLOP_ROWS=0 $B --config 3 > gpurun_out/c6_3seg.log 2>&1
$B --config 4 > gpurun_out/c6_4smem.log 2>&1
SPNNZ_FLOP_SMEM=0 $B --config 4 > gpurun_out/c6_4nosmem.log 2>&1
$B --config 1 > gpurun_out/c6_1.log 2>&1
ncu --set full --clock-control none --import-source on -k "regex:k_flop" -c 1 -o gpurun_out/prof6_cfg3rows -f python bench.py --config 3 --profile-steps 1 > gpurun_out/prof6_cfg3rows.log 2>&1
ncu --set full --clock-control none --import-source on -k "regex:k_flop_smem" -c 1 -o gpurun_out/prof6_cfg4smem -f python bench.py --config 4 --profile-steps 1 > gpurun_out/prof6_cfg4smem.log 2>&1
