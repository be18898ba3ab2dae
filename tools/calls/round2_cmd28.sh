ncu --set full --clock-control none --import-source on -k "regex:k_flop_rb" -c 1 -o gpurun_out/prof28_cfg4 -f python bench.py --config 4 --profile-steps 1 > gpurun_out/prof28_4.log 2>&1
ncu --set full --clock-control none --import-source on -k "regex:k_flop_rb" -c 1 -o gpurun_out/prof28_cfg3 -f python bench.py --config 3 --profile-steps 1 > gpurun_out/prof28_3.log 2>&1
