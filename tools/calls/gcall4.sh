mkdir -p gpurun_out
python bench.py --config 4 --profile-steps 1 > gpurun_out/plain4.log 2>&1 || exit 1
ncu --set full --clock-control none --import-source on -k "regex:k_flop_rs|k_degree" -c 2 -o gpurun_out/p_rs4 -f python bench.py --config 4 --profile-steps 1 > gpurun_out/p_rs4.log 2>&1
