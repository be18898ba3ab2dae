# ncu --set full of the config-4 row-block FLOP kernel, config-2 heavy run, config-3 predict
mkdir -p gpurun_out
for c in 4 2 3; do python bench.py --config $c --profile-steps 1 > gpurun_out/plain$c.log 2>&1 || { echo "plain $c failed"; exit 1; }; done
ncu --set full --clock-control none --import-source on -k "regex:k_flop_rb" -c 1 -o gpurun_out/p_rb4 -f python bench.py --config 4 --profile-steps 1 > gpurun_out/p_rb4.log 2>&1
ncu --set full --clock-control none --import-source on -k "regex:k_heavy_run|k_sym_block_hash" -c 4 -o gpurun_out/p_hv2 -f python bench.py --config 2 --profile-steps 1 > gpurun_out/p_hv2.log 2>&1
ncu --set full --clock-control none --import-source on -k "regex:k_predict|k_flop_rb" -c 2 -o gpurun_out/p_pr3 -f python bench.py --config 3 --profile-steps 1 > gpurun_out/p_pr3.log 2>&1
ls -la gpurun_out
