mkdir -p gpurun_out
python bench.py --config 5 --profile-steps 1 > gpurun_out/plain5.log 2>&1 && ncu --set full --clock-control none --import-source on -k "regex:k_heavy_sort_units|k_sym_block_hash<1024" -c 2 -o gpurun_out/p_sort5 -f python bench.py --config 5 --profile-steps 1 > gpurun_out/p_sort5.log 2>&1
