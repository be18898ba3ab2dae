mkdir -p gpurun_out
python bench.py --config 2 --profile-steps 1 > gpurun_out/plain2.log 2>&1 && ncu --set full --clock-control none --import-source on -k "regex:k_heavy_run" -c 1 -o gpurun_out/p_hr2 -f python bench.py --config 2 --profile-steps 1 > gpurun_out/p_hr2.log 2>&1
