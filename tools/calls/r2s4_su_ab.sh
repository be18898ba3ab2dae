mkdir -p gpurun_out/su
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/su/gputest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/su/gputest.log
for r in 1 2 3; do
python bench.py --config 5 --no-e2e --no-cpu-baseline --no-accuracy > gpurun_out/su/b_su8_r$r.log 2>&1
SPNNZ_GPU_LIB=build/var_su16/libspnnz_gpu.so python bench.py --config 5 --no-e2e --no-cpu-baseline --no-accuracy > gpurun_out/su/b_su16_r$r.log 2>&1
done
