mkdir -p gpurun_out/uz
for r in 1 2 3; do
python bench.py --config 5 --no-e2e --no-cpu-baseline --no-accuracy > gpurun_out/uz/b_base_r$r.log 2>&1
SPNNZ_GPU_LIB=build/var_uswz/libspnnz_gpu.so python bench.py --config 5 --no-e2e --no-cpu-baseline --no-accuracy > gpurun_out/uz/b_uswz_r$r.log 2>&1
done
SPNNZ_GPU_LIB=build/var_uswz/libspnnz_gpu.so timeout 900 python -m pytest tests -m gpu -x -q -k "heavy or bin or fuzz or config" > gpurun_out/uz/gputest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/uz/gputest.log
