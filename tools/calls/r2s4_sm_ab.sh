mkdir -p gpurun_out/sm
for r in 1 2; do
python bench.py --config 5 --no-e2e --no-cpu-baseline --no-accuracy > gpurun_out/sm/b_base_r$r.log 2>&1
SPNNZ_GPU_LIB=build/var_sm0/libspnnz_gpu.so python bench.py --config 5 --no-e2e --no-cpu-baseline --no-accuracy > gpurun_out/sm/b_sm0_r$r.log 2>&1
done
