mkdir -p gpurun_out/ru
for r in 1 2; do
python bench.py --config 2 --no-e2e --no-cpu-baseline --no-accuracy > gpurun_out/ru/b_base_r$r.log 2>&1
for v in ru4 ru16; do
SPNNZ_GPU_LIB=build/var_$v/libspnnz_gpu.so python bench.py --config 2 --no-e2e --no-cpu-baseline --no-accuracy > gpurun_out/ru/b_${v}_r$r.log 2>&1
done; done
