mkdir -p gpurun_out/st
for r in 1 2; do
python bench.py --config 5 --no-e2e --no-cpu-baseline --no-accuracy > gpurun_out/st/b_base_r$r.log 2>&1
for v in sg2 sg4; do
SPNNZ_GPU_LIB=build/var_$v/libspnnz_gpu.so python bench.py --config 5 --no-e2e --no-cpu-baseline --no-accuracy > gpurun_out/st/b_${v}_r$r.log 2>&1
done; done
