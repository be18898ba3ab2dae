mkdir -p gpurun_out/uu
for r in 1 2; do
for c in 5 2; do
python bench.py --config $c --no-e2e --no-cpu-baseline --no-accuracy > gpurun_out/uu/b_base_c${c}_r$r.log 2>&1
for v in u8 su8 su2; do
  SPNNZ_GPU_LIB=build/var_$v/libspnnz_gpu.so python bench.py --config $c --no-e2e --no-cpu-baseline --no-accuracy > gpurun_out/uu/b_${v}_c${c}_r$r.log 2>&1
done; done; done
