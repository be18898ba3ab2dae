mkdir -p gpurun_out/sw
for r in 1 2; do
python bench.py --config 5 --no-e2e --no-cpu-baseline --no-accuracy > gpurun_out/sw/b_base_r$r.log 2>&1
for v in hb128 hb512 t4u16 t4u4 rg2 rg4; do
  SPNNZ_GPU_LIB=build/var_$v/libspnnz_gpu.so python bench.py --config 5 --no-e2e --no-cpu-baseline --no-accuracy > gpurun_out/sw/b_${v}_r$r.log 2>&1
done; done
