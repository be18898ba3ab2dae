mkdir -p gpurun_out/un
for r in 1 2; do
python bench.py --config 5 --no-e2e --no-cpu-baseline --no-accuracy > gpurun_out/un/b_base_r$r.log 2>&1
for v in t5u8 t5u2 t3u8; do
  SPNNZ_GPU_LIB=build/var_$v/libspnnz_gpu.so python bench.py --config 5 --no-e2e --no-cpu-baseline --no-accuracy > gpurun_out/un/b_${v}_r$r.log 2>&1
done; done
SPNNZ_GPU_LIB=build/var_t5u8/libspnnz_gpu.so ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/un/launches_t5u8.csv python bench.py --config 5 --profile-steps 1 > /dev/null 2>&1
