mkdir -p gpurun_out
SPNNZ_GPU_LIB=build/var_h128/libspnnz_gpu.so timeout 600 python -m pytest tests -m gpu -x -q -k "heavy or every_bin or config_vs" > gpurun_out/t40.log 2>&1; echo "h128 tests rc=$?"; tail -1 gpurun_out/t40.log
for v in 0 1 2; do
  SPNNZ_GPU_LIB=build/var_h128/libspnnz_gpu.so SPNNZ_HEAVY_BESIDE=$v python tools/timeline.py 5 3 2>&1 | grep -E "timeline|heavy " | tail -7
  SPNNZ_GPU_LIB=build/var_h128/libspnnz_gpu.so SPNNZ_HEAVY_BESIDE=$v python bench.py --config 5 --no-e2e --no-cpu-baseline --no-accuracy 2>&1 | tail -1 | cut -c1-140
done
python bench.py --config 5 --no-e2e --no-cpu-baseline --no-accuracy 2>&1 | tail -1 | cut -c1-140
