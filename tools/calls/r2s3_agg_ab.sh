# R == 1 heavy bitmap insert aggregation A/B: default (match+redux), agg0 (off), agg2 (shuffle runs)
mkdir -p gpurun_out/c16
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/c16/gputest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/c16/gputest.log
SPNNZ_GPU_LIB=build/var_agg2/libspnnz_gpu.so timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "bin or heavy or fuzz or config" > gpurun_out/c16/gputest_agg2.log 2>&1; echo "pytest rc=$?" >> gpurun_out/c16/gputest_agg2.log
for r in 1 2; do
for v in agg1 agg0 agg2; do
  lib=""; [ $v != agg1 ] && lib=build/var_$v/libspnnz_gpu.so
  for c in 2 5; do
    SPNNZ_GPU_LIB=$lib timeout 300 python bench.py --config $c --no-e2e --no-cpu-baseline --no-accuracy > gpurun_out/c16/b_${v}_c${c}_r$r.log 2>&1
  done
done; done
