#!/bin/bash
# The bounds-checked build (device asserts, -DSPNNZ_DEBUG_BOUNDS=1) with
# guard bands on every library buffer, over the GPU parity tests and the
# sanitizer case list -- the memory-safety pass while compute-sanitizer is
# closed on the GPU pool.  Build first: tools/variants.sh bounds "-DSPNNZ_DEBUG_BOUNDS=1"
mkdir -p gpurun_out
export SPNNZ_GPU_LIB=build/var_bounds/libspnnz_gpu.so SPNNZ_GUARD=1
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/bounds_tests.log 2>&1; echo "parity tests under bounds checks + guard bands: rc=$?"; tail -2 gpurun_out/bounds_tests.log
timeout 900 python tools/sanitize_cases.py > gpurun_out/bounds_cases.log 2>&1; echo "sanitizer cases: rc=$?"; tail -4 gpurun_out/bounds_cases.log
timeout 300 python tools/bounds_negative.py > gpurun_out/bounds_negative.log 2>&1; echo "negative check: rc=$?"; tail -1 gpurun_out/bounds_negative.log
