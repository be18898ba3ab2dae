mkdir -p gpurun_out/f2
run() { # name, env...
  n=$1; shift
  for c in 2 5; do env "$@" python bench.py --config $c --no-e2e --no-cpu-baseline --no-accuracy > gpurun_out/f2/b_${n}_c$c.log 2>&1; done
}
run base A=1
run nol1 SPNNZ_FLOP_NOL1=1
run l1 SPNNZ_FLOP_NOL1=0
run pf SPNNZ_FLOP_PREFETCH=1184
run mb1536 SPNNZ_GPU_LIB=build/var_mb1536/libspnnz_gpu.so
run mb2048 SPNNZ_GPU_LIB=build/var_mb2048/libspnnz_gpu.so
run base2 A=1
