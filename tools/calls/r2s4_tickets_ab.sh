# bins 3-5 rows by ticket (default) vs static striding (var_notick): configs 5, 2, 3 alternating, then parity
mkdir -p gpurun_out/t1
for r in 1 2 3; do
for c in 5 2; do
  python bench.py --config $c --no-e2e --no-cpu-baseline --no-accuracy > gpurun_out/t1/b_tick_c${c}_r$r.log 2>&1
  SPNNZ_GPU_LIB=build/var_notick/libspnnz_gpu.so python bench.py --config $c --no-e2e --no-cpu-baseline --no-accuracy > gpurun_out/t1/b_notick_c${c}_r$r.log 2>&1
done; done
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/t1/launches_tick5.csv python bench.py --config 5 --profile-steps 1 > /dev/null 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/t1/gputest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/t1/gputest.log
