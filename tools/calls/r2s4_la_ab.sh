# shared-window addresses held in registers (sort rank loop, bins 3-5 inserts): in-tree vs HEAD~ (var_head)
mkdir -p gpurun_out/la
for r in 1 2 3; do
for c in 5 2; do
  python bench.py --config $c --no-e2e --no-cpu-baseline --no-accuracy > gpurun_out/la/b_new_c${c}_r$r.log 2>&1
  SPNNZ_GPU_LIB=build/var_head/libspnnz_gpu.so python bench.py --config $c --no-e2e --no-cpu-baseline --no-accuracy > gpurun_out/la/b_head_c${c}_r$r.log 2>&1
done; done
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/la/launches_new5.csv python bench.py --config 5 --profile-steps 1 > /dev/null 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/la/gputest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/la/gputest.log
