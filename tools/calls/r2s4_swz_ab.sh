mkdir -p gpurun_out/sz
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/sz/gputest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/sz/gputest.log
for r in 1 2 3; do
python bench.py --config 2 --no-e2e --no-cpu-baseline --no-accuracy > gpurun_out/sz/b_swz_r$r.log 2>&1
SPNNZ_BITMAP_SWZ=0 python bench.py --config 2 --no-e2e --no-cpu-baseline --no-accuracy > gpurun_out/sz/b_plain_r$r.log 2>&1
done
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/sz/launches_swz2.csv python bench.py --config 2 --profile-steps 1 > /dev/null 2>&1
