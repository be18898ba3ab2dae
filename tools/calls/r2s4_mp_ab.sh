# multipass hash tier (rows of 24576 < FLOP <= SPNNZ_MP_MAX) vs the heavy path: parity first, then A/B
mkdir -p gpurun_out/mp
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/mp/gputest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/mp/gputest.log
for r in 1 2; do
for m in 0 49152 98304 196608; do
for c in 5 2; do
  SPNNZ_MP_MAX=$m python bench.py --config $c --no-e2e --no-cpu-baseline --no-accuracy > gpurun_out/mp/b_m${m}_c${c}_r$r.log 2>&1
done; done; done
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/mp/launches_mp5.csv python bench.py --config 5 --profile-steps 1 > /dev/null 2>&1
