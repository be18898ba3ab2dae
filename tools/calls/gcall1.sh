set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/gputest.log 2>&1; echo "gputest rc=$?"
tail -3 gpurun_out/gputest.log
bash tools/qb.sh "5 1 2 3 4"
for c in 5 1 2 3 4; do tail -1 gpurun_out/bench_cfg$c.log | cut -c1-600; done
