mkdir -p gpurun_out/v2
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/v2/gputest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/v2/gputest.log
for c in 5 2 4; do python bench.py --config $c --no-e2e --no-cpu-baseline --no-accuracy > gpurun_out/v2/b_c${c}.log 2>&1; done
