python -m pytest tests -m gpu -x -q -k "flop or guard" > gpurun_out/t26.log 2>&1; echo rc=$? >> gpurun_out/t26.log
B="python bench.py --no-e2e --no-cpu-baseline --no-accuracy"
for c in 3 4 1; do $B --config $c > gpurun_out/c26_$c.log 2>&1; done
