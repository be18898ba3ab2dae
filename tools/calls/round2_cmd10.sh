B="python bench.py --no-e2e --no-cpu-baseline --no-accuracy"
for c in 1 4 3 2 5; do $B --config $c > gpurun_out/c10_$c.log 2>&1; done
SPNNZ_GRAPH=0 $B --config 1 > gpurun_out/c10_1nog.log 2>&1
SPNNZ_GRAPH=0 $B --config 4 > gpurun_out/c10_4nog.log 2>&1
python -m pytest tests -m gpu -x -q -k "repeat or flop_known or config_vs" > gpurun_out/t10.log 2>&1; echo rc=$? >> gpurun_out/t10.log
