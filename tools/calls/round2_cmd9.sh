python -m pytest tests -m gpu -x -q > gpurun_out/t9.log 2>&1; echo rc=$? >> gpurun_out/t9.log
B="python bench.py --no-e2e --no-cpu-baseline --no-accuracy"
for c in 1 4 3 2 5; do $B --config $c > gpurun_out/c9_$c.log 2>&1; done
SPNNZ_FLOP_RB=0 $B --config 4 > gpurun_out/c9_4tiles.log 2>&1
SPNNZ_FLOP_RB=0 $B --config 3 > gpurun_out/c9_3rows.log 2>&1
SPNNZ_GRAPH=0 $B --config 1 > gpurun_out/c9_1nog.log 2>&1
