B="python bench.py --no-e2e --no-cpu-baseline --no-accuracy"
$B --config 3 > gpurun_out/c27_3.log 2>&1
SPNNZ_RB_PERSIST=0 $B --config 3 > gpurun_out/c27_3np.log 2>&1
$B --config 3 > gpurun_out/c27_3b.log 2>&1
python -m pytest tests -m gpu -x -q -k "flop_row_mode or flop_degree" > gpurun_out/t27.log 2>&1; echo rc=$? >> gpurun_out/t27.log
