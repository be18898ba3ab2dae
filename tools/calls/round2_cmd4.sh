python -m pytest tests -m gpu -x -q -k "flop" > gpurun_out/t4.log 2>&1; echo rc=$? >> gpurun_out/t4.log
B="python bench.py --no-e2e --no-cpu-baseline --no-accuracy"
$B --config 3 > gpurun_out/c4_3rows.log 2>&1
SPNNZ_FLOP_ROWS=0 $B --config 3 > gpurun_out/c4_3seg.log 2>&1
$B --config 4 > gpurun_out/c4_4smem.log 2>&1
SPNNZ_FLOP_SMEM=0 $B --config 4 > gpurun_out/c4_4nosmem.log 2>&1
$B --config 5 > gpurun_out/c4_5p0.log 2>&1
SPNNZ_FLOP_PREFETCH=1480 $B --config 5 > gpurun_out/c4_5p1480.log 2>&1
SPNNZ_FLOP_PREFETCH=3000 $B --config 5 > gpurun_out/c4_5p3000.log 2>&1
$B --config 2 > gpurun_out/c4_2p0.log 2>&1
SPNNZ_FLOP_PREFETCH=1480 $B --config 2 > gpurun_out/c4_2p1480.log 2>&1
