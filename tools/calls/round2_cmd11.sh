B="python bench.py --no-e2e --no-cpu-baseline --no-accuracy"
for c in 1 4 3; do $B --config $c > gpurun_out/c11_$c.log 2>&1; SPNNZ_GRAPH=0 $B --config $c > gpurun_out/c11_${c}nog.log 2>&1; done
$B --config 2 > gpurun_out/c11_2.log 2>&1
SPNNZ_GRAPH=0 $B --config 2 > gpurun_out/c11_2nog.log 2>&1
compute-sanitizer --tool memcheck --leak-check full --error-exitcode 9 python tools/sanitize_cases.py > gpurun_out/san_memcheck.log 2>&1; echo rc=$? >> gpurun_out/san_memcheck.log
