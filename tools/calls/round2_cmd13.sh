python tools/sanitize_cases.py > gpurun_out/san_plain.log 2>&1; echo rc=$? >> gpurun_out/san_plain.log
SPNNZ_GUARD=1 python tools/sanitize_cases.py > gpurun_out/san_guard.log 2>&1; echo rc=$? >> gpurun_out/san_guard.log
B="python bench.py --no-e2e --no-cpu-baseline --no-accuracy"
$B --config 2 > gpurun_out/c13_2.log 2>&1
python -m pytest tests -m gpu -x -q -k "every_bin or heavy or fuzz or config_vs" > gpurun_out/t13.log 2>&1; echo rc=$? >> gpurun_out/t13.log
