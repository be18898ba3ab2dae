mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -k "flop or small or repeat or corpus" > gpurun_out/t31.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/t31.log
python tools/latency_probe.py
timeout 300 build/spnnz_corpus --overhead 2>&1 | tail -5
timeout 300 build/spnnz_corpus 2>&1 | tail -3
