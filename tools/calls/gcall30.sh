mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/t30.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/t30.log
python tools/latency_probe.py
SPNNZ_SYM_SMALL=0 python tools/latency_probe.py
bash tools/qb.sh "1 4"; python tools/qb_show.py 1 4
timeout 300 build/spnnz_corpus --overhead 2>&1 | tail -5
