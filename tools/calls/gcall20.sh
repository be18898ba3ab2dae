mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/t20.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/t20.log
bash tools/qb.sh "5 2 3 4 1"; python tools/qb_show.py 5 2 3 4 1
