mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/t28.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/t28.log
bash tools/qb.sh "3 5"; python tools/qb_show.py 3 5
