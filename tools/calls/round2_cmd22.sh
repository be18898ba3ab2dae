bash tools/ab.sh 2 notest
bash tools/ab.sh 5 notest
python -m pytest tests -m gpu -x -q -k "every_bin or heavy or fuzz or config_vs" > gpurun_out/t22.log 2>&1; echo rc=$? >> gpurun_out/t22.log
