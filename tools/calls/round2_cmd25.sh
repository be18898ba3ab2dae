bash tools/ab.sh 3 rb1400 rb900
python -m pytest tests -m gpu -x -q -k "flop" > gpurun_out/t25.log 2>&1; echo rc=$? >> gpurun_out/t25.log
