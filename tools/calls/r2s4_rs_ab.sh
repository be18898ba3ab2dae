# config-4 row streams: shared-table pattern probe + chunks-in-flight A/B
mkdir -p gpurun_out
for r in 1 2; do
bash tools/ab.sh 4 a3 a1
for v in base a3 a1; do cp gpurun_out/ab_4_$v.log gpurun_out/ab_4_${v}_r$r.log; done
done
python bench.py --config 1 --no-e2e --no-cpu-baseline --no-accuracy > gpurun_out/ab_1_base.log 2>&1
timeout 600 python -m pytest tests -m gpu -x -q -k "flop or rs or smem" > gpurun_out/gputest_flop.log 2>&1; echo "rc=$?" >> gpurun_out/gputest_flop.log
