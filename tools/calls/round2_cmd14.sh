bash tools/ab.sh 5 b4w b5u8 t4u4
bash tools/ab.sh 2 b4w b5u8
B="python bench.py --no-e2e --no-cpu-baseline --no-accuracy"
for c in 1 2 3 4; do SPNNZ_FUSED_PREDICT=1 $B --config $c > gpurun_out/c14_${c}fused.log 2>&1; $B --config $c > gpurun_out/c14_${c}.log 2>&1; done
