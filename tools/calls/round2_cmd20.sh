B="python bench.py --no-e2e --no-cpu-baseline --no-accuracy"
for c in 1 4 3 2 5; do $B --config $c > gpurun_out/c20_$c.log 2>&1; SPNNZ_TIERS_BESIDE=1 $B --config $c > gpurun_out/c20_${c}tb.log 2>&1; done
ncu --set full --clock-control none --import-source on -k "regex:k_flop_rb" -c 1 -o gpurun_out/prof20_cfg4rb -f python bench.py --config 4 --profile-steps 1 > gpurun_out/prof20.log 2>&1
