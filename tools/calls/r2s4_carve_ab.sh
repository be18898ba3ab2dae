mkdir -p gpurun_out/cv
for v in none 100 75 50 35 25; do
  for c in 2 5; do
    if [ $v = none ]; then python bench.py --config $c --no-e2e --no-cpu-baseline --no-accuracy > gpurun_out/cv/b_${v}_c$c.log 2>&1
    else SPNNZ_FLOP_CARVEOUT=$v python bench.py --config $c --no-e2e --no-cpu-baseline --no-accuracy > gpurun_out/cv/b_${v}_c$c.log 2>&1; fi
  done
done
