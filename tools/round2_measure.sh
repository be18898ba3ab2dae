#!/bin/bash
# Round-2 judged artefacts (one gpurun call): full bench lines per config
# (uncapped + cap 300), the reference arm per config, per-kernel launch lists
# and ncu --set full captures of the FLOP pass and the symbolic / predict
# kernels.  Summaries: tools/profile_round.py --round r02 ...
set -x
O=gpurun_out/m
mkdir -p $O
for c in 5 1 2 3 4; do python bench.py --config $c > $O/bench_cfg$c.log 2>&1; done
for c in 5 1 2 3 4; do python bench.py --config $c --cap 300 --no-accuracy > $O/bench_cfg${c}_cap300.log 2>&1; done
for c in 5 1 2 3 4; do python bench.py --impl reference --config $c > $O/ref_cfg$c.log 2>&1; done
python bench.py --impl reference --config 5 --cap 300 > $O/ref_cfg5_cap300.log 2>&1
for c in 5 1 2 3 4; do
  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_cfg$c.csv \
      python bench.py --config $c --profile-steps 1 > /dev/null 2>&1
done
for c in 5 2 3 4; do
  ncu --set full --clock-control none --import-source on -k "regex:k_degree|k_tile_rows|k_flop" \
      -o $O/flop_cfg$c -f python bench.py --config $c --profile-steps 1 > $O/flop_cfg$c.log 2>&1
  ncu --set full --clock-control none --import-source on -k "regex:k_predict|k_sym_block_hash|k_heavy_run|k_heavy_sort" \
      -o $O/symp_cfg$c -f python bench.py --config $c --profile-steps 1 > $O/symp_cfg$c.log 2>&1
done
