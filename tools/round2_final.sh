#!/bin/bash
# Round-2 final judged artefacts (one gpurun call) into gpurun_out/m2/: full
# bench lines per config (uncapped + cap 300), the reference arm per config,
# per-kernel launch lists, ncu --set full of the FLOP pass and of the
# symbolic / predict kernels per config, the shard projection and the corpus.
# Summaries: tools/profile_round.py --round r02 ....
# gpurun brings back at most 64 MiB: run it as two calls, PART=bench (default:
# everything but the full ncu captures) and PART=ncu (the eight captures).
O=gpurun_out/m2
mkdir -p $O
T="timeout 900"
PART=${PART:-bench}
if [ "$PART" = bench ]; then
for c in 5 1 2 3 4; do $T python bench.py --config $c > $O/bench_cfg$c.log 2>&1; done
for c in 5 1 2 3 4; do $T python bench.py --config $c --cap 300 --no-accuracy > $O/bench_cfg${c}_cap300.log 2>&1; done
for c in 5 1 2 3 4; do $T python bench.py --impl reference --config $c > $O/ref_cfg$c.log 2>&1; done
$T python bench.py --impl reference --config 5 --cap 300 > $O/ref_cfg5_cap300.log 2>&1
$T python tools/shard_projection.py --config 5 --ranks 1 2 4 8 > $O/proj5.json 2> $O/proj5.err
$T build/spnnz_corpus --csv $O/corpus.csv --json $O/corpus.json > $O/corpus.txt 2>&1
$T build/spnnz_corpus --overhead > $O/overhead.txt 2>&1
$T python tools/latency_probe.py > $O/latency.txt 2>&1
for c in 5 1 2 3 4; do
  $T ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_cfg$c.csv \
      python bench.py --config $c --profile-steps 1 > /dev/null 2>&1
done
fi
if [ "$PART" = ncu ]; then
for c in 5 2 3 4; do
  $T ncu --set full --clock-control none --import-source on -k "regex:k_degree|k_tile_rows|k_flop" \
      -o $O/flop_cfg$c -f python bench.py --config $c --profile-steps 1 > $O/flop_cfg$c.log 2>&1
  $T ncu --set full --clock-control none --import-source on -k "regex:k_predict|k_sym_block_hash|k_heavy_run|k_heavy_sort" \
      -o $O/symp_cfg$c -f python bench.py --config $c --profile-steps 1 > $O/symp_cfg$c.log 2>&1
done
fi
ls -la $O
