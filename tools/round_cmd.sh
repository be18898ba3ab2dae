# One gpurun call that refreshes the round's judged artefacts
set -x
python bench.py > gpurun_out/bench_full.log 2>&1
python bench.py --cap 300 --no-e2e --no-accuracy > gpurun_out/bench_cap300.log 2>&1
for c in 2 3 4; do python bench.py --config $c --no-e2e --no-cpu-baseline --no-accuracy > gpurun_out/bench_cfg$c.log 2>&1; done
bash tools/qprof.sh "5 2 3 4"
bash tools/qfull.sh 5 "^k_flop$" prof_cfg5 1
bash tools/qfull.sh 5 "k_sym_block_hash|k_heavy_sort_units|k_heavy_run_units|k_heavy_run_small|k_predict" prof_cfg5_symbolic_predict 8
timeout 900 python tools/shard_projection.py > gpurun_out/shard_proj.json 2> gpurun_out/shard_proj.err
