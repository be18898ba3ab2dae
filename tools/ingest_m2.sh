#!/bin/bash
# Turns what tools/round2_final.sh brought back (gpurun_out/m2/) into the
# judged files under profiles/ (round tag $1, default r02): bench lines,
# reference-arm lines, launch lists, ncu summaries, FLOP traffic, the shard
# projection and the corpus reports.
R=${1:-r02}
O=gpurun_out/m2
P=profiles
last_json() { grep '^{' "$1" | tail -1 | python -c "import json,sys; print(json.dumps(json.loads(sys.stdin.read()), indent=1))"; }
for c in 1 2 3 4 5; do
  last_json $O/bench_cfg$c.log > $P/${R}_bench_cfg$c.json
  last_json $O/bench_cfg${c}_cap300.log > $P/${R}_bench_cfg${c}_cap300.json
  last_json $O/ref_cfg$c.log > $P/${R}_ref_cfg$c.json
done
last_json $O/ref_cfg5_cap300.log > $P/${R}_ref_cfg5_cap300.json
python -c "import json; print(json.dumps(json.load(open('$O/proj5.json')), indent=1))" > $P/${R}_shard_projection_cfg5.json
cp $O/corpus.csv $P/${R}_corpus_default.csv
cp $O/corpus.json $P/${R}_corpus_default.json
{ cat $O/corpus.txt; echo; echo "--- overhead criterion (acceptance.cpp:264-294 specs)"; cat $O/overhead.txt; echo;
  echo "--- per-call wall latency (tools/latency_probe.py, us)"; cat $O/latency.txt; } > $P/${R}_corpus_default.txt
L=""; for c in 1 2 3 4 5; do L="$L --launches $O/launches_cfg$c.csv"; done
F=""; T=""; for c in 2 3 4 5; do F="$F --full $O/flop_cfg$c.ncu-rep --full $O/symp_cfg$c.ncu-rep"; T="$T --traffic $c=$O/flop_cfg$c.ncu-rep"; done
python tools/profile_round.py --round $R $L $F $T
