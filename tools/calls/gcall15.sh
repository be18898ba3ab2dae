# round-2 shard projection (config 5) and the corpus harness (default corpus + the overhead criterion)
mkdir -p gpurun_out
timeout 900 python tools/shard_projection.py --config 5 --ranks 1 2 4 8 > gpurun_out/proj5.json 2> gpurun_out/proj5.err; echo "proj rc=$?"
timeout 600 build/spnnz_corpus --csv gpurun_out/corpus.csv --json gpurun_out/corpus.json > gpurun_out/corpus.txt 2>&1; echo "corpus rc=$?"
timeout 600 build/spnnz_corpus --overhead > gpurun_out/overhead.txt 2>&1; echo "overhead rc=$?"
tail -5 gpurun_out/corpus.txt; tail -8 gpurun_out/overhead.txt
python -c "
import json; d=json.load(open('gpurun_out/proj5.json'))
for n,v in d['per_world'].items(): print(n, round(v['max_ms'],3), round(v['imbalance'],3), v.get('projected_speedup'), v.get('projected_efficiency'))
"
