python -m pytest tests -m gpu -x -q > gpurun_out/t16.log 2>&1; echo rc=$? >> gpurun_out/t16.log
./build/spnnz_corpus --overhead > gpurun_out/overhead.log 2>&1; echo rc=$? >> gpurun_out/overhead.log
./build/spnnz_corpus --csv gpurun_out/corpus.csv --json gpurun_out/corpus.json > gpurun_out/corpus.txt 2>&1; echo rc=$? >> gpurun_out/corpus.txt
B="python bench.py --no-e2e --no-cpu-baseline --no-accuracy"
$B --config 3 > gpurun_out/c16_3.log 2>&1
$B --config 4 > gpurun_out/c16_4.log 2>&1
timeout 900 python tools/shard_projection.py > gpurun_out/shard_proj.json 2> gpurun_out/shard_proj.err
