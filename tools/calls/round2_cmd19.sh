python -m pytest tests -m gpu -x -q > gpurun_out/t19.log 2>&1; echo rc=$? >> gpurun_out/t19.log
python tools/latency_probe.py > gpurun_out/latency19.log 2>&1
./build/spnnz_corpus --csv gpurun_out/corpus19.csv --json gpurun_out/corpus19.json > gpurun_out/corpus19.txt 2>&1
./build/spnnz_corpus --overhead > gpurun_out/overhead19.log 2>&1
timeout 900 python tools/shard_projection.py > gpurun_out/shard_proj19.json 2> gpurun_out/shard_proj19.err
