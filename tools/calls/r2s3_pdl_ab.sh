# PDL A/B (SPNNZ_PDL=1 default vs 0) + parity
mkdir -p gpurun_out/c15
export SPNNZ_DEBUG_GRAPH=1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/c15/gputest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/c15/gputest.log
for r in 1 2; do
for p in 1 0; do
for c in 1 2 3 4 5; do
  SPNNZ_PDL=$p timeout 300 python bench.py --config $c --no-e2e --no-cpu-baseline --no-accuracy > gpurun_out/c15/b_p${p}_c${c}_r$r.log 2>&1
done; done; done
