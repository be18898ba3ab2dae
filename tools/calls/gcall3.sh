# row-stream FLOP kernel: parity tests, then config 4 / 1 A/B (staged rb, prefetch depth)
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -k "flop or detached_rect or config_vs_reference or fuzz" > gpurun_out/t3.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/t3.log
for c in 4 1; do
  bash tools/ab.sh $c a2 a4
  SPNNZ_FLOP_RS=0 python bench.py --config $c --no-e2e --no-cpu-baseline --no-accuracy > gpurun_out/ab_${c}_rb.log 2>&1
done
for f in gpurun_out/ab_*.log; do python - "$f" <<'PY'
import json,sys
try:
    d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
    print(sys.argv[1], round(d['ms_per_step']*1000,1), {k:round(v*1000,1) for k,v in d['phases_ms'].items()}, d['execution']['flop_kernel'], round(d['roofline']['frac'],3))
except Exception as e: print(sys.argv[1], 'fail', e)
PY
done
