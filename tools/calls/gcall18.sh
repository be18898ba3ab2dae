mkdir -p gpurun_out; rm -f gpurun_out/ab_*.log
for c in 5 2 4; do
  bash tools/ab.sh $c
  SPNNZ_HEAVY_BESIDE=1 python bench.py --config $c --no-e2e --no-cpu-baseline --no-accuracy > gpurun_out/ab_${c}_hb.log 2>&1
  SPNNZ_HEAVY_BESIDE=1 SPNNZ_TIERS_BESIDE=1 python bench.py --config $c --no-e2e --no-cpu-baseline --no-accuracy > gpurun_out/ab_${c}_hbtb.log 2>&1
done
for f in gpurun_out/ab_*.log; do python - "$f" <<'PY'
import json,sys
try:
    d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
    print(sys.argv[1], round(d['ms_per_step']*1000,1), {k:round(v*1000,1) for k,v in d['phases_ms'].items()})
except Exception as e: print(sys.argv[1], 'fail', e, open(sys.argv[1]).read()[-500:])
PY
done
