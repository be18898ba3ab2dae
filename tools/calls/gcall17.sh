mkdir -p gpurun_out; rm -f gpurun_out/ab_*.log
timeout 1200 python -m pytest tests -m gpu -x -q -k "heavy or bin or config_vs or fuzz or unsorted" > gpurun_out/t17.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/t17.log
for c in 5 2; do bash tools/ab.sh $c b4 u8 b4u; done
for f in gpurun_out/ab_*.log; do python - "$f" <<'PY'
import json,sys
try:
    d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
    print(sys.argv[1], round(d['ms_per_step']*1000,1), {k:round(v*1000,1) for k,v in d['phases_ms'].items()})
except Exception as e: print(sys.argv[1], 'fail', e, open(sys.argv[1]).read()[-500:])
PY
done
