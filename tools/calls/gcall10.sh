mkdir -p gpurun_out; rm -f gpurun_out/ab_*.log
timeout 900 python -m pytest tests -m gpu -x -q -k "predict or config_vs or fuzz" > gpurun_out/t10.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/t10.log
for c in 2 3 5; do bash tools/ab.sh $c u2 u8 m4; done
for f in gpurun_out/ab_*.log; do python - "$f" <<'PY'
import json,sys
try:
    d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
    print(sys.argv[1], round(d['ms_per_step']*1000,1), {k:round(v*1000,1) for k,v in d['phases_ms'].items()}, round(d['roofline_predict']['frac'],3))
except Exception as e: print(sys.argv[1], 'fail', e)
PY
done
