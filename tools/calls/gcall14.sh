mkdir -p gpurun_out; rm -f gpurun_out/ab_*.log
bash tools/ab.sh 5
SPNNZ_HEAVY_INTERVALS=1 python bench.py --config 5 --no-e2e --no-cpu-baseline --no-accuracy > gpurun_out/ab_5_iv.log 2>&1
bash tools/ab.sh 2
for f in gpurun_out/ab_*.log; do python - "$f" <<'PY'
import json,sys
try:
    d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
    print(sys.argv[1], round(d['ms_per_step']*1000,1), {k:round(v*1000,1) for k,v in d['phases_ms'].items()})
except Exception as e: print(sys.argv[1], 'fail', e)
PY
done
SPNNZ_HEAVY_INTERVALS=1 ncu --metrics gpu__time_duration.sum -k regex:k_heavy --clock-control none --csv --log-file gpurun_out/iv5.csv python bench.py --config 5 --profile-steps 1 > /dev/null 2>&1
grep -o '"[a-z_]*k_heavy[a-z_]*[^"]*".*"gpu__time_duration.sum","ns","[0-9]*"' gpurun_out/iv5.csv | sed 's/(.*"ns",/ /' 
