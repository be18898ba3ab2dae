mkdir -p gpurun_out; rm -f gpurun_out/ab_*.log
timeout 1200 python -m pytest tests -m gpu -x -q -k "heavy or bin or config_vs or fuzz or unsorted or with_plan or corpus" > gpurun_out/t16.log 2>&1; echo "tests rc=$?"; tail -5 gpurun_out/t16.log
bash tools/ab.sh 5 e8
SPNNZ_HEAVY_SWEEP=0 python bench.py --config 5 --no-e2e --no-cpu-baseline --no-accuracy > gpurun_out/ab_5_bk.log 2>&1
for f in gpurun_out/ab_*.log; do python - "$f" <<'PY'
import json,sys
try:
    d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
    print(sys.argv[1], round(d['ms_per_step']*1000,1), {k:round(v*1000,1) for k,v in d['phases_ms'].items()})
except Exception as e: print(sys.argv[1], 'fail', e, open(sys.argv[1]).read()[-500:])
PY
done
python bench.py --config 5 --profile-steps 1 > gpurun_out/plain5.log 2>&1 && ncu --metrics gpu__time_duration.sum -k regex:"k_heavy|k_sym" --clock-control none --csv --log-file gpurun_out/sw5.csv python bench.py --config 5 --profile-steps 1 > /dev/null 2>&1
python tools/launches.py gpurun_out/sw5.csv 2>/dev/null | head -20 || true
