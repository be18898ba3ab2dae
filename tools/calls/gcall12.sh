mkdir -p gpurun_out; rm -f gpurun_out/ab_*.log
timeout 1200 python -m pytest tests -m gpu -x -q -k "heavy or bin or config_vs or fuzz or unsorted or with_plan" > gpurun_out/t12.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/t12.log
bash tools/ab.sh 5 mt
for f in gpurun_out/ab_*.log; do python - "$f" <<'PY'
import json,sys
try:
    d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
    print(sys.argv[1], round(d['ms_per_step']*1000,1), {k:round(v*1000,1) for k,v in d['phases_ms'].items()})
except Exception as e: print(sys.argv[1], 'fail', e)
PY
done
python bench.py --config 5 --profile-steps 1 > gpurun_out/plain5.log 2>&1 && ncu --metrics gpu__time_duration.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum,l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum -k regex:k_heavy --clock-control none --csv --log-file gpurun_out/hv5.csv python bench.py --config 5 --profile-steps 1 > /dev/null 2>&1
python - <<'PY'
import csv
rows=list(csv.reader(open('gpurun_out/hv5.csv')))
h=None
for r in rows:
    if r and r[0]=='ID': h=r; continue
    if h and len(r)==len(h):
        d=dict(zip(h,r)); print(d['Kernel Name'][:40], d['Metric Name'], d['Metric Value'])
PY
