mkdir -p gpurun_out; rm -f gpurun_out/ab_*.log
for rep in 1 2; do bash tools/ab.sh 5 su8 su6; for f in gpurun_out/ab_5_*.log; do cp $f ${f%.log}_r$rep.txt; done; done
for f in gpurun_out/ab_5_*_r*.txt; do python - "$f" <<'PY'
import json,sys
try:
  d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
  print(sys.argv[1], round(d['ms_per_step']*1000,1), {k:round(v*1000,1) for k,v in d['phases_ms'].items()})
except Exception as e: print(sys.argv[1], 'fail', e)
PY
done
