mkdir -p gpurun_out; rm -f gpurun_out/ab_*.log gpurun_out/ab_*_r*.txt
for rep in 1 2 3 4; do bash tools/ab.sh 5 old; for f in gpurun_out/ab_5_*.log; do cp $f ${f%.log}_r$rep.txt; done; done
for f in gpurun_out/ab_*_r*.txt; do python - "$f" <<'PY'
import json,sys
try:
  d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
  print(sys.argv[1], round(d['ms_per_step']*1000,1), round(d['ms_per_step_median_rank0']*1000,1), round(d['phases_ms']['symbolic']*1000,1))
except Exception as e: print(sys.argv[1], 'fail', e)
PY
done
