mkdir -p gpurun_out; rm -f gpurun_out/ab_*.log gpurun_out/ab_*_r*.txt
timeout 900 python -m pytest tests -m gpu -x -q -k "heavy or bin or config_vs or batching" > gpurun_out/t67.log 2>&1; echo "nopc tests rc=$?"; tail -1 gpurun_out/t67.log
for rep in 1 2; do for c in 5 2; do bash tools/ab.sh $c nopc; for f in gpurun_out/ab_${c}_*.log; do cp $f ${f%.log}_r$rep.txt; done; done; done
for f in gpurun_out/ab_*_r*.txt; do python - "$f" <<'PY'
import json,sys
try:
  d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
  print(sys.argv[1], round(d['ms_per_step']*1000,1), round(d['phases_ms']['symbolic']*1000,1))
except Exception as e: print(sys.argv[1], 'fail', e)
PY
done
