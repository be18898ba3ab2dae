mkdir -p gpurun_out; rm -f gpurun_out/ab_*.log
for rep in 1 2; do for c in 2 5; do bash tools/ab.sh $c t64 t256 t32; for f in gpurun_out/ab_${c}_*.log; do cp $f ${f%.log}_r$rep.txt; done; done; done
for f in gpurun_out/ab_*_r*.txt; do python - "$f" <<'PY'
import json,sys
try:
  d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
  print(sys.argv[1], round(d['ms_per_step']*1000,1), round(d['phases_ms']['symbolic']*1000,1))
except Exception as e: print(sys.argv[1], 'fail', e)
PY
done
