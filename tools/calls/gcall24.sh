mkdir -p gpurun_out; rm -f gpurun_out/ab_*.log
timeout 1200 python -m pytest tests -m gpu -x -q -k "heavy or bin or config_vs or fuzz or unsorted or batching" > gpurun_out/t24.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/t24.log
for rep in 1 2; do bash tools/ab.sh 2; cp gpurun_out/ab_2_base.log gpurun_out/ab_2_base_r$rep.txt; bash tools/ab.sh 5; cp gpurun_out/ab_5_base.log gpurun_out/ab_5_base_r$rep.txt; done
for f in gpurun_out/ab_*_r*.txt; do python - "$f" <<'PY'
import json,sys
d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
print(sys.argv[1], round(d['ms_per_step']*1000,1), {k:round(v*1000,1) for k,v in d['phases_ms'].items()})
PY
done
