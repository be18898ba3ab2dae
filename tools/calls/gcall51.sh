mkdir -p gpurun_out; rm -f gpurun_out/rep_*.log
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/t51.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/t51.log
for rep in 1 2; do for c in 2 5; do
    python bench.py --config $c --no-e2e --no-cpu-baseline --no-accuracy > gpurun_out/rep_${c}_base_$rep.log 2>&1
done; done
python - <<'PY'
import json,glob,collections
r=collections.defaultdict(list)
for f in glob.glob('gpurun_out/rep_*.log'):
    _,c,v,k=f[:-4].split('/')[-1].split('_')
    try:
        d=json.loads(open(f).read().strip().splitlines()[-1]); r[(c,v)].append((round(d['ms_per_step']*1000,1), round(d['phases_ms']['symbolic']*1000,1)))
    except Exception as e: print(f,e)
for k in sorted(r): print(k, sorted(r[k]))
PY
