mkdir -p gpurun_out; rm -f gpurun_out/rep_*.log
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/t43.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/t43.log
for rep in 1 2; do for c in 3 4 1; do
  for v in base s0; do
    case $v in base) E="";; s0) E="SPNNZ_SYM_SMALL=0";; esac
    env $E python bench.py --config $c --no-e2e --no-cpu-baseline --no-accuracy > gpurun_out/rep_${c}_${v}_$rep.log 2>&1
  done
done; done
python - <<'PY'
import json,glob,collections
r=collections.defaultdict(list)
for f in glob.glob('gpurun_out/rep_*.log'):
    _,c,v,k=f[:-4].split('/')[-1].split('_')
    try: r[(c,v)].append(json.loads(open(f).read().strip().splitlines()[-1])['ms_per_step']*1000)
    except Exception as e: print(f,e)
for k in sorted(r): print(k, [round(x,1) for x in sorted(r[k])])
PY
python tools/latency_probe.py
