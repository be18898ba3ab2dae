mkdir -p gpurun_out; rm -f gpurun_out/rep_*.log
for rep in 1 2; do for c in 5 2; do
  for v in base hb2; do
    case $v in base) E="";; hb2) E="SPNNZ_HEAVY_BESIDE=2";; esac
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
for v in 0 1 2; do SPNNZ_HEAVY_BESIDE=$v python tools/shard_projection.py --config 5 --ranks 8 > gpurun_out/proj8_$v.json 2>/dev/null; python -c "
import json; d=json.load(open('gpurun_out/proj8_$v.json'))
for n,v in d['per_world'].items(): print('hb=$v', n, round(v['max_ms'],3), round(v['imbalance'],3))"; done
