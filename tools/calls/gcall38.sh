mkdir -p gpurun_out; rm -f gpurun_out/rep_*.log
for c in 5; do
  for v in base p10 p8 p6 p8h p6h p4h; do
    case $v in base) E="";; p10) E="SPNNZ_FLOP_PERSIST=10";; p8) E="SPNNZ_FLOP_PERSIST=8";; p6) E="SPNNZ_FLOP_PERSIST=6";;
      p8h) E="SPNNZ_FLOP_PERSIST=8 SPNNZ_HEAVY_BESIDE=2 SPNNZ_HEAVY_PRIO=1";; p6h) E="SPNNZ_FLOP_PERSIST=6 SPNNZ_HEAVY_BESIDE=2 SPNNZ_HEAVY_PRIO=1";;
      p4h) E="SPNNZ_FLOP_PERSIST=4 SPNNZ_HEAVY_BESIDE=2 SPNNZ_HEAVY_PRIO=1";; esac
    env $E python bench.py --config $c --no-e2e --no-cpu-baseline --no-accuracy > gpurun_out/rep_${c}_${v}_1.log 2>&1
  done
done
python - <<'PY'
import json,glob,collections
for f in sorted(glob.glob('gpurun_out/rep_*.log')):
    try:
        d=json.loads(open(f).read().strip().splitlines()[-1]); print(f, round(d['ms_per_step']*1000,1), {k:round(v*1000,1) for k,v in d['phases_ms'].items()})
    except Exception as e: print(f,e)
PY
SPNNZ_FLOP_PERSIST=6 SPNNZ_HEAVY_BESIDE=2 SPNNZ_HEAVY_PRIO=1 python tools/timeline.py 5 3 2>&1 | grep -E "timeline|heavy " | tail -7
