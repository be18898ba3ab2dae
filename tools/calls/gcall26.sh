mkdir -p gpurun_out; rm -f gpurun_out/ab_*.log
for v in s20 s20g3; do SPNNZ_GPU_LIB=build/var_$v/libspnnz_gpu.so timeout 600 python -m pytest tests -m gpu -x -q -k "every_bin or heavy_skewed" > gpurun_out/t26_$v.log 2>&1; echo "$v tests rc=$?"; done
for rep in 1 2; do bash tools/ab.sh 5 s20 s20g3; for f in gpurun_out/ab_5_*.log; do cp $f ${f%.log}_r$rep.txt; done; done
for f in gpurun_out/ab_5_*_r*.txt; do python - "$f" <<'PY'
import json,sys
try:
  d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
  print(sys.argv[1], round(d['ms_per_step']*1000,1), {k:round(v*1000,1) for k,v in d['phases_ms'].items()})
except Exception as e: print(sys.argv[1], 'fail', e)
PY
done
