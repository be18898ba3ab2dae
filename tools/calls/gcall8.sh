mkdir -p gpurun_out; rm -f gpurun_out/ab_*.log
timeout 900 python -m pytest tests -m gpu -x -q -k "flop or detached_rect" > gpurun_out/t8.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/t8.log
for c in 4 1; do bash tools/ab.sh $c nr f1; done
for f in gpurun_out/ab_*.log; do python - "$f" <<'PY'
import json,sys
try:
    d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
    print(sys.argv[1], round(d['ms_per_step']*1000,1), {k:round(v*1000,1) for k,v in d['phases_ms'].items()}, d['execution']['flop_kernel'][:12], round(d['roofline']['frac'],3))
except Exception as e: print(sys.argv[1], 'fail', e)
PY
done
python bench.py --config 4 --profile-steps 1 > gpurun_out/plain4.log 2>&1 && ncu --metrics gpu__time_duration.sum -k regex:k_flop_rs --csv --log-file gpurun_out/rs_base.csv python bench.py --config 4 --profile-steps 3 > /dev/null 2>&1
SPNNZ_GPU_LIB=build/var_nr/libspnnz_gpu.so ncu --metrics gpu__time_duration.sum -k regex:k_flop_rs --csv --log-file gpurun_out/rs_nr.csv python bench.py --config 4 --profile-steps 3 > /dev/null 2>&1
grep k_flop_rs gpurun_out/rs_base.csv | tail -3; grep k_flop_rs gpurun_out/rs_nr.csv | tail -3
