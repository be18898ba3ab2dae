mkdir -p gpurun_out; rm -f gpurun_out/ab_*.log
timeout 900 python -m pytest tests -m gpu -x -q -k "flop or detached or fuzz or config_vs" > gpurun_out/t6.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/t6.log
for c in 4 1; do bash tools/ab.sh $c f1 f3; SPNNZ_FLOP_RS=0 python bench.py --config $c --no-e2e --no-cpu-baseline --no-accuracy > gpurun_out/ab_${c}_rb.log 2>&1; done
for f in gpurun_out/ab_*.log; do python - "$f" <<'PY'
import json,sys
try:
    d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
    print(sys.argv[1], round(d['ms_per_step']*1000,1), {k:round(v*1000,1) for k,v in d['phases_ms'].items()}, d['execution']['flop_kernel'][:12], round(d['roofline']['frac'],3))
except Exception as e: print(sys.argv[1], 'fail', e)
PY
done
python bench.py --config 4 --profile-steps 1 > gpurun_out/plain4.log 2>&1 && ncu --set full --clock-control none --import-source on -k "regex:k_flop_rs" -c 1 -o gpurun_out/p_rs4c -f python bench.py --config 4 --profile-steps 1 > gpurun_out/p_rs4c.log 2>&1
