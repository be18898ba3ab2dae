"""Prints the quick-bench lines written by tools/qb.sh."""
import json
import sys

for c in (sys.argv[1:] or ["5", "2", "3", "4"]):
    try:
        d = json.loads(open(f"gpurun_out/bench_cfg{c}.log").read().strip().splitlines()[-1])
    except Exception as e:  # noqa: BLE001
        print(c, "failed", e)
        continue
    ph = {k: round(v, 3) for k, v in d.get("phases_ms", {}).items()}
    print(f"cfg{c} {d['value']:.3e} {d['ms_per_step']:.3f} ms {ph}")
