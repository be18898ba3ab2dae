"""Prints tools/ab.sh results: python tools/ab_show.py <cfg> base g1 g2 ..."""
import json
import sys

cfg = sys.argv[1]
for v in sys.argv[2:]:
    try:
        d = json.loads(open(f"gpurun_out/ab_{cfg}_{v}.log").read().strip().splitlines()[-1])
        ph = {k: round(x, 3) for k, x in d["phases_ms"].items()}
        print(f"{v:8s} {d['ms_per_step']:.3f} ms {ph}")
    except Exception as e:  # noqa: BLE001
        print(v, "failed", e)
