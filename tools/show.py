"""Summary of bench.py JSON lines in gpurun_out/<name>.log files:
  python tools/show.py c4_3rows c4_3seg ...   (globs allowed: 'c4_*')"""
import glob
import json
import os
import sys

names = []
for a in sys.argv[1:]:
    hits = sorted(glob.glob(os.path.join("gpurun_out", a + ".log")))
    names += [os.path.basename(h)[:-4] for h in hits] or [a]
for n in names:
    try:
        lines = [l for l in open(f"gpurun_out/{n}.log") if l.startswith("{")]
        d = json.loads(lines[-1])
    except Exception as e:  # noqa: BLE001
        print(f"{n:16s} failed: {e}")
        continue
    ph = {k: round(v * 1000, 1) for k, v in d.get("phases_ms", {}).items()}
    r = d.get("roofline", {})
    print(f"{n:16s} {d['ms_per_step']*1000:8.1f} us  flop frac {r.get('frac', 0):.3f}  floor "
          f"{(r.get('pattern_ceiling_ms') or 0)*1000:.1f} us  phases(us) {ph}")
