"""Summarise bench logs named b_<variant>_c<config>_r<run>.log in a directory:
mean step ms and phase ms per (variant, config)."""
import glob, json, os, re, sys
from collections import defaultdict

d = sys.argv[1]
rows = defaultdict(list)
for f in sorted(glob.glob(os.path.join(d, "b_*_c*_r*.log"))):
    m = re.match(r"b_(.+)_c(\d+)_r(\d+)\.log", os.path.basename(f))
    lines = [x for x in open(f) if x.startswith("{")]
    if not lines:
        print("no line:", f, open(f).read()[-300:])
        continue
    j = json.loads(lines[-1])
    rows[(m.group(2), m.group(1))].append(j)
for (c, v), js in sorted(rows.items()):
    ms = [j["ms_per_step"] for j in js]
    ph = js[-1].get("phases_ms", {})
    print(f"cfg {c} {v:>10}: step " + " ".join(f"{x*1e3:8.1f}" for x in ms) + " us | " +
          " ".join(f"{k} {val*1e3:.1f}" for k, val in ph.items()))
