"""Per-source-line instruction and stall shares of one kernel in an ncu report:
python tools/ncu_lines.py report.ncu-rep "<kernel name regex>" [top] [stall|inst]"""
import csv
import re
import subprocess
import sys


def lines(path, kernel_re, top=25, by="stall"):
    out = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv", "--print-source",
                          "cuda,sass", "-k", f"regex:{kernel_re}"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    cur, hdr, agg = None, None, {}
    for r in rows:
        if len(r) >= 2 and r[0] == "File Path":
            cur = r[1].split("/")[-1]
            continue
        if len(r) >= 2 and r[0] == "Line No":
            hdr = r
            continue
        if hdr is None or len(r) < 8 or r[0] == "":
            continue
        try:
            ex, st = float(r[7] or 0), float(r[4] or 0)
        except ValueError:
            continue
        k = (cur, int(r[0]))
        e = agg.setdefault(k, [0.0, 0.0, r[1][:90]])
        e[0] += ex
        e[1] += st
    tot = sum(v[0] for v in agg.values()) or 1
    tst = sum(v[1] for v in agg.values()) or 1
    res = []
    for k, (ex, st, src) in sorted(agg.items(), key=lambda kv: -kv[1][1 if by == "stall" else 0])[:top]:
        res.append(f"{ex / tot * 100:5.1f}% inst {st / tst * 100:5.1f}% stall {k[0]}:{k[1]}: {src}")
    res.append(f"total warp instructions {tot:.3e}")
    return "\n".join(res)


if __name__ == "__main__":
    print(lines(sys.argv[1], sys.argv[2], int(sys.argv[3]) if len(sys.argv) > 3 else 25,
                sys.argv[4] if len(sys.argv) > 4 else "stall"))
