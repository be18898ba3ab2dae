"""Top SASS instructions of an ncu --set full report by warp-stall samples
(needs --import-source / -lineinfo captures): address, samples, L1 shared
wavefronts (actual / ideal), instruction.
  python tools/ncu_sass_top.py gpurun_out/prof.ncu-rep [N] [kernel-substring]"""
import csv
import subprocess
import sys


def main():
    path = sys.argv[1]
    top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
    want = sys.argv[3] if len(sys.argv) > 3 else ""
    out = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout.splitlines()
    kernel, hdr, rows = None, None, []
    for line in out:
        r = next(csv.reader([line]))
        if r and r[0] == "Kernel Name":
            kernel = r[1]
            hdr = None
            continue
        if r and r[0] == "Address":
            hdr = r
            continue
        if hdr and len(r) == len(hdr) and (want in (kernel or "")):
            rows.append((kernel, dict(zip(hdr, r))))
    tot = sum(int(d["Warp Stall Sampling (All Samples)"] or 0) for _, d in rows) or 1
    rows.sort(key=lambda kd: -int(kd[1]["Warp Stall Sampling (All Samples)"] or 0))
    print(f"total samples {tot}")
    stalls = [c for c in (hdr or []) if c.startswith("stall_") and "Not Issued" not in c]
    agg = {c: 0 for c in stalls}
    for _, d in rows:
        for c in stalls:
            agg[c] += int(d.get(c) or 0)
    print("stall reasons:", ", ".join(f"{c[6:]} {100*v/tot:.0f}%" for c, v in
                                      sorted(agg.items(), key=lambda kv: -kv[1]) if v))
    for k, d in rows[:top]:
        s = int(d["Warp Stall Sampling (All Samples)"] or 0)
        why = max(stalls, key=lambda c: int(d.get(c) or 0)) if stalls else ""
        print(f"{100*s/tot:5.1f}%  {why[6:]:12s} wf {d.get('L1 Wavefronts Shared','')}/{d.get('L1 Wavefronts Shared Ideal','')}"
              f"  {d['Address'][-5:]}  {d['Source'].strip()[:70]}")


if __name__ == "__main__":
    main()
