"""Writes the judged profile summaries into profiles/ from ncu artefacts that a
gpurun call brought back into gpurun_out/:

  python tools/profile_round.py --round r01 \
      --launches gpurun_out/launches_cfg5.csv [--launches ...] \
      --full gpurun_out/prof_flop5.ncu-rep [--full ...]

For every launch list: profiles/<round>_launches_<name>.md (per-kernel count,
mean, total, share).  For every full capture: profiles/<round>_ncu_<name>.md
(key counters per kernel).  The k_flop capture also writes
--traffic CFG=capture: profiles/flop_traffic.json[CFG], the DRAM bytes of one
FLOP pass (all its kernels), which bench.py reports as roofline.traffic.
"""
import argparse
import json
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
sys.path.insert(0, HERE)

import launches as L  # noqa: E402
import ncu_summary as N  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--round", required=True)
    ap.add_argument("--launches", action="append", default=[])
    ap.add_argument("--full", action="append", default=[])
    ap.add_argument("--note", default="")
    ap.add_argument("--traffic", action="append", default=[],
                    help="CFG=path.ncu-rep: a full capture of one FLOP pass of config CFG")
    args = ap.parse_args()
    out = os.path.join(ROOT, "profiles")
    os.makedirs(out, exist_ok=True)
    for p in args.launches:
        name = os.path.splitext(os.path.basename(p))[0]
        with open(os.path.join(out, f"{args.round}_{name}.md"), "w") as f:
            f.write(f"# {args.round} launch list: {name}\n\n")
            f.write("`ncu --metrics gpu__time_duration.sum --clock-control none` over "
                    "`bench.py --config <c> --profile-steps 1` (tools/qprof.sh: load + one "
                    "predictor pass; per-launch times are cold-cache and serialised: compare "
                    "shares, not absolutes).\n\n```\n")
            f.write(L.summarize(p) + "\n```\n")
            if args.note:
                f.write("\n" + args.note + "\n")
    for p in args.full:
        name = os.path.splitext(os.path.basename(p))[0]
        data, units = N.rows(p)
        with open(os.path.join(out, f"{args.round}_{name}.md"), "w") as f:
            f.write(f"# {args.round} ncu --set full: {name}\n\n")
            for d in data:
                f.write(f"## {d.get('Kernel Name', '?')[:120]}\n\n| counter | value |\n|---|---|\n")
                for w in N.WANT[1:]:
                    if w in d:
                        f.write(f"| {w} | {d[w]} {units.get(w, '')} |\n")
                f.write("\n")
    # per-config DRAM traffic of one FLOP pass: the sum over its kernels
    # (k_degree, k_tile_rows, k_flop / k_flop_smem / k_flop_rb, k_flop_fixup)
    if args.traffic:
        path = os.path.join(out, "flop_traffic.json")
        try:
            allt = json.load(open(path))
            if "kernel" in allt:  # the round-1 single-config format
                allt = {}
        except Exception:
            allt = {}
        for spec in args.traffic:
            cfg, rep = spec.split("=", 1)
            data, units = N.rows(rep)

            def num(d, k):
                v = float(d[k].replace(",", ""))
                scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(units.get(k, ""), 1)
                return v * scale

            def dur_ms(d):
                u = units.get("gpu__time_duration.sum", "ms")
                return float(d["gpu__time_duration.sum"].replace(",", "")) * {
                    "ns": 1e-6, "nsecond": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0}.get(u, 1.0)

            ks = [d for d in data if any(x in d.get("Kernel Name", "") for x in ("k_degree", "k_tile_rows", "k_flop"))]
            main_k = max(ks, key=dur_ms)
            rd = sum(num(d, "dram__bytes_read.sum") for d in ks)
            wr = sum(num(d, "dram__bytes_write.sum") for d in ks)
            allt[cfg] = {"kernels": [d["Kernel Name"].split("(")[0] for d in ks],
                         "source": f"profiles/{args.round}_{os.path.splitext(os.path.basename(rep))[0]}.md",
                         "round": args.round,
                         "dram_bytes_per_launch": rd + wr, "dram_read": rd, "dram_write": wr,
                         "duration_ms": sum(dur_ms(d) for d in ks),
                         "l2_hit_rate_pct": float(main_k.get("lts__t_sector_hit_rate.pct", "nan").replace(",", "")),
                         "l1_hit_rate_pct": float(main_k.get("l1tex__t_sector_hit_rate.pct", "nan").replace(",", "")),
                         "l2_read_requests": float(main_k.get("lts__t_requests_srcunit_tex_op_read.sum",
                                                              "nan").replace(",", ""))}
        with open(path, "w") as g:
            json.dump(allt, g, indent=1)


if __name__ == "__main__":
    main()
