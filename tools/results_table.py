"""Prints DESIGN.md §8's results table from profiles/<round>_bench_cfg*.json and
profiles/<round>_ref_cfg*.json:  python tools/results_table.py [r02]"""
import json
import os
import sys

R = sys.argv[1] if len(sys.argv) > 1 else "r02"
P = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "profiles")


def load(name):
    return json.load(open(os.path.join(P, f"{R}_{name}.json")))


print("| config | step (device) | A-nnz/s device | e2e A-nnz/s | reference | e2e / ref | FLOP pass | of HBM | of pattern floor | predict of HBM | symbolic | products/s | launches/step |")
print("|---|---|---|---|---|---|---|---|---|---|---|---|---|")
for c, cap in [(1, ""), (2, ""), (3, ""), (4, ""), (5, ""), (5, "_cap300")]:
    d = load(f"bench_cfg{c}{cap}")
    try:
        r = load(f"ref_cfg{c}{cap}")
    except FileNotFoundError:
        r = None
    ph, rf = d["phases_ms"], d["roofline"]
    e2e = d["e2e"]["value"] if d.get("e2e") else None
    ref = r["value"] if r else (d["cpu_baseline"]["value"] if d.get("cpu_baseline") else None)
    cores = r["cpu_baseline"]["cores"] if r else None
    pf = rf.get("pattern_ceiling_frac")
    print(f"| {c}{' cap 300' if cap else ''} | {d['ms_per_step'] * 1e3:.1f} us | {d['value']:.3g} | "
          f"{e2e and format(e2e, '.3g')} | {ref and format(ref, '.3g')} ({cores} cores) | "
          f"{(e2e / ref) if e2e and ref else float('nan'):.1f}x | {ph['flop'] * 1e3:.1f} us | "
          f"{rf['frac'] * 100:.1f} % | {pf and format(pf * 100, '.0f')} % | "
          f"{d['roofline_predict'].get('frac', 0) * 100:.0f} % | {ph['symbolic'] * 1e3:.0f} us | "
          f"{d['roofline_symbolic']['products_per_s']:.3g} | {d['gpu_launches'] / d['steps']:.0f} |")
    if d.get("accuracy"):
        a = d["accuracy"]
        print(f"|   | accuracy: |eps2| {a['abs_rel_err_z2'] * 100:.4f} %, exact pass {a['exact_pass_s'] * 1e3:.1f} ms, "
              f"overhead {a['overhead_fraction']:.4f}, clocks {d['clocks']} |")
