"""Generates tests/golden/* from the REFERENCE ITSELF (oracle/_ref, the
unmodified reference headers compiled in place by oracle/Makefile).

Run here, where /root/reference exists:  python tests/golden/make_golden.py [--big]
Outputs (committed):
  refkat.json        SplitMix64 / make_sample_plan known answers
  trials.json        per-trial totals + digests for the reference's own test
                     loops (test_flop.cpp:56-68, test_symbolic.cpp:63-77,
                     acceptance.cpp:147-169, test_predict.cpp:184-217)
  with_plan.json     run_prediction_with_plan on hand-built profiles (the
                     profile as an input: zeroed / inflated rows, another
                     total, a capacity violation) -- full arrays
  cfg1.npz           config 1 full arrays (flop, exact nnz, plans, ceil views)
  configs.json       configs 2-5: input digests, totals, report scalars and
                     per-row array digests (exact pass skipped for config 5)
"""
from __future__ import annotations

import argparse
import hashlib
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

from oracle.pyoracle import Reference  # noqa: E402
from paper_2207_13848_b200 import gen  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))
UNCAPPED = -1


def digest(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()[:32]


def refkat(R: Reference) -> dict:
    out = {"splitmix": {}, "plans": []}
    for seed in (0, 1, 42, 1234567, 2**64 - 1):
        out["splitmix"][str(seed)] = [hex(x) for x in R.splitmix(seed, 5)]
    for m, seed, frac, cap in [(4096, 1, 0.01, 300), (1 << 20, 2, 0.003, UNCAPPED),
                               (1 << 21, 3, 0.001, UNCAPPED), (1 << 20, 4, 0.005, UNCAPPED),
                               (1 << 24, 5, 0.001, UNCAPPED), (1 << 24, 5, 0.001, 300),
                               (1000, 1, 0.003, 300), (1000000, 1, 0.003, 300), (100, 1, 0.003, 300),
                               (1, 1, 0.003, 300), (100000, 1, 0.003, 300), (13514, 1, 0.003, 300),
                               (1000, 1, 0.01, 50), (100000, 1, 0.01, 50), (5000, 42, 0.003, 300),
                               (7, 99, 1.0, 300), (2**31 - 1, 77, 1e-6, UNCAPPED)]:
        rows, n, p = R.make_sample_plan(m, seed, frac, cap)
        out["plans"].append({"m": m, "seed": seed, "fraction": frac, "cap": cap, "n": n, "p": p,
                             "head": rows[:8].tolist(), "last": int(rows[-1]),
                             "digest": digest(rows)})
    return out


def trials(R: Reference) -> dict:
    out = {}

    def run(name, seed, count, dims, dens):
        rng = gen.SplitMix64(seed)
        rec = []
        for t in range(count):
            m, k, n = dims(rng)
            da, db = dens(rng)
            a = gen.random_pattern(m, k, da, rng)
            b = gen.random_pattern(k, n, db, rng)
            ha, hb = R.matrix(a), R.matrix(b)
            flop, F, mx, prof = R.compute_flop(ha, hb, a.rows, keep_profile=True)
            nnz, Z = R.exact_symbolic(ha, hb, prof, a.rows)
            rec.append({"m": m, "k": k, "n": n, "F": F, "max": mx, "Z": Z,
                        "flop": digest(flop), "nnz": digest(nnz),
                        "a": digest(a.col) + digest(a.rpt)[:8]})
            R.L.ref_profile_free(prof)
            R.free_matrix(ha)
            R.free_matrix(hb)
        out[name] = {"seed": seed, "trials": rec}

    # test_flop.cpp:56-68: 200 trials, dims 1+next_below(60), density 0.02+0.3u (same for A, B)
    def dims60(r):
        return 1 + r.next_below(60), 1 + r.next_below(60), 1 + r.next_below(60)

    def dens_flop(r):
        d = 0.02 + 0.3 * r.next_double()
        return d, d
    run("flop_dense_oracle", 2024, 200, dims60, dens_flop)

    # test_symbolic.cpp:63-77: 100 trials, dims 1+next_below(80), density 0.01+0.25u
    def dims80(r):
        return 1 + r.next_below(80), 1 + r.next_below(80), 1 + r.next_below(80)

    def dens_sym(r):
        d = 0.01 + 0.25 * r.next_double()
        return d, d
    run("symbolic_dense_oracle", 31337, 100, dims80, dens_sym)

    # acceptance.cpp:147-169: 1000 trials up to 200^3, separate densities
    def dims200(r):
        return 1 + r.next_below(200), 1 + r.next_below(200), 1 + r.next_below(200)

    def dens_acc(r):
        return 0.002 + 0.25 * r.next_double(), 0.002 + 0.25 * r.next_double()
    run("acceptance_oracle", 42424242, 1000, dims200, dens_acc)

    # test_predict.cpp:184-217: 40 pipelines, n = 20+next_below(150), density 0.1, seed from rng
    rng = gen.SplitMix64(123)
    rec = []
    for t in range(40):
        n = 20 + rng.next_below(150)
        a = gen.random_pattern(n, n, 0.1, rng)
        b = gen.random_pattern(n, n, 0.1, rng)
        seed = rng.next_u64()
        ha, hb = R.matrix(a), R.matrix(b)
        rep, ceil = R.run_pipeline(ha, hb, seed, 0.003, 300, a.rows)
        rows, _, _ = R.make_sample_plan(n, seed, 0.003, 300)
        rec.append({"n": n, "seed": seed, "report": {k: getattr(rep, k) for k, _ in rep._fields_},
                    "ceil": digest(ceil), "rows": rows.tolist()})
        R.free_matrix(ha)
        R.free_matrix(hb)
    out["predict_pipeline"] = {"seed": 123, "trials": rec}
    return out


def with_plan_cases(R: Reference) -> dict:
    """spnnz::run_prediction_with_plan (predict.hpp:202-216) on HAND-BUILT
    profiles: the profile is the function's input, so its flop is each row's
    hash-table size (tsize 0 counts 0, symbolic.hpp:35-36), f* and the views
    come from it and F is its total_flop.  Edits keep tsize >= the row's true
    FLOP (a smaller table would never terminate in the reference), except
    the capacity case, which the reference rejects (symbolic.hpp:37-40)."""
    rng = gen.SplitMix64(777)
    cases = []
    for t in range(12):
        m = 30 + rng.next_below(120)
        k = m if t % 3 else 20 + rng.next_below(100)
        n = 30 + rng.next_below(120)
        a = gen.random_pattern(m, k, 0.02 + 0.2 * rng.next_double(), rng)
        b = a if k == m and t % 3 == 1 else gen.random_pattern(k, n, 0.02 + 0.2 * rng.next_double(), rng)
        ha = R.matrix(a)
        hb = ha if b is a else R.matrix(b)
        flop, F, mx, _ = R.compute_flop(ha, hb, a.rows)
        kind = ["true", "zeroed", "inflated", "total", "capacity", "zeroed+inflated"][t % 6]
        f = flop.copy()
        total, cap = F, mx
        if "inflated" in kind:
            for i in range(m):
                f[i] = f[i] * (1 + rng.next_below(3)) + rng.next_below(5)
            cap = int(f.max())
            total = int(f.sum())
        if "zeroed" in kind:  # after inflating: a zeroed row stays 0
            for i in range(m):
                if rng.next_below(3) == 0:
                    f[i] = 0
        if kind == "total":
            total = F * 3 + 17
        if kind == "capacity":
            cap = mx - 1
        nsamp = 1 + rng.next_below(2 * m)
        rows = np.array([rng.next_below(m) for _ in range(nsamp)], np.int32)
        if kind == "capacity":
            rows = np.arange(m, dtype=np.int32)  # exhaustive: the max row is drawn
        p = nsamp / m if kind != "capacity" else 1.0
        rec = {"kind": kind, "m": m, "k": k, "n": n, "same": b is a,
               "a": {"rpt": a.rpt.tolist(), "col": a.col.tolist()},
               "b": None if b is a else {"rpt": b.rpt.tolist(), "col": b.col.tolist()},
               "flop": f.tolist(), "total": int(total), "max": int(cap),
               "rows": rows.tolist(), "p": p}
        try:
            rep, real, ceil = R.run_with_plan(ha, hb, f, total, cap, rows, p)
            rec["report"] = {k2: getattr(rep, k2) for k2, _ in rep._fields_}
            rec["real"] = real.tolist()
            rec["ceil"] = ceil.tolist()
        except ValueError as e:
            rec["error"] = str(e)
        cases.append(rec)
        R.free_matrix(ha)
        if hb != ha:
            R.free_matrix(hb)
    return {"seed": 777, "cases": cases}


def config_record(R: Reference, cfg: int, exact: bool) -> dict:
    a, b = gen.make_config(cfg)
    info = gen.CONFIGS[cfg]
    ha = R.matrix(a)
    hb = ha if b is a else R.matrix(b)
    t0 = time.time()
    flop, F, mx, prof = R.compute_flop(ha, hb, a.rows, keep_profile=True)
    rec = {"name": info["name"], "rows": a.rows, "cols": a.cols, "nnz": a.nnz(),
           "input": {"a_rpt": digest(a.rpt), "a_col": digest(a.col),
                     "b_rpt": digest(b.rpt), "b_col": digest(b.col)},
           "F": F, "max": mx, "flop": digest(flop), "modes": {}}
    for label, cap in (("uncapped", UNCAPPED), ("cap300", 300)):
        rows, n, p = R.make_sample_plan(a.rows, info["seed"], info["fraction"], cap)
        per, z = R.sampled_symbolic(ha, hb, prof, rows)
        rep, ceil = R.run_pipeline(ha, hb, info["seed"], info["fraction"], cap, a.rows)
        rec["modes"][label] = {"n": n, "p": p, "rows": digest(rows), "per_sample": digest(per),
                               "z_star": z, "report": {k: getattr(rep, k) for k, _ in rep._fields_},
                               "ceil": digest(ceil)}
        real = R.predict_row_structure(prof, rep.predicted_cr, a.rows)
        rec["modes"][label]["real"] = digest(real)
    if exact:
        nnz, Z = R.exact_symbolic(ha, hb, prof, a.rows)
        rec["Z"] = Z
        rec["exact_nnz"] = digest(nnz)
        for label in rec["modes"]:
            r = rec["modes"][label]["report"]
            rec["modes"][label]["errors"] = R.error_report(r["z1_star"], r["z2_star"],
                                                           r["sampled_flop"], Z, F, r["p"])
    rec["seconds"] = time.time() - t0
    R.L.ref_profile_free(prof)
    R.free_matrix(ha)
    if hb != ha:
        R.free_matrix(hb)
    return rec, a, b, flop


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--big", action="store_true", help="also configs 2-5 (minutes)")
    ap.add_argument("--configs", default="2,3,4,5")
    args = ap.parse_args()
    if not Reference.available():
        sys.exit("oracle/_ref not built: run `make -C oracle` where /root/reference exists")
    R = Reference(threads=0)
    with open(os.path.join(OUT, "refkat.json"), "w") as f:
        json.dump(refkat(R), f, indent=1)
    with open(os.path.join(OUT, "trials.json"), "w") as f:
        json.dump(trials(R), f)
    with open(os.path.join(OUT, "with_plan.json"), "w") as f:
        json.dump(with_plan_cases(R), f)
    # config 1: full arrays
    rec, a, b, flop = config_record(R, 1, exact=True)
    ha = R.matrix(a)
    _, _, _, prof = R.compute_flop(ha, ha, a.rows, keep_profile=True)
    nnz, _ = R.exact_symbolic(ha, ha, prof, a.rows)
    arrays = {"flop": flop, "exact_nnz": nnz}
    for label, cap in (("uncapped", UNCAPPED), ("cap300", 300)):
        rows, _, _ = R.make_sample_plan(a.rows, 1, 0.01, cap)
        per, _ = R.sampled_symbolic(ha, ha, prof, rows)
        rep, ceil = R.run_pipeline(ha, ha, 1, 0.01, cap, a.rows)
        arrays[f"rows_{label}"] = rows
        arrays[f"per_sample_{label}"] = per
        arrays[f"ceil_{label}"] = ceil
        arrays[f"real_{label}"] = R.predict_row_structure(prof, rep.predicted_cr, a.rows)
    np.savez_compressed(os.path.join(OUT, "cfg1.npz"), **arrays)
    R.L.ref_profile_free(prof)
    R.free_matrix(ha)
    recs = {"1": rec}
    if args.big:
        for cfg in [int(x) for x in args.configs.split(",")]:
            print(f"config {cfg} ...", flush=True)
            r, *_ = config_record(R, cfg, exact=(cfg != 5))
            recs[str(cfg)] = r
            print(f"  done in {r['seconds']:.1f}s", flush=True)
            with open(os.path.join(OUT, "configs.json"), "w") as f:
                json.dump(recs, f, indent=1)
    path = os.path.join(OUT, "configs.json")
    if os.path.exists(path) and not args.big:
        old = json.load(open(path))
        old.update(recs)
        recs = old
    with open(path, "w") as f:
        json.dump(recs, f, indent=1)


if __name__ == "__main__":
    main()
