"""Small workloads for compute-sanitizer (memcheck / racecheck / synccheck):
every kernel family of the library on inputs the tools finish in minutes,
each result checked against the CPU oracle so a run that passes the tool is
also a correct run.  No torch (nothing but this library's kernels runs).

  compute-sanitizer --tool racecheck python tools/sanitize_cases.py [--quick]

Cases: config 1 (flop, sampled + exact symbolic, both sample caps), every
symbolic bin including heavy rows on the three heavy geometries (B.cols 2^20
one range, 2^24 unit-sorted ranges, 2^28 count/place buckets), the exact
pass in forced small heavy batches (merge-pool reuse), the FLOP kernels
(row blocks with the shared degree table, tile groups, banded row mode,
global gathers), run_prediction_with_plan on hand-built profiles, and
repeated calls (cached heavy sizes, CUDA-graph capture and replay).
"""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from oracle.pyoracle import Oracle  # noqa: E402  (the checker)
from paper_2207_13848_b200 import gen  # noqa: E402
from paper_2207_13848_b200.spnnz import CsrMatrix, FlopProfile, Predictor, SamplePlan, SamplePolicy  # noqa: E402


def csr(rows, cols, lists):
    rpt = np.zeros(rows + 1, np.int64)
    for i, r in enumerate(lists):
        rpt[i + 1] = rpt[i] + len(r)
    col = np.array([c for r in lists for c in r], np.int32)
    return CsrMatrix(rows, cols, rpt, col)


def check_all(P, O, a, b, seed=7, frac=0.05):
    P.load(a, None if b is a else b)
    pr = P.compute_flop()
    f, F, mx = O.compute_flop(a, b)
    assert (pr.flop_per_row == f).all() and pr.total_flop == F and pr.max_flop_row == mx
    ex = P.exact_symbolic()
    nnz, Z = O.exact_symbolic(a, b, f, mx)
    assert (ex.nnz_per_row == nnz).all() and ex.total_nnz == Z
    for cap in (-1, 300):
        rep = P.run_prediction(seed, SamplePolicy(frac, cap))
        orep, _, oceil, _ = O.run_prediction(a, b, seed, frac, cap)
        assert rep.stats.sampled_nnz == orep.sampled_nnz and rep.z2_star == orep.z2_star
        assert np.array_equal(rep.predicted_row_nnz_ceil, oceil)


def tier_case(ncols):
    rng = np.random.default_rng(ncols)
    nc = 3000
    b_lens = [1, 2, 3, 1, 2, 3, 1, 2, 3, 4] + list(rng.integers(0, 60, 2988)) + [2000, 2999]
    b = [sorted(int(c) * (ncols // nc) for c in rng.choice(nc, int(L), replace=False)) for L in b_lens]
    lens = [0, 1, 2, 5, 10, 40, 100, 200, 300, 700, 1500, 2500] + list(rng.integers(0, 200, 100))
    a = [sorted(int(c) for c in rng.choice(nc, int(L), replace=False)) for L in lens]
    a += [[0], [1, 2], [3, 4, 5], list(range(10))]
    return csr(len(a), nc, a), csr(nc, ncols, b)


def main():
    quick = "--quick" in sys.argv
    O = Oracle(threads=0)
    P = Predictor(0)
    done = []
    a, b = gen.make_config(1)
    check_all(P, O, a, b, 1, 0.01)
    done.append("config 1")
    for ncols in ([1 << 20] if quick else [1 << 20, 1 << 24, 1 << 28]):
        a, b = tier_case(ncols)
        check_all(P, O, a, b)
        done.append(f"every bin, B.cols 2^{ncols.bit_length() - 1}")
    os.environ["SPNNZ_HEAVY_BATCH_PRODUCTS"] = "20000"  # exact pass in many heavy batches
    a, b = tier_case(1 << 24)
    check_all(P, O, a, b)
    del os.environ["SPNNZ_HEAVY_BATCH_PRODUCTS"]
    done.append("small heavy batches")
    # FLOP kernels
    for env in ({"SPNNZ_FLOP_RB": "1"}, {"SPNNZ_FLOP_RB": "0"}, {"SPNNZ_FLOP_RB": "0", "SPNNZ_FLOP_SMEM": "0"},
                {"SPNNZ_FLOP_ROWS": "1", "SPNNZ_FLOP_SMEM": "0"}):
        os.environ.update(env)
        s = gen.stencil27(12, 10, 9)
        check_all(P, O, s, s)
        r = gen.uniform_len(6000, 4096, 0, 40, 3)
        rb_ = gen.uniform_len(4096, 20000, 0, 20, 4)
        check_all(P, O, r, rb_)
        for k in env:
            del os.environ[k]
        done.append(f"flop kernels {env}")
    # run_prediction_with_plan on hand-built profiles (the reference's outputs)
    cases = json.load(open(os.path.join(ROOT, "tests", "golden", "with_plan.json")))["cases"]
    for rec in cases[:6]:
        a = CsrMatrix(rec["m"], rec["k"], np.array(rec["a"]["rpt"], np.int64), np.array(rec["a"]["col"], np.int32))
        b = a if rec["same"] else CsrMatrix(rec["k"], rec["n"], np.array(rec["b"]["rpt"], np.int64),
                                            np.array(rec["b"]["col"], np.int32))
        P.load(a, None if rec["same"] else b)
        prof = FlopProfile(np.array(rec["flop"], np.int64), rec["total"], rec["max"])
        rows = np.array(rec["rows"], np.int32)
        try:
            rep = P.run_prediction_with_plan(SamplePlan(rows, len(rows), rec["p"], 0), prof)
            assert rep.stats.sampled_nnz == rec["report"]["sampled_nnz"]
            assert np.array_equal(rep.predicted_row_nnz_ceil, np.array(rec["ceil"], np.int64))
        except ValueError:
            assert "error" in rec
    done.append("with_plan, hand-built profiles")
    # repeated calls: cached heavy sizes, graph capture and replay
    a, b = tier_case(1 << 20)
    P.load(a, b)
    outs = [P.run_prediction(5, SamplePolicy(0.5, -1)) for _ in range(4)]
    assert all(o.stats.sampled_nnz == outs[0].stats.sampled_nnz for o in outs)
    done.append("repeated calls (graph replay)")
    if os.environ.get("SPNNZ_GUARD") == "1":  # guard bands after every library buffer
        import ctypes
        from paper_2207_13848_b200.capi import check, lib
        n, bad = ctypes.c_int64(), ctypes.c_int64()
        check(lib().spnnz_gpu_check_guards(ctypes.byref(n), ctypes.byref(bad)))
        assert n.value > 0 and bad.value == 0, f"{bad.value} of {n.value} guard bands overwritten"
        done.append(f"guard bands intact ({n.value} buffers)")
    P.close()
    print("sanitize cases ok:", "; ".join(done))


if __name__ == "__main__":
    main()
