"""The corpus harness (include/spnnz_gpu/harness.hpp, built as
build/spnnz_corpus) on the GPU: every case's sample count, exact NNZ, CR and
errors equal the oracle's computation of the reference's run_case
(bench.hpp:171-229), and the summary its summarize (:231-279)."""
import json
import math
import os
import subprocess

import numpy as np
import pytest

from paper_2207_13848_b200 import gen
from paper_2207_13848_b200.spnnz import CsrMatrix

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
EXE = os.path.join(ROOT, "build", "spnnz_corpus")
M64 = (1 << 64) - 1


def g6(v):
    return "na" if not math.isfinite(v) else "%.6g" % v


def case_seed(seed, idx):  # SplitMix64::fork(seed, idx).next_u64() (rng.hpp:34-37)
    m = gen.SplitMix64(seed ^ ((idx * 0xD1B54A32D192ED03) & M64))
    return gen.SplitMix64(m.next_u64()).next_u64()


def keep_left(m, n):
    rows = [m.col[m.rpt[i]:m.rpt[i + 1]] for i in range(m.rows)]
    rows = [r[r < n] for r in rows]
    rpt = np.concatenate([[0], np.cumsum([len(r) for r in rows])]).astype(np.int64)
    return CsrMatrix(m.rows, n, rpt, np.concatenate(rows + [np.zeros(0, np.int32)]).astype(np.int32))


def keep_top(m, n):
    return CsrMatrix(n, m.cols, m.rpt[: n + 1].copy(), m.col[: m.rpt[n]].copy())


SPECS = ["synth:uniform:2000x2000:nnz=4:seed=7", "synth:banded:1500x1500:nnz=6:bw=20:seed=3",
         "synth:power-law:2500x1800:nnz=5:skew=0.9:seed=11"]


def test_corpus_harness_matches_oracle(tmp_path, oracle):
    if not os.path.exists(EXE):
        pytest.skip("build/spnnz_corpus not built")
    lst = tmp_path / "list.txt"
    lst.write_text("# corpus\n" + "\n".join(SPECS) + "\n\n")
    out_json, out_csv = tmp_path / "r.json", tmp_path / "r.csv"
    r = subprocess.run([EXE, "--list", str(lst), "--json", str(out_json), "--csv", str(out_csv),
                        "--no-timings", "--seed", "42"], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr
    rep = json.loads(out_json.read_text())
    assert out_csv.read_text().splitlines()[0] == \
        "a,b,sample_num,cr,nnz_c,eps1_pct,eps_f_pct,eps2_pct,t_flop_s,t_predict_s,t_exact_s"
    mats = []
    for s in SPECS:
        sp = gen.parse_synthetic_spec(s)
        name = gen.synthetic_name(sp["model"], sp["rows"], sp["cols"], sp["target"], sp["seed"],
                                  sp["bandwidth"], sp["skew"])
        mats.append((name, gen.synthetic(sp["model"], sp["rows"], sp["cols"], sp["target"], sp["seed"],
                                         sp["bandwidth"], sp["skew"])))
    n = len(mats)
    assert len(rep["cases"]) == n * n and rep["failures"] == []
    e1s, efs, wins, abs1, absf, abs2 = [], [], 0, [], [], []
    for idx, c in enumerate(rep["cases"]):
        (an, a), (bn, b) = mats[idx // n], mats[idx % n]
        if a.cols > b.rows:
            a = keep_left(a, b.rows)
        elif a.cols < b.rows:
            b = keep_top(b, a.cols)
        f, F, mx = oracle.compute_flop(a, b)
        _, Z = oracle.exact_symbolic(a, b, f, mx)
        rows, num, p = oracle.make_sample_plan(a.rows, case_seed(42, idx), 0.003, 300)
        _, zs = oracle.sampled_symbolic(a, b, f, mx, rows)
        fs = oracle.sampled_flop(f, rows)
        z1, z2, _ = oracle.estimators(fs, zs, F, p)
        eps1, epsf, eps2, _ = oracle.error_report(z1, z2, fs, Z, F, p)
        assert (c["a"], c["b"], c["sample_num"], c["nnz_c"]) == (an, bn, num, Z)
        assert c["cr"] == g6(F / Z)
        assert (c["eps1_pct"], c["eps_f_pct"], c["eps2_pct"]) == (g6(eps1 * 100), g6(epsf * 100), g6(eps2 * 100))
        assert c["t_flop_s"] == "na"
        e1s.append(eps1)
        efs.append(epsf)
        wins += abs(eps2) < abs(eps1)
        abs1.append(abs(eps1))
        absf.append(abs(epsf))
        abs2.append(abs(eps2))
    s = rep["summary"]
    assert (s["cases_total"], s["cases_failed"], s["cases_degenerate"]) == (n * n, 0, 0)
    assert s["win_rate"] == g6(wins / (n * n))
    assert s["worst_abs_eps2_pct"] == g6(max(abs2) * 100)
    np.testing.assert_allclose(float(s["mean_abs_eps1_pct"]), np.mean(abs1) * 100, rtol=1e-5)
    np.testing.assert_allclose(float(s["pearson_eps1_epsf"]), np.corrcoef(e1s, efs)[0, 1], rtol=1e-4)


def test_corpus_harness_rejects_bad_sources(tmp_path):
    if not os.path.exists(EXE):
        pytest.skip("build/spnnz_corpus not built")
    lst = tmp_path / "list.txt"
    lst.write_text("HB/bcsstk01\n")
    r = subprocess.run([EXE, "--list", str(lst), "--no-timings"], capture_output=True, text=True, timeout=120)
    assert r.returncode == 1 and "network" in r.stderr
