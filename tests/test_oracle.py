"""CPU: pins the C oracle (oracle/spnnz_oracle.c) before it is trusted as the
GPU checker.  Two anchors:
  * the reference's own known-answer tests, restated
    (proj/tests/test_flop.cpp, test_symbolic.cpp, test_predict.cpp,
    acceptance.cpp) -- cited per test;
  * golden fixtures produced by the reference itself (tests/golden/, made by
    make_golden.py from oracle/_ref).
"""
import math

import numpy as np
import pytest

from paper_2207_13848_b200 import gen
from tests.util import dense_bool_multiply_row_nnz, dense_flop_count, digest, identity, upper_2x2, csr

UNCAPPED = -1


# ----------------------------------------------------------- rng / sampler
def test_splitmix_known_answers(oracle, golden):
    for seed, vals in golden["refkat"]["splitmix"].items():
        assert [hex(x) for x in oracle.splitmix(int(seed), 5)] == vals
    assert oracle.splitmix(0, 1)[0] == 0xE220A8397B1DCDAF


def test_sample_plan_matches_reference_plans(oracle, golden):
    for rec in golden["refkat"]["plans"]:
        rows, n, p = oracle.make_sample_plan(rec["m"], rec["seed"], rec["fraction"], rec["cap"])
        assert n == rec["n"] and p == rec["p"]
        assert rows[:8].tolist() == rec["head"] and int(rows[-1]) == rec["last"]
        assert digest(rows) == rec["digest"]


def test_sample_count_formula(oracle):
    # test_predict.cpp:26-33 and :52-58
    for m, n in [(1000, 3), (1000000, 300), (100, 1), (1, 1), (100000, 300), (13514, 41)]:
        assert oracle.sample_count(m, 0.003, 300)[0] == n
    assert oracle.sample_count(1000, 0.01, 50)[0] == 10
    assert oracle.sample_count(100000, 0.01, 50)[0] == 50
    _, p = oracle.sample_count(5000, 0.003, 300)
    assert p == 15.0 / 5000.0  # test_predict.cpp:39
    with pytest.raises(ValueError):  # test_predict.cpp:48-50
        oracle.sample_count(0, 0.003, 300)


def test_survey_sample_indices(oracle):
    # SURVEY.md §8c, derived from the reference make_sample_plan
    rows, n, _ = oracle.make_sample_plan(4096, 1, 0.01, 300)
    assert n == 41 and rows[:5].tolist() == [2320, 3054, 3977, 1820, 1819] and rows[-1] == 3530
    rows, n, _ = oracle.make_sample_plan(1 << 20, 2, 0.003, UNCAPPED)
    assert n == 3146 and rows[:5].tolist() == [619907, 785540, 624571, 802600, 326724]
    rows, n, _ = oracle.make_sample_plan(1 << 24, 5, 0.001, 300)
    assert rows[-1] == 14209307


# ------------------------------------------------------------------ flop
def test_flop_identity_and_upper(oracle):
    eye = identity(4)  # test_flop.cpp:26-32
    f, t, m = oracle.compute_flop(eye, eye)
    assert f.tolist() == [1, 1, 1, 1] and t == 4 and m == 1
    u = upper_2x2()  # test_flop.cpp:34-40
    f, t, m = oracle.compute_flop(u, u)
    assert f.tolist() == [3, 1] and t == 4 and m == 3


def test_flop_rejects_mismatch_and_empty(oracle):
    with pytest.raises(ValueError):  # test_flop.cpp:42-44
        oracle.compute_flop(identity(3), identity(4))
    empty = csr(0, 0, [])  # test_flop.cpp:46-54
    f, t, m = oracle.compute_flop(empty, empty)
    assert len(f) == 0 and t == 0 and m == 0


def test_flop_dense_oracle_trials(oracle, golden):
    # test_flop.cpp:56-68 (seed 2024, 200 trials), pinned to the reference run
    rng = gen.SplitMix64(2024)
    for rec in golden["trials"]["flop_dense_oracle"]["trials"]:
        m, k, n = 1 + rng.next_below(60), 1 + rng.next_below(60), 1 + rng.next_below(60)
        d = 0.02 + 0.3 * rng.next_double()
        a = gen.random_pattern(m, k, d, rng)
        b = gen.random_pattern(k, n, d, rng)
        assert (m, k, n) == (rec["m"], rec["k"], rec["n"])
        f, t, mx = oracle.compute_flop(a, b)
        assert t == rec["F"] == dense_flop_count(a, b)
        assert mx == rec["max"] and digest(f) == rec["flop"]


def test_flop_b_column_invariance(oracle):
    # test_flop.cpp:70-89
    rng = gen.SplitMix64(5)
    a = gen.random_pattern(20, 20, 0.2, rng)
    b = gen.random_pattern(20, 30, 0.2, rng)
    shifted = csr(b.rows, b.cols, [list(range(int(b.rpt[i + 1] - b.rpt[i]))) for i in range(b.rows)])
    f1, t1, _ = oracle.compute_flop(a, b)
    f2, t2, _ = oracle.compute_flop(a, shifted)
    assert (f1 == f2).all() and t1 == t2


def test_flop_thread_invariance():
    # test_flop.cpp:91-102
    from oracle.pyoracle import Oracle
    rng = gen.SplitMix64(6)
    a = gen.random_pattern(123, 77, 0.1, rng)
    b = gen.random_pattern(77, 91, 0.1, rng)
    base = Oracle(threads=1).compute_flop(a, b)
    for th in (2, 3, 8):
        f, t, m = Oracle(threads=th).compute_flop(a, b)
        assert (f == base[0]).all() and t == base[1] and m == base[2]


def test_sampled_flop(oracle):
    # test_flop.cpp:104-123
    eye = identity(4)
    f, _, _ = oracle.compute_flop(eye, eye)
    assert oracle.sampled_flop(f, [0, 1, 2, 3]) == 4
    assert oracle.sampled_flop(f, []) == 0
    u = upper_2x2()
    fu, _, _ = oracle.compute_flop(u, u)
    assert oracle.sampled_flop(fu, [0, 0]) == 6
    f2, _, _ = oracle.compute_flop(identity(2), identity(2))
    with pytest.raises(ValueError):
        oracle.sampled_flop(f2, [2])


# -------------------------------------------------------------- symbolic
def test_symbolic_known_answers(oracle):
    u = upper_2x2()  # test_symbolic.cpp:55-61
    f, _, mx = oracle.compute_flop(u, u)
    nnz, z = oracle.exact_symbolic(u, u, f, mx)
    assert nnz.tolist() == [2, 1] and z == 3
    a = csr(1, 2, [[0, 1]])  # test_symbolic.cpp:37-43: union {0,1}
    b = csr(2, 2, [[0, 1], [1]])
    f, _, mx = oracle.compute_flop(a, b)
    assert oracle.exact_symbolic(a, b, f, mx)[0].tolist() == [2]
    a0 = csr(1, 2, [[]])  # test_symbolic.cpp:45-53: empty row
    f, _, mx = oracle.compute_flop(a0, identity(2))
    assert oracle.exact_symbolic(a0, identity(2), f, mx)[0].tolist() == [0]
    eye = identity(3)  # test_symbolic.cpp:29-35
    f, _, mx = oracle.compute_flop(eye, eye)
    assert oracle.exact_symbolic(eye, eye, f, mx)[0].tolist() == [1, 1, 1]
    # sampled edge cases, test_symbolic.cpp:135-149
    f, _, mx = oracle.compute_flop(u, u)
    assert oracle.sampled_symbolic(u, u, f, mx, [])[1] == 0
    assert oracle.sampled_symbolic(u, u, f, mx, [0])[1] == 2
    assert oracle.sampled_symbolic(u, u, f, mx, [0, 0, 1])[1] == 5
    with pytest.raises(ValueError):
        oracle.sampled_symbolic(u, u, f, mx, [2])


def test_symbolic_dense_oracle_trials(oracle, golden):
    # test_symbolic.cpp:63-77 (seed 31337, 100 trials)
    rng = gen.SplitMix64(31337)
    for rec in golden["trials"]["symbolic_dense_oracle"]["trials"]:
        m, k, n = 1 + rng.next_below(80), 1 + rng.next_below(80), 1 + rng.next_below(80)
        d = 0.01 + 0.25 * rng.next_double()
        a = gen.random_pattern(m, k, d, rng)
        b = gen.random_pattern(k, n, d, rng)
        f, _, mx = oracle.compute_flop(a, b)
        nnz, z = oracle.exact_symbolic(a, b, f, mx)
        assert (nnz == dense_bool_multiply_row_nnz(a, b)).all()
        assert z == rec["Z"] and digest(nnz) == rec["nnz"]
        assert (nnz <= f).all() and ((f == 0) | (nnz >= 1)).all()  # :79-92


def test_acceptance_oracle_trials(oracle, golden):
    # acceptance.cpp:147-169 (seed 42424242, 1000 trials up to 200^3)
    rng = gen.SplitMix64(42424242)
    mism = 0
    for i, rec in enumerate(golden["trials"]["acceptance_oracle"]["trials"]):
        m, k, n = 1 + rng.next_below(200), 1 + rng.next_below(200), 1 + rng.next_below(200)
        da, db = 0.002 + 0.25 * rng.next_double(), 0.002 + 0.25 * rng.next_double()
        a = gen.random_pattern(m, k, da, rng)
        b = gen.random_pattern(k, n, db, rng)
        f, _, mx = oracle.compute_flop(a, b)
        nnz, z = oracle.exact_symbolic(a, b, f, mx)
        mism += digest(nnz) != rec["nnz"] or z != rec["Z"] or digest(f) != rec["flop"]
        if i % 50 == 0:  # the dense check is cubic; sample it
            assert (nnz == dense_bool_multiply_row_nnz(a, b)).all()
    assert mism == 0


def test_sampled_all_rows_equals_exact(oracle):
    # test_symbolic.cpp:124-133
    rng = gen.SplitMix64(11)
    a = gen.random_pattern(60, 60, 0.12, rng)
    b = gen.random_pattern(60, 60, 0.12, rng)
    f, _, mx = oracle.compute_flop(a, b)
    assert oracle.sampled_symbolic(a, b, f, mx, np.arange(60))[1] == oracle.exact_symbolic(a, b, f, mx)[1]


# ------------------------------------------------------------ estimators
def test_estimator_arithmetic(oracle):
    z1, z2, cr = oracle.estimators(300, 100, 30000, 0.003)  # test_predict.cpp:74-81
    assert cr == 3.0 and z2 == 10000.0
    assert math.isclose(z1, 100 / 0.003)
    z1, z2, cr = oracle.estimators(0, 0, 12345, 0.5)  # :83-88 degenerate
    assert cr == 1.0 and z2 == 12345.0 and z1 == 0.0
    with pytest.raises(ValueError):  # :60-72
        oracle.estimators(1, 1, 1, 0.0)


def test_row_structure_views(oracle):
    # test_predict.cpp:90-112
    f = np.array([3, 1, 0], np.int64)
    assert oracle.predict_row_structure(f, 1.0).tolist() == [3.0, 1.0, 0.0]
    r = oracle.predict_row_structure(f, 4.0 / 3.0)
    assert math.isclose(r[0], 2.25, rel_tol=1e-12) and math.isclose(r[1], 0.75, rel_tol=1e-12)
    assert oracle.predict_row_structure_ceil(f, 4.0 / 3.0).tolist() == [3, 1, 0]
    with pytest.raises(ValueError):
        oracle.predict_row_structure(f, 0.0)
    with pytest.raises(ValueError):
        oracle.predict_row_structure_ceil(f, -1.0)


def test_error_report_examples(oracle):
    # test_predict.cpp:114-144
    e1, ef, e2, res = oracle.error_report(125.0, 1000.0 / 130.0 * 12.5, 130, 100, 1000, 0.1)
    assert math.isclose(e1, 0.25, rel_tol=1e-12) and math.isclose(ef, 0.30, rel_tol=1e-12)
    assert abs(abs(e2) * 100 - 3.85) < 0.005 and res <= 1e-9 * max(1.0, abs(e2))
    for bad in [(1.0, 1.0, 1, 0, 10, 0.1), (1.0, 1.0, 1, 10, 0, 0.1), (1.0, 1.0, 1, 10, 10, 0.0)]:
        with pytest.raises(ValueError):
            oracle.error_report(*bad)


def test_identity_predicts_exactly(oracle):
    # test_predict.cpp:146-157
    for n in (10, 100, 1000):
        for seed in (1, 7, 99):
            eye = identity(n)
            rep, *_ = oracle.run_prediction(eye, eye, seed, 0.003, 300)
            assert rep.predicted_cr == 1.0 and rep.z2_star == float(n)


def test_pipeline_matches_reference_runs(oracle, golden):
    # test_predict.cpp:184-217 loop, pinned to the reference's own pipeline
    rng = gen.SplitMix64(123)
    for rec in golden["trials"]["predict_pipeline"]["trials"]:
        n = 20 + rng.next_below(150)
        a = gen.random_pattern(n, n, 0.1, rng)
        b = gen.random_pattern(n, n, 0.1, rng)
        seed = rng.next_u64()
        assert (n, seed) == (rec["n"], rec["seed"])
        rep, flop, ceil, real = oracle.run_prediction(a, b, seed, 0.003, 300)
        for k, v in rec["report"].items():
            assert getattr(rep, k) == v, k
        assert digest(ceil) == rec["ceil"]
        # properties, test_predict.cpp:194-205
        assert math.isclose(rep.z2_star * rep.predicted_cr, rep.total_flop, rel_tol=1e-12)
        assert rep.sampled_nnz <= rep.sampled_flop
        assert math.isclose(real.sum(), rep.z2_star, rel_tol=1e-9)


def test_exhaustive_plan_is_exact(oracle):
    # test_predict.cpp:159-182, acceptance.cpp:201-231
    rng = gen.SplitMix64(77)
    for _ in range(10):
        n = 5 + rng.next_below(60)
        a = gen.random_pattern(n, n, 0.15, rng)
        b = gen.random_pattern(n, n, 0.15, rng)
        f, F, mx = oracle.compute_flop(a, b)
        _, Z = oracle.exact_symbolic(a, b, f, mx)
        if Z == 0:
            continue
        _, z = oracle.sampled_symbolic(a, b, f, mx, np.arange(n))
        fs = oracle.sampled_flop(f, np.arange(n))
        z1, z2, _ = oracle.estimators(fs, z, F, 1.0)
        assert z1 == Z and z2 == Z
        assert oracle.error_report(z1, z2, fs, Z, F, 1.0)[:3] == (0.0, 0.0, 0.0)


# ------------------------------------------------------------ configs
def test_config1_matches_reference_arrays(oracle, golden):
    a, b = gen.make_config(1)
    c1 = golden["configs"]["1"]
    assert digest(a.rpt) == c1["input"]["a_rpt"] and digest(a.col) == c1["input"]["a_col"]
    arr = golden["cfg1"]
    f, F, mx = oracle.compute_flop(a, b)
    assert (f == arr["flop"]).all() and F == c1["F"] and mx == c1["max"]
    nnz, Z = oracle.exact_symbolic(a, b, f, mx)
    assert (nnz == arr["exact_nnz"]).all() and Z == c1["Z"]
    for label, cap in (("uncapped", UNCAPPED), ("cap300", 300)):
        rep, _, ceil, real = oracle.run_prediction(a, b, 1, 0.01, cap)
        for k, v in c1["modes"][label]["report"].items():
            assert getattr(rep, k) == v, k
        assert (ceil == arr[f"ceil_{label}"]).all()
        assert (real == arr[f"real_{label}"]).all()


@pytest.mark.parametrize("cfg", [3, 4])
def test_config_digests(oracle, golden, cfg):
    """Configs 3 and 4 end to end on the oracle vs the reference's digests
    (seconds on CPU); config 3 also against the stencil closed forms."""
    if str(cfg) not in golden["configs"]:
        pytest.skip("configs.json lacks this config (make_golden.py --big)")
    rec = golden["configs"][str(cfg)]
    a, b = gen.make_config(cfg)
    assert digest(a.rpt) == rec["input"]["a_rpt"] and digest(a.col) == rec["input"]["a_col"]
    f, F, mx = oracle.compute_flop(a, b)
    assert F == rec["F"] and mx == rec["max"] and digest(f) == rec["flop"]
    if cfg == 3:
        assert a.nnz() == 382 ** 3 and F == 1142 ** 3 and rec["Z"] == 634 ** 3
    info = gen.CONFIGS[cfg]
    for label, cap in (("uncapped", UNCAPPED), ("cap300", 300)):
        rep, _, ceil, _ = oracle.run_prediction(a, b, info["seed"], info["fraction"], cap)
        for k, v in rec["modes"][label]["report"].items():
            assert getattr(rep, k) == v, k
        assert digest(ceil) == rec["modes"][label]["ceil"]


def test_reference_ceil_pipeline_equals_full_pipeline():
    """bench.py's CPU arm composes the reference's functions without the real
    per-row view (the GPU step's outputs); its report and integer view equal
    those of the reference's run_prediction_with_plan pipeline."""
    from oracle.pyoracle import Reference
    if not Reference.available():
        pytest.skip("oracle/_ref not built")
    R = Reference(threads=2)
    a, _ = gen.make_config(1)
    h = R.matrix(a)
    try:
        for cap in (UNCAPPED, 300, 5):
            full, c_full = R.run_pipeline(h, h, 1, 0.01, cap, a.rows)
            lean, c_lean = R.run_pipeline(h, h, 1, 0.01, cap, a.rows, real_view=False)
            for k, _t in full._fields_:
                assert getattr(full, k) == getattr(lean, k), k
            assert (c_full == c_lean).all()
    finally:
        R.free_matrix(h)


@pytest.mark.parametrize("cfg", [1, 2, 3, 4, 5])
def test_config_error_reports_restated(oracle, golden, cfg):
    """The reference's error_report of every config's pinned exact Z
    (config 5: tests/golden/make_cfg5_exact.py, the reference's exact_symbolic
    over row slices) is reproduced by the oracle's restatement
    (predict.hpp:163-188), and Z <= F with the sampled CR >= 1."""
    rec = golden["configs"].get(str(cfg))
    if not rec or "Z" not in rec:
        pytest.skip("no exact Z pinned for this config")
    assert 0 < rec["Z"] <= rec["F"]
    for label, m in rec["modes"].items():
        if "errors" not in m:
            continue
        r = m["report"]
        e = oracle.error_report(r["z1_star"], r["z2_star"], r["sampled_flop"], rec["Z"], rec["F"], r["p"])
        assert list(e) == m["errors"], label
        assert r["predicted_cr"] >= 1.0


def test_config5_exact_pin_is_the_slicewise_reference():
    """Config 5's pin records how it was made, and the slicing was validated
    on config 2 (the same script's self-check against make_golden.py's
    whole-matrix reference run)."""
    import json
    import os
    rec = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "configs.json")))["5"]
    assert rec["Z"] == 127786666282
    assert "exact_symbolic" in rec["exact_method"] and len(rec["exact_nnz_blocks"]) == 16
