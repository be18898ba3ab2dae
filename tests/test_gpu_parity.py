"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle and
the reference's golden fixtures, bit-exact for every integer output and for
the IEEE-double CR / Z1* / Z2* (north_star allows 1e-12 relative; we assert
equality).  Restates the reference's hot-path tests (proj/tests/test_flop.cpp,
test_symbolic.cpp, test_predict.cpp, acceptance.cpp) on the device.
"""
import os

import numpy as np
import pytest

from paper_2207_13848_b200 import gen, spnnz
from paper_2207_13848_b200.spnnz import Predictor, SamplePlan, SamplePolicy
from tests.util import csr, dense_bool_multiply_row_nnz, dense_flop_count, digest, identity, upper_2x2

pytestmark = pytest.mark.gpu
UNCAPPED = -1
CR_RTOL = 1e-12  # north_star tolerance for the compression ratio (we also check ==)


@pytest.fixture(scope="module")
def P():
    p = Predictor(0)
    yield p
    p.close()


def gpu_exact(P, a, b):
    P.load(a, b)
    prof = P.compute_flop()
    ex = P.exact_symbolic()
    return prof, ex


# ------------------------------------------------------------------ flop
def test_flop_known_answers(P):
    eye = identity(4)
    P.load(eye, eye)
    pr = P.compute_flop()
    assert pr.flop_per_row.tolist() == [1, 1, 1, 1] and pr.total_flop == 4 and pr.max_flop_row == 1
    u = upper_2x2()
    P.load(u, u)
    pr = P.compute_flop()
    assert pr.flop_per_row.tolist() == [3, 1] and pr.total_flop == 4 and pr.max_flop_row == 3


def test_flop_errors_and_empty(P):
    P.load(identity(3), identity(4))
    with pytest.raises(ValueError):  # test_flop.cpp:42-44
        P.compute_flop()
    e = csr(0, 0, [])
    P.load(e, e)
    pr = P.compute_flop()
    assert len(pr.flop_per_row) == 0 and pr.total_flop == 0 and pr.max_flop_row == 0


def test_flop_trials_vs_reference(P, golden):
    # test_flop.cpp:56-68 (200 trials, seed 2024) against the reference's digests
    rng = gen.SplitMix64(2024)
    for rec in golden["trials"]["flop_dense_oracle"]["trials"]:
        m, k, n = 1 + rng.next_below(60), 1 + rng.next_below(60), 1 + rng.next_below(60)
        d = 0.02 + 0.3 * rng.next_double()
        a = gen.random_pattern(m, k, d, rng)
        b = gen.random_pattern(k, n, d, rng)
        P.load(a, b)
        pr = P.compute_flop()
        assert pr.total_flop == rec["F"] == dense_flop_count(a, b)
        assert pr.max_flop_row == rec["max"] and digest(pr.flop_per_row) == rec["flop"]


def test_flop_long_rows_and_empty_rows(P, oracle):
    """Rows spanning many merge-path tiles (carry chains) and long runs of
    empty rows (tiles with no nonzeros)."""
    rows = [list(range(0, 20000, 2)), [], [], list(range(5)), [7] * 0, list(range(30000))]
    rows += [[] for _ in range(5000)] + [[1, 2, 3]] + [list(range(i % 97)) for i in range(3000)]
    a = csr(len(rows), 30000, rows)
    b = gen.uniform_len(30000, 4000, 0, 40, 11)
    P.load(a, b)
    pr = P.compute_flop()
    f, F, mx = oracle.compute_flop(a, b)
    assert (pr.flop_per_row == f).all() and pr.total_flop == F and pr.max_flop_row == mx


def test_flop_tiles_owning_over_65535_rows(P, oracle):
    """Tiles owning more than 2^16 rows (long runs of empty rows between
    short ones): the row a start position belongs to is far from the tile's
    first row."""
    rng = np.random.default_rng(7)
    m = 300_000
    rows = [[] for _ in range(m)]
    for r in sorted(rng.choice(m, 900, replace=False)):
        rows[int(r)] = sorted(int(c) for c in rng.choice(5000, int(rng.integers(1, 6)), replace=False))
    rows[0] = list(range(3000))  # the first tile: rows 0.. plus the sparse run
    rows[m - 1] = list(range(4000, 4100))
    a = csr(m, 5000, rows)
    b = gen.uniform_len(5000, 5000, 0, 30, 12)
    P.load(a, b)
    pr = P.compute_flop()
    f, F, mx = oracle.compute_flop(a, b)
    assert (pr.flop_per_row == f).all() and pr.total_flop == F and pr.max_flop_row == mx


def _long_b(k, n, seed, long_rows=(3, 7), long_len=70000):
    """B with short random rows plus rows of >= 65535 entries (the uint16
    degree escape)."""
    rng = np.random.default_rng(seed)
    lens = rng.integers(0, 9, size=k)
    for r in long_rows:
        lens[r] = long_len
    rpt = np.zeros(k + 1, np.int64)
    np.cumsum(lens, out=rpt[1:])
    col = np.empty(int(rpt[-1]), np.int32)
    for r in range(k):
        if lens[r]:
            col[rpt[r]:rpt[r + 1]] = np.sort(rng.choice(n, int(lens[r]), replace=False))
    return spnnz.CsrMatrix(k, n, rpt, col)


# the FLOP-pass kernels: (row blocks?, shared degree table?, row streams?)
FLOP_KERNELS = {"tiles-smem": ("0", "1", "1"), "tiles-global": ("0", "0", "1"), "rs-smem": ("1", "1", "1"),
                "rb-smem": ("1", "1", "0"), "rb-global": ("1", "0", "1")}


def _flop_kernel_env(monkeypatch, kernel):
    rb, smem, rs = FLOP_KERNELS[kernel]
    monkeypatch.setenv("SPNNZ_FLOP_RB", rb)
    monkeypatch.setenv("SPNNZ_FLOP_SMEM", smem)
    monkeypatch.setenv("SPNNZ_FLOP_RS", rs)


# largest K whose degree table fits beside the row-block staging (74496),
# beside the tile groups (81280) and beside the row streams' scratch (99328), and one
# more of each
@pytest.mark.parametrize("k", [74496, 74497, 81280, 81281, 99328, 99329])
@pytest.mark.parametrize("kernel", list(FLOP_KERNELS))
def test_flop_degree_table_threshold(oracle, monkeypatch, k, kernel):
    """The shared-memory degree tables (row streams, persistent row-block and
    tile-group blocks) on both sides of their size limits, and the
    global-memory kernels, incl. B rows past the uint16 escape and A rows
    spanning tiles / blocks / a warp's whole row range."""
    _flop_kernel_env(monkeypatch, kernel)
    rng = np.random.default_rng(k)
    m = 4000
    rows = [sorted(int(c) for c in rng.choice(k, int(rng.integers(0, 60)), replace=False)) for _ in range(m)]
    rows[5] = list(range(0, k, 7))  # ~11.7 K entries: several tiles
    rows[6] = [3, 7, 9]  # the escape rows
    rows[100:400] = [[] for _ in range(300)]
    a = csr(m, k, rows)
    b = _long_b(k, 100000, k)
    P = Predictor(0)
    P.load(a, b)
    pr = P.compute_flop()
    f, F, mx = oracle.compute_flop(a, b)
    assert (pr.flop_per_row == f).all() and pr.total_flop == F and pr.max_flop_row == mx
    P.close()


@pytest.mark.parametrize("rows_mode", ["1", "0"])
@pytest.mark.parametrize("kernel", list(FLOP_KERNELS))
@pytest.mark.parametrize("shape", ["stencil", "random", "long+empty"])
def test_flop_row_mode(oracle, monkeypatch, rows_mode, kernel, shape):
    """Every FLOP-pass kernel (tiles / row blocks, shared / global degree
    table) with row-per-thread tiles (banded A) forced on and off, on a
    stencil (where load() picks them) and on shapes it would not pick
    (a 10 K-entry row, empty runs, rows longer than a row block's staging):
    per-row FLOP, F and max identical to the oracle, plain and fused."""
    monkeypatch.setenv("SPNNZ_FLOP_ROWS", rows_mode)
    _flop_kernel_env(monkeypatch, kernel)
    if shape == "stencil":
        a = gen.stencil27(40, 30, 20)
        b = a
    elif shape == "random":
        a = gen.uniform_len(60000, 50000, 0, 40, 3)
        b = gen.uniform_len(50000, 30000, 0, 20, 4)
    else:
        rows = [list(range(0, 30000, 3)), []] + [list(range(i % 50)) for i in range(20000)]
        rows += [[] for _ in range(7000)] + [list(range(5000))] + [[i % 29999, 29999] for i in range(5000)]
        a = csr(len(rows), 30000, rows)
        b = gen.uniform_len(30000, 8000, 0, 30, 5)
    P = Predictor(0)
    P.load(a, None if b is a else b)
    pr = P.compute_flop()
    f, F, mx = oracle.compute_flop(a, b)
    assert (pr.flop_per_row == f).all() and pr.total_flop == F and pr.max_flop_row == mx
    # the fused predictor's emit path runs inside the same tile code
    monkeypatch.setenv("SPNNZ_FUSED_PREDICT", "1")
    rep = P.run_prediction(9, SamplePolicy(0.05, -1))
    orep, of, oceil, oreal = oracle.run_prediction(a, b, 9, 0.05, -1)
    assert np.array_equal(rep.predicted_row_nnz_ceil, oceil) and rep.z2_star == orep.z2_star
    P.close()


# -------------------------------------------------------------- sampler
def test_sampler_matches_reference(P, golden):
    for rec in golden["refkat"]["plans"]:
        plan = spnnz.make_sample_plan(rec["m"], rec["seed"], SamplePolicy(rec["fraction"], rec["cap"]))
        assert plan.sample_num == rec["n"] and plan.p == rec["p"]
        assert plan.sample_rows[:8].tolist() == rec["head"] and int(plan.sample_rows[-1]) == rec["last"]
        assert digest(plan.sample_rows) == rec["digest"]
    with pytest.raises(ValueError):
        spnnz.make_sample_plan(0, 1)


def test_sampler_large_vs_oracle(P, oracle):
    for m, seed, frac in [(2**31 - 1, 5, 1e-4), (12345678, 2**63 + 11, 0.01), (3, 0, 1.0)]:
        plan = spnnz.make_sample_plan(m, seed, SamplePolicy(frac, UNCAPPED))
        rows, n, p = oracle.make_sample_plan(m, seed, frac, UNCAPPED)
        assert plan.sample_num == n and plan.p == p and (plan.sample_rows == rows).all()


# -------------------------------------------------------------- symbolic
def test_symbolic_known_answers(P):
    u = upper_2x2()
    prof, ex = gpu_exact(P, u, u)
    assert ex.nnz_per_row.tolist() == [2, 1] and ex.total_nnz == 3  # test_symbolic.cpp:55-61
    a, b = csr(1, 2, [[0, 1]]), csr(2, 2, [[0, 1], [1]])
    assert gpu_exact(P, a, b)[1].nnz_per_row.tolist() == [2]  # :37-43
    a0 = csr(1, 2, [[]])
    assert gpu_exact(P, a0, identity(2))[1].nnz_per_row.tolist() == [0]  # :45-53
    P.load(u, u)
    P.compute_flop()
    assert P.sampled_symbolic([]).total_nnz == 0  # :135-149
    assert P.sampled_symbolic([0]).total_nnz == 2
    r = P.sampled_symbolic([0, 0, 1])
    assert r.total_nnz == 5 and r.nnz_per_row.tolist() == [2, 2, 1]
    with pytest.raises(ValueError):
        P.sampled_symbolic([2])
    with pytest.raises(ValueError):
        P.sampled_symbolic([-1])


def test_symbolic_profile_mismatch_rejected():
    # test_symbolic.cpp:157-163
    eye3, eye4 = identity(3), identity(4)
    prof3 = spnnz.compute_flop(eye3, eye3)
    with pytest.raises(ValueError):
        spnnz.exact_symbolic(eye4, eye4, prof3)
    with pytest.raises(ValueError):
        spnnz.exact_symbolic(eye3, eye4, prof3)


def test_symbolic_trials_vs_reference(P, golden):
    # test_symbolic.cpp:63-77 (100 trials, seed 31337)
    rng = gen.SplitMix64(31337)
    for rec in golden["trials"]["symbolic_dense_oracle"]["trials"]:
        m, k, n = 1 + rng.next_below(80), 1 + rng.next_below(80), 1 + rng.next_below(80)
        d = 0.01 + 0.25 * rng.next_double()
        a = gen.random_pattern(m, k, d, rng)
        b = gen.random_pattern(k, n, d, rng)
        prof, ex = gpu_exact(P, a, b)
        assert (ex.nnz_per_row == dense_bool_multiply_row_nnz(a, b)).all()
        assert ex.total_nnz == rec["Z"] and digest(ex.nnz_per_row) == rec["nnz"]


def test_acceptance_oracle_trials(P, golden):
    # acceptance.cpp:147-169: 1000 trials up to 200x200x200, zero mismatches
    rng = gen.SplitMix64(42424242)
    mism = 0
    for rec in golden["trials"]["acceptance_oracle"]["trials"]:
        m, k, n = 1 + rng.next_below(200), 1 + rng.next_below(200), 1 + rng.next_below(200)
        da, db = 0.002 + 0.25 * rng.next_double(), 0.002 + 0.25 * rng.next_double()
        a = gen.random_pattern(m, k, da, rng)
        b = gen.random_pattern(k, n, db, rng)
        prof, ex = gpu_exact(P, a, b)
        mism += (digest(ex.nnz_per_row) != rec["nnz"] or ex.total_nnz != rec["Z"]
                 or digest(prof.flop_per_row) != rec["flop"])
    assert mism == 0


def tier_matrix(n_rows, n_cols, lens, b_lens, seed):
    """A with the given row lengths, B with the given lengths, uniform cols."""
    rng = np.random.default_rng(seed)
    rows_a = [np.sort(rng.choice(n_cols, size=min(L, n_cols), replace=False)).tolist() for L in lens]
    a = csr(n_rows, n_cols, rows_a)
    rows_b = [np.sort(rng.choice(n_cols, size=min(L, n_cols), replace=False)).tolist() for L in b_lens]
    b = csr(n_cols, n_cols, rows_b)
    return a, b


# heavy-row algorithms (heavy.cu): the default sort-agnostic bucket paths and
# the opt-in sorted-B interval path
# "multipass": the opt-in multipass hash tier (SPNNZ_MP_MAX) takes the rows
# up to 98304 products, the default heavy path the heavier ones
HEAVY_PATHS = ["default", "intervals", "multipass"]


def heavy_path(monkeypatch, path):
    if path == "intervals":
        monkeypatch.setenv("SPNNZ_HEAVY_INTERVALS", "1")
    if path == "multipass":
        monkeypatch.setenv("SPNNZ_MP_MAX", "98304")


@pytest.mark.parametrize("path", HEAVY_PATHS)
@pytest.mark.parametrize("ncols", [3000, 1 << 20, 1 << 24, 1 << 28])
def test_every_bin_vs_oracle(oracle, ncols, path, monkeypatch):
    """Rows whose FLOP lands in every bin (<=32, <=512, <=2048, <=8192,
    <=32768, heavy) including duplicates-heavy rows, for small and large B.cols
    (one range, unit-sorted ranges, > 256 ranges), on both heavy paths."""
    heavy_path(monkeypatch, path)
    P = Predictor(0)
    rng = np.random.default_rng(ncols)
    lens = [0, 1, 2, 5, 10, 40, 100, 200, 300, 700, 1500, 2500] + list(rng.integers(0, 200, 200))
    b_lens = [1, 2, 3, 1, 2, 3, 1, 2, 3, 4] + list(rng.integers(0, 60, 2988)) + [2000, 2999]
    nc = 3000
    a, b = tier_matrix(len(lens), nc, lens, b_lens, 1)
    # rows whose products stay <= 32 (bin 1): entries pointing at B rows 0-9
    extra = [[0], [1, 2], [3, 4, 5], list(range(10))]
    a = csr(a.rows + len(extra), nc, [a.col[a.rpt[i]:a.rpt[i + 1]].tolist() for i in range(a.rows)] + extra)
    # widen B's column space so the bitmap tier sees ncols bits
    b = csr(b.rows, ncols, [list((np.array(b.col[b.rpt[i]:b.rpt[i + 1]]) * (ncols // nc)).tolist())
                           for i in range(b.rows)])
    a = csr(a.rows, b.rows, [a.col[a.rpt[i]:a.rpt[i + 1]].tolist() for i in range(a.rows)])
    prof, ex = gpu_exact(P, a, b)
    f, F, mx = oracle.compute_flop(a, b)
    nnz, Z = oracle.exact_symbolic(a, b, f, mx)
    assert (prof.flop_per_row == f).all()
    bins = np.digitize(f, [1, 33, 513, 2049, 8193, 32769])
    assert set(bins.tolist()) >= {0, 1, 2, 3, 4, 5, 6}, "matrix must exercise every bin"
    assert (ex.nnz_per_row == nnz).all() and ex.total_nnz == Z
    rows = np.arange(a.rows, dtype=np.int32)[::-1].copy()
    s = P.sampled_symbolic(rows)
    assert (s.nnz_per_row == nnz[rows]).all() and s.total_nnz == Z
    P.close()


@pytest.mark.parametrize("path", HEAVY_PATHS)
@pytest.mark.parametrize("ncols", [1 << 20, 1 << 28])
def test_heavy_skewed_intervals(oracle, ncols, path, monkeypatch):
    """Heavy rows whose products all fall in the first column interval: on a
    2^28-column B the interval is wider than the bitmap, so the hash runs in
    several key-hash passes; on 2^20 columns one bitmap interval takes all."""
    rng = np.random.default_rng(7)
    nb = 5000
    b_rows = [np.sort(rng.choice(ncols >> 7, size=int(rng.integers(10, 60)), replace=False)).tolist()
              for _ in range(nb)]
    b = csr(nb, ncols, b_rows)
    a_rows = [np.sort(rng.choice(nb, size=L, replace=False)).tolist() for L in (3000, 4000, 2500, 50)]
    a = csr(len(a_rows), nb, a_rows)
    heavy_path(monkeypatch, path)
    q = Predictor(0)
    q.load(a, b)
    prof = q.compute_flop()
    ex = q.exact_symbolic()
    f, F, mx = oracle.compute_flop(a, b)
    nnz, Z = oracle.exact_symbolic(a, b, f, mx)
    assert (prof.flop_per_row == f).all() and f[:3].min() > 3 * 24576
    assert (ex.nnz_per_row == nnz).all() and ex.total_nnz == Z
    q.close()


@pytest.mark.parametrize("path", HEAVY_PATHS)
def test_unsorted_b_rows(oracle, path, monkeypatch):
    """B rows in arbitrary order (with the interval path requested, the
    sortedness check at load must route the heavy rows to the sort-agnostic
    path): counts still exact."""
    heavy_path(monkeypatch, path)
    rng = np.random.default_rng(11)
    lens = [3000, 2000, 100, 5, 2500]
    a, b = tier_matrix(len(lens), 4000, lens, list(rng.integers(5, 40, 4000)), 9)
    cols = [np.array(b.col[b.rpt[i]:b.rpt[i + 1]]) for i in range(b.rows)]
    for c in cols:
        rng.shuffle(c)
    wide = 1 << 24
    b = csr(b.rows, wide, [(c * (wide // 4000)).tolist() for c in cols])
    q = Predictor(0)
    q.load(a, b)
    q.compute_flop()
    ex = q.exact_symbolic()
    f, F, mx = oracle.compute_flop(a, b)
    nnz, Z = oracle.exact_symbolic(a, b, f, mx)
    assert f.max() > 32768
    assert (ex.nnz_per_row == nnz).all() and ex.total_nnz == Z
    q.close()


@pytest.mark.parametrize("path", HEAVY_PATHS)
def test_heavy_batching(oracle, monkeypatch, path):
    """Heavy rows split over several batches (budget forced down to 100 K
    products): the batch loop, and the merge-bitmap pool returning to zero
    after each use, must keep the counts exact."""
    monkeypatch.setenv("SPNNZ_HEAVY_BATCH_PRODUCTS", "100000")
    heavy_path(monkeypatch, path)
    q = Predictor(0)
    rng = np.random.default_rng(3)
    lens = [3000, 2500, 2800, 2900, 2700, 10, 3000]
    a, b = tier_matrix(len(lens), 4000, lens, list(rng.integers(5, 40, 4000)), 5)
    q.load(a, b)
    q.compute_flop()
    ex = q.exact_symbolic()
    f, F, mx = oracle.compute_flop(a, b)
    nnz, Z = oracle.exact_symbolic(a, b, f, mx)
    assert (f[[0, 1, 2, 3, 4, 6]] > 32768).all()
    assert (ex.nnz_per_row == nnz).all()
    ex2 = q.exact_symbolic()  # pool must be clean again
    assert (ex2.nnz_per_row == nnz).all()
    q.close()


# ------------------------------------------------------------ predictor
def test_predict_views(P):
    prof = spnnz.FlopProfile(np.array([3, 1, 0], np.int64), 4, 3)  # test_predict.cpp:90-112
    assert spnnz.predict_row_structure(prof, 1.0).tolist() == [3.0, 1.0, 0.0]
    r = spnnz.predict_row_structure(prof, 4.0 / 3.0)
    assert r[0] == 3 / (4.0 / 3.0) and r[1] == 1 / (4.0 / 3.0) and r[2] == 0.0
    assert spnnz.predict_row_structure_ceil(prof, 4.0 / 3.0).tolist() == [3, 1, 0]
    with pytest.raises(ValueError):
        spnnz.predict_row_structure(prof, 0.0)
    with pytest.raises(ValueError):
        spnnz.predict_row_structure_ceil(prof, -1.0)


def test_predict_views_bitwise_vs_oracle(oracle):
    rng = np.random.default_rng(1)
    f = np.concatenate([rng.integers(0, 2**40, 5001), [0, 1, 2**53 + 1, 2**62]]).astype(np.int64)
    prof = spnnz.FlopProfile(f, int(f.sum() % 2**62), int(f.max()))
    for cr in (1.0, 1.0000000001, 4.0 / 3.0, 2.15, 5.844, 1e-3, 1e9):
        assert (spnnz.predict_row_structure_ceil(prof, cr) == oracle.predict_row_structure_ceil(f, cr)).all()
        assert (spnnz.predict_row_structure(prof, cr) == oracle.predict_row_structure(f, cr)).all()


def test_predict_division_random_ratios(oracle):
    """Per-row views bit-identical to the CPU division for random ratios,
    including quotients that are exact integers and near-halfway cases
    (flop = k * cr rounded).  (The fused predictor's certified reciprocal
    path, FastDiv, is checked on whole configs by test_config_fused_predictor.)"""
    rng = np.random.default_rng(2)
    f = np.concatenate([rng.integers(1, 2**31, 20000), rng.integers(2**31, 2**62, 20000),
                        np.arange(1, 5000)]).astype(np.int64)
    crs = list(rng.uniform(1.0, 64.0, 24)) + list(1.0 + rng.uniform(0, 1e-9, 4)) + [3.0, 7.0, 1.5, 1.25]
    for cr in crs:
        near = np.unique(np.round(np.arange(1, 3000) * cr)).astype(np.int64)  # quotients near integers
        g = np.concatenate([f, near])
        prof = spnnz.FlopProfile(g, int(g.sum() % 2**62), int(g.max()))
        assert (spnnz.predict_row_structure(prof, cr) == oracle.predict_row_structure(g, cr)).all(), cr
        assert (spnnz.predict_row_structure_ceil(prof, cr) == oracle.predict_row_structure_ceil(g, cr)).all(), cr


def test_identity_predicts_exactly():
    # test_predict.cpp:146-157
    for n in (10, 100, 1000):
        for seed in (1, 7, 99):
            eye = identity(n)
            rep = spnnz.run_prediction(eye, eye, seed)
            assert rep.predicted_cr == 1.0 and rep.z2_star == float(n)
            assert abs(rep.z1_star - n) <= 1e-9 * n


def test_pipeline_vs_reference_runs(golden):
    # test_predict.cpp:184-217 against the reference's own pipeline
    rng = gen.SplitMix64(123)
    for rec in golden["trials"]["predict_pipeline"]["trials"]:
        n = 20 + rng.next_below(150)
        a = gen.random_pattern(n, n, 0.1, rng)
        b = gen.random_pattern(n, n, 0.1, rng)
        seed = rng.next_u64()
        rep = spnnz.run_prediction(a, b, seed)
        ref = rec["report"]
        assert rep.total_flop == ref["total_flop"] and rep.stats.sampled_flop == ref["sampled_flop"]
        assert rep.stats.sampled_nnz == ref["sampled_nnz"] and rep.plan.sample_num == ref["sample_num"]
        assert rep.plan.p == ref["p"] and rep.z1_star == ref["z1_star"] and rep.z2_star == ref["z2_star"]
        assert rep.predicted_cr == ref["predicted_cr"] and rep.stats.sampled_cr == ref["sampled_cr"]
        assert digest(rep.predicted_row_nnz_ceil) == rec["ceil"]
        assert rep.plan.sample_rows.tolist() == rec["rows"]


def test_exhaustive_plan_is_exact():
    # test_predict.cpp:159-182, acceptance.cpp:201-231
    rng = gen.SplitMix64(77)
    for _ in range(10):
        n = 5 + rng.next_below(60)
        a = gen.random_pattern(n, n, 0.15, rng)
        b = gen.random_pattern(n, n, 0.15, rng)
        prof = spnnz.compute_flop(a, b)
        ex = spnnz.exact_symbolic(a, b, prof)
        if ex.total_nnz == 0:
            continue
        rep = spnnz.run_prediction_with_plan(a, b, prof, spnnz.exhaustive_plan(n))
        assert rep.z1_star == ex.total_nnz and rep.z2_star == ex.total_nnz
        e = spnnz.error_report(rep.z1_star, rep.z2_star, rep.stats.sampled_flop, ex.total_nnz,
                               prof.total_flop, rep.plan.p)
        assert (e.eps1, e.eps_f, e.eps2) == (0.0, 0.0, 0.0)


def _golden_csr(rec, key, rows, cols):
    m = rec[key]
    return spnnz.CsrMatrix(rows, cols, np.array(m["rpt"], np.int64), np.array(m["col"], np.int32))


@pytest.mark.parametrize("api", ["python", "capi-device-rows"])
def test_with_plan_hand_built_profiles(golden, api):
    """run_prediction_with_plan on a caller's profile (predict.hpp:202-216):
    zeroed rows count 0, inflated rows change f* / F / the views but not the
    counts, another total_flop moves Z2*, a capacity violation is the
    reference's invalid_argument -- against the reference's own outputs
    (tests/golden/with_plan.json, oracle/_ref)."""
    import torch
    P = Predictor(0)
    for rec in golden["with_plan"]["cases"]:
        a = _golden_csr(rec, "a", rec["m"], rec["k"])
        b = a if rec["same"] else _golden_csr(rec, "b", rec["k"], rec["n"])
        prof = spnnz.FlopProfile(np.array(rec["flop"], np.int64), rec["total"], rec["max"])
        rows = np.array(rec["rows"], np.int32)
        plan = SamplePlan(rows, len(rows), rec["p"], 0)
        if api == "capi-device-rows":
            plan = SamplePlan(torch.tensor(rows, device="cuda"), len(rows), rec["p"], 0)
        P.load(a, None if rec["same"] else b)
        if "error" in rec:
            with pytest.raises(ValueError, match="exceeds capacity"):
                P.run_prediction_with_plan(plan, prof)
            assert rec["error"].startswith("HashAccumulator: tsize")
            continue
        rep = P.run_prediction_with_plan(plan, prof)
        r = rec["report"]
        assert rep.total_flop == r["total_flop"] == rec["total"], rec["kind"]
        assert rep.stats.sampled_flop == r["sampled_flop"], rec["kind"]
        assert rep.stats.sampled_nnz == r["sampled_nnz"], rec["kind"]
        assert rep.stats.sampled_cr == r["sampled_cr"]
        assert rep.z1_star == r["z1_star"] and rep.z2_star == r["z2_star"], rec["kind"]
        assert rep.predicted_cr == r["predicted_cr"]
        assert np.array_equal(rep.predicted_row_nnz, np.array(rec["real"])), rec["kind"]
        assert np.array_equal(rep.predicted_row_nnz_ceil, np.array(rec["ceil"], np.int64)), rec["kind"]
        # the standalone sampled_symbolic on the same profile agrees
        P.set_profile(prof)
        s = P.sampled_symbolic(rows)
        assert s.total_nnz == r["sampled_nnz"]
    P.close()


def test_predict_sampled_equals_reference_task(golden):
    """spnnz_gpu_predict_sampled (the harness's predict task in one call) gives
    run_prediction's scalars for the same seed and policy (the reference's
    run_prediction = compute_flop + make_sample_plan + run_prediction_with_plan),
    on every repeat (cached sizes, graph replay)."""
    for cfg in (1, 4):
        info = gen.CONFIGS[cfg]
        a, b = gen.make_config(cfg)
        P = Predictor(0)
        P.load(a, None if b is a else b)
        pol = SamplePolicy(info["fraction"], UNCAPPED)
        full = P.run_prediction(info["seed"], pol)
        for _ in range(4):
            r = P.predict_sampled(info["seed"], pol)
            assert (r.stats.sampled_flop, r.stats.sampled_nnz, r.z1_star, r.z2_star, r.predicted_cr) == \
                (full.stats.sampled_flop, full.stats.sampled_nnz, full.z1_star, full.z2_star, full.predicted_cr)
            assert np.array_equal(r.plan.sample_rows, full.plan.sample_rows)
        ref = golden["configs"][str(cfg)]["modes"]["uncapped"]["report"]
        assert r.z2_star == ref["z2_star"] and r.stats.sampled_nnz == ref["sampled_nnz"]
        P.close()


def test_with_plan_uses_profile_not_a_flop_pass():
    """The free function hands the caller's profile through: a profile whose
    total differs from the matrices' moves Z2* exactly as the reference's
    expression F*z*/f* says (predict.hpp:120-121)."""
    rng = gen.SplitMix64(91)
    a = gen.random_pattern(200, 200, 0.05, rng)
    prof = spnnz.compute_flop(a, a)
    plan = spnnz.make_sample_plan(a.rows, 5, SamplePolicy(0.1, -1))
    base = spnnz.run_prediction_with_plan(a, a, prof, plan)
    prof2 = spnnz.FlopProfile(prof.flop_per_row.copy(), prof.total_flop * 7 + 3, prof.max_flop_row)
    rep = spnnz.run_prediction_with_plan(a, a, prof2, plan)
    assert rep.total_flop == prof2.total_flop
    f, z = rep.stats.sampled_flop, rep.stats.sampled_nnz
    assert (f, z) == (base.stats.sampled_flop, base.stats.sampled_nnz)
    assert rep.z2_star == float(prof2.total_flop) * float(z) / float(f)


def test_free_function_composition(oracle):
    """collect_sample_stats / estimators over GPU pieces equal run_prediction."""
    rng = gen.SplitMix64(55)
    a = gen.random_pattern(400, 400, 0.05, rng)
    b = gen.random_pattern(400, 400, 0.05, rng)
    prof = spnnz.compute_flop(a, b)
    plan = spnnz.make_sample_plan(a.rows, 42)
    sampled = spnnz.sampled_symbolic(a, b, prof, plan.sample_rows)
    stats = spnnz.collect_sample_stats(prof, plan, sampled)
    pp = spnnz.predict_proposed(stats, prof.total_flop)
    rep = spnnz.run_prediction(a, b, 42)
    assert stats.sampled_flop == rep.stats.sampled_flop and stats.sampled_nnz == rep.stats.sampled_nnz
    assert pp.z2_star == rep.z2_star and pp.predicted_cr == rep.predicted_cr
    assert spnnz.predict_reference(stats, plan) == rep.z1_star
    assert spnnz.sampled_flop(prof, [0, 0]) == 2 * prof.flop_per_row[0]
    ora = oracle.run_prediction(a, b, 42, 0.003, 300)[0]
    assert ora.z2_star == rep.z2_star and ora.sampled_nnz == rep.stats.sampled_nnz


# ---------------------------------------------------------- configs 1-5
def test_config1_full_arrays(P, golden):
    a, b = gen.make_config(1)
    arr, rec = golden["cfg1"], golden["configs"]["1"]
    P.load(a, b)
    prof = P.compute_flop()
    assert (prof.flop_per_row == arr["flop"]).all() and prof.total_flop == rec["F"]
    ex = P.exact_symbolic()
    assert (ex.nnz_per_row == arr["exact_nnz"]).all() and ex.total_nnz == rec["Z"]
    for label, cap in (("uncapped", UNCAPPED), ("cap300", 300)):
        rep = P.run_prediction(1, SamplePolicy(0.01, cap))
        ref = rec["modes"][label]["report"]
        for k in ("total_flop", "sampled_flop", "sampled_nnz", "p", "z1_star", "z2_star", "predicted_cr"):
            got = getattr(rep, k) if hasattr(rep, k) else getattr(rep.stats, k, None)
            if got is None:
                got = getattr(rep.plan, k)
            assert got == ref[k], k
        assert (rep.predicted_row_nnz_ceil == arr[f"ceil_{label}"]).all()
        assert (rep.predicted_row_nnz == arr[f"real_{label}"]).all()
        assert (rep.plan.sample_rows == arr[f"rows_{label}"]).all()
        s = P.sampled_symbolic(rep.plan.sample_rows)
        assert (s.nnz_per_row == arr[f"per_sample_{label}"]).all()


@pytest.mark.parametrize("cfg", [1, 2, 4, 5])
def test_config_fused_predictor(golden, cfg, monkeypatch):
    """SPNNZ_FUSED_PREDICT=1 (CR first, one pass writing flop and
    the prediction): same report, sample rows and per-row views as the
    reference."""
    rec = golden["configs"][str(cfg)]
    info = gen.CONFIGS[cfg]
    a, b = gen.make_config(cfg)
    monkeypatch.setenv("SPNNZ_FUSED_PREDICT", "1")
    q = Predictor(0)
    q.load(a, b)
    m = rec["modes"]["uncapped"]
    rep = q.run_prediction(info["seed"], SamplePolicy(info["fraction"], UNCAPPED))
    ref = m["report"]
    assert rep.total_flop == ref["total_flop"] and rep.stats.sampled_flop == ref["sampled_flop"]
    assert rep.stats.sampled_nnz == ref["sampled_nnz"] and rep.predicted_cr == ref["predicted_cr"]
    assert rep.z1_star == ref["z1_star"] and rep.z2_star == ref["z2_star"]
    if cfg == 1:
        arr = golden["cfg1"]
        assert (rep.predicted_row_nnz_ceil == arr["ceil_uncapped"]).all()
        assert (rep.predicted_row_nnz == arr["real_uncapped"]).all()
    else:
        assert digest(rep.predicted_row_nnz_ceil) == m["ceil"]
        assert digest(rep.predicted_row_nnz) == m["real"]
    prof = q.compute_flop()
    assert prof.total_flop == ref["total_flop"]
    q.close()


@pytest.mark.parametrize("cfg", [2, 5])
def test_config_interval_path_sampled(golden, cfg, monkeypatch):
    """The interval heavy-row path reproduces the reference's sampled NNZ on
    the skewed configs (the default path is checked below)."""
    path = "intervals"
    rec = golden["configs"][str(cfg)]
    info = gen.CONFIGS[cfg]
    a, b = gen.make_config(cfg)
    heavy_path(monkeypatch, path)
    q = Predictor(0)
    q.load(a, b)
    q.compute_flop()
    rep = q.run_prediction(info["seed"], SamplePolicy(info["fraction"], UNCAPPED))
    assert rep.stats.sampled_nnz == rec["modes"]["uncapped"]["report"]["sampled_nnz"]
    q.close()


@pytest.mark.parametrize("cfg", [2, 3, 4, 5])
def test_config_vs_reference_digests(P, golden, cfg):
    if str(cfg) not in golden["configs"]:
        pytest.skip("configs.json lacks this config (make_golden.py --big)")
    rec = golden["configs"][str(cfg)]
    info = gen.CONFIGS[cfg]
    a, b = gen.make_config(cfg)
    assert digest(a.rpt) == rec["input"]["a_rpt"] and digest(a.col) == rec["input"]["a_col"]
    P.load(a, b)
    prof = P.compute_flop()
    assert prof.total_flop == rec["F"] and prof.max_flop_row == rec["max"]
    assert digest(prof.flop_per_row) == rec["flop"]
    for label, cap in (("uncapped", UNCAPPED), ("cap300", 300)):
        m = rec["modes"][label]
        rep = P.run_prediction(info["seed"], SamplePolicy(info["fraction"], cap))
        ref = m["report"]
        assert rep.total_flop == ref["total_flop"]
        assert rep.stats.sampled_flop == ref["sampled_flop"] and rep.stats.sampled_nnz == ref["sampled_nnz"]
        assert rep.plan.sample_num == ref["sample_num"] and rep.plan.p == ref["p"]
        assert rep.predicted_cr == ref["predicted_cr"]
        assert abs(rep.predicted_cr - ref["predicted_cr"]) <= CR_RTOL * ref["predicted_cr"]
        assert rep.z1_star == ref["z1_star"] and rep.z2_star == ref["z2_star"]
        assert digest(rep.plan.sample_rows) == m["rows"]
        assert digest(rep.predicted_row_nnz_ceil) == m["ceil"]
        assert digest(rep.predicted_row_nnz) == m["real"]
        s = P.sampled_symbolic(rep.plan.sample_rows)
        assert s.total_nnz == m["z_star"] and digest(s.nnz_per_row) == m["per_sample"]
    if "Z" in rec:
        # config 5: pinned to the reference's own exact_symbolic (row slices,
        # tests/golden/make_cfg5_exact.py); per-2^20-row digests localise a miss
        ex = P.exact_symbolic()
        if "exact_nnz_blocks" in rec:
            blk = 1 << 20
            got = [digest(ex.nnz_per_row[i:i + blk]) for i in range(0, a.rows, blk)]
            bad = [i for i, (x, y) in enumerate(zip(got, rec["exact_nnz_blocks"])) if x != y]
            assert not bad, f"exact per-row NNZ differs in row blocks {bad}"
        assert ex.total_nnz == rec["Z"] and digest(ex.nnz_per_row) == rec["exact_nnz"]
        for label in rec["modes"]:
            if "errors" in rec["modes"][label]:
                r = rec["modes"][label]["report"]
                e = spnnz.error_report(r["z1_star"], r["z2_star"], r["sampled_flop"], ex.total_nnz,
                                       prof.total_flop, r["p"])
                assert [e.eps1, e.eps_f, e.eps2, e.identity_residual] == rec["modes"][label]["errors"]
        if cfg == 3:
            assert ex.total_nnz == 634 ** 3 and prof.total_flop == 1142 ** 3


def test_config5_exact_properties(P):
    """Config 5 has no CPU exact pass (hours); check size-independent
    properties of the GPU exact pass: nnz <= flop, nnz >= 1 where flop >= 1,
    the sampled pass equals the exact pass at the sampled rows, and the
    sampled CR is >= 1."""
    a, b = gen.make_config(5)
    P.load(a, b)
    prof = P.compute_flop()
    ex = P.exact_symbolic()
    f, z = prof.flop_per_row, ex.nnz_per_row
    assert (z <= f).all() and ((f == 0) | (z >= 1)).all()
    assert ex.total_nnz == int(z.sum())
    rep = P.run_prediction(5, SamplePolicy(0.001, UNCAPPED))
    rows = rep.plan.sample_rows
    assert rep.stats.sampled_nnz == int(z[rows].sum())
    assert rep.stats.sampled_flop == int(f[rows].sum())
    assert rep.predicted_cr >= 1.0
    e = spnnz.error_report(rep.z1_star, rep.z2_star, rep.stats.sampled_flop, ex.total_nnz,
                           prof.total_flop, rep.plan.p)
    assert e.identity_residual <= 1e-9 * max(1.0, abs(e.eps2))
    print(f"cfg5: Z={ex.total_nnz} eps1={e.eps1:+.4%} eps2={e.eps2:+.4%}")


def test_nccl_one_rank_communicator_matches_plain_context():
    """The NCCL path (dlopen of libnccl, ncclCommInitRank, the grouped
    all-reduces on the pipeline stream) with a one-rank communicator gives
    the communicator-free context's results exactly."""
    a, b = gen.make_config(1)
    plain = Predictor(0)
    comm = Predictor(0, 0, 1, Predictor.nccl_unique_id())
    try:
        reps = []
        for P_ in (plain, comm):
            P_.load(a, b)
            rep = P_.run_prediction(1, SamplePolicy(0.05, UNCAPPED))
            ex = P_.exact_symbolic()
            reps.append((rep, ex))
        (r0, e0), (r1, e1) = reps
        assert r1.total_flop == r0.total_flop and r1.max_flop_row == r0.max_flop_row
        assert r1.stats.sampled_flop == r0.stats.sampled_flop
        assert r1.stats.sampled_nnz == r0.stats.sampled_nnz
        assert r1.predicted_cr == r0.predicted_cr and r1.z2_star == r0.z2_star
        assert np.array_equal(r1.predicted_row_nnz_ceil, r0.predicted_row_nnz_ceil)
        assert e1.total_nnz == e0.total_nnz and np.array_equal(e1.nnz_per_row, e0.nnz_per_row)
    finally:
        plain.close()
        comm.close()


def test_detached_shards_combine_to_single_gpu(oracle):
    """world > 1 without NCCL on one GPU: every rank's local pass, combined on
    the host, equals the 1-GPU result (bit-exact), for 2, 3 and 8 shards."""
    a, b = gen.make_config(2)
    single = Predictor(0)
    single.load(a, b)
    ref = single.run_prediction(2, SamplePolicy(0.003, UNCAPPED))
    single.close()
    for world in (2, 3, 8):
        F = fs = zs = 0
        flops, shards = [], []
        for r in range(world):
            q = Predictor(0, r, world)
            q.load(a, b)
            pr = q.compute_flop()
            flops.append(pr.flop_per_row)
            F += pr.total_flop
            mine = ref.plan.sample_rows[(ref.plan.sample_rows >= q.row_lo) & (ref.plan.sample_rows < q.row_hi)]
            fs += q.sampled_flop(mine)
            zs += q.sampled_symbolic(mine).total_nnz
            shards.append(q)
        assert F == ref.total_flop and fs == ref.stats.sampled_flop and zs == ref.stats.sampled_nnz
        assert (np.concatenate(flops) == oracle.compute_flop(a, b)[0]).all()
        cr = spnnz.predict_proposed(spnnz.SampleStats(fs, zs), F).predicted_cr
        assert cr == ref.predicted_cr
        ceil = np.concatenate([q.predict_row_structure_ceil(cr) for q in shards])
        assert (ceil == ref.predicted_row_nnz_ceil).all()
        for q in shards:
            q.close()


@pytest.mark.parametrize("escapes", [False, True])
def test_detached_rect_shards_row_streams(oracle, escapes):
    """A != B row shards whose entries start at unaligned offsets (the row
    streams' 16-byte chunk alignment and the shard allocation's bounds), B's
    degree table in shared memory, with and without uint16 escapes: the
    shards' per-row FLOP concatenates to the oracle's."""
    a = gen.uniform_len(50001, 3000, 0, 33, 11)
    b = _long_b(3000, 100000, 12) if escapes else gen.uniform_len(3000, 70000, 0, 25, 12)
    f = oracle.compute_flop(a, b)[0]
    for world in (3, 7):
        parts = []
        for r in range(world):
            q = Predictor(0, r, world)
            q.load(a, b)
            parts.append(q.compute_flop().flop_per_row)
            q.close()
        assert (np.concatenate(parts) == f).all()


def test_detached_pipeline_shards_sum_to_single_gpu():
    """run_prediction on detached shards (world > 1, no NCCL): for C = A*A the
    sampled rows are split by list position (balanced heavy rows), and the
    per-rank F, f*, z* still add up to the single-GPU totals."""
    a, b = gen.make_config(2)
    single = Predictor(0)
    single.load(a, b)
    ref = single.run_prediction(2, SamplePolicy(0.003, UNCAPPED))
    single.close()
    for world in (2, 4, 8):
        F = fs = zs = 0
        for r in range(world):
            q = Predictor(0, r, world)
            q.load(a, b)
            rep = q.run_prediction(2, SamplePolicy(0.003, UNCAPPED))
            F += rep.total_flop
            fs += rep.stats.sampled_flop
            zs += rep.stats.sampled_nnz
            q.close()
        assert (F, fs, zs) == (ref.total_flop, ref.stats.sampled_flop, ref.stats.sampled_nnz)


def test_detached_shards_sampled_flop_chunk_edges(oracle):
    """The balanced split derives each rank's sampled-row FLOP directly (rows
    cut into 128-entry chunks, one warp each): row lengths on and around the
    chunk edges, empty rows and repeated draws, summed over 3 ranks, equal the
    oracle's sampled FLOP."""
    rng = np.random.default_rng(77)
    n = 6000
    lens = np.tile([0, 1, 127, 128, 129, 255, 256, 257, 1000, 3000], n // 10)
    rows = [np.sort(rng.choice(n, size=L, replace=False)).astype(np.int32) for L in lens]
    a = csr(n, n, rows)
    flop, F, _ = oracle.compute_flop(a, a)
    for fraction in (0.05, 1.0):
        plan = spnnz.make_sample_plan(n, 9, SamplePolicy(fraction, UNCAPPED))
        want = int(flop[plan.sample_rows.astype(np.int64)].sum())
        fs = 0
        for r in range(3):
            q = Predictor(0, r, 3)
            q.load(a)
            rep = q.run_prediction(9, SamplePolicy(fraction, UNCAPPED))
            fs += rep.stats.sampled_flop
            q.close()
        assert fs == want


def test_repeat_runs_deterministic(P):
    a, b = gen.make_config(4)
    P.load(a, b)
    r1 = P.run_prediction(4, SamplePolicy(0.005, UNCAPPED))
    r2 = P.run_prediction(4, SamplePolicy(0.005, UNCAPPED))
    assert r1.stats.sampled_nnz == r2.stats.sampled_nnz and r1.z2_star == r2.z2_star
    assert (r1.predicted_row_nnz_ceil == r2.predicted_row_nnz_ceil).all()


def _rep_tuple(r):
    return (r.total_flop, r.stats.sampled_flop, r.stats.sampled_nnz, r.predicted_cr, r.z1_star, r.z2_star)


@pytest.mark.parametrize("small", ["1", "0"])
@pytest.mark.parametrize("maxlen", [13, 40])
def test_small_fused_path_vs_oracle(oracle, small, maxlen, monkeypatch):
    """The fused small-problem kernel (every row's FLOP <= 512, the context's
    own profile: taken from the second call on, then captured into a graph and
    replayed) against the tiered path and the oracle: z*, f*, the drawn rows,
    the ceil view; an exact pass between two replays (which rewrites the host
    mirror of the bin counts) must not trip the advance-size check."""
    monkeypatch.setenv("SPNNZ_SYM_SMALL", small)
    monkeypatch.setenv("SPNNZ_STRICT_SIZES", "1")
    a = gen.uniform_len(30000, 30000, 0, maxlen, 5)
    orep, of, oceil, _ = oracle.run_prediction(a, a, 7, 0.05, -1)
    # maxlen 13: every row in bin 2 (one kernel); 40: rows of bin 3 too (two)
    assert of.max() <= 512 if maxlen == 13 else 512 < of.max() <= 2048
    P = Predictor(0)
    P.load(a)
    for k in range(4):
        rep = P.run_prediction(7, SamplePolicy(0.05, UNCAPPED))
        assert rep.stats.sampled_nnz == orep.sampled_nnz and rep.stats.sampled_flop == orep.sampled_flop, k
        assert rep.z2_star == orep.z2_star and rep.total_flop == orep.total_flop
        assert np.array_equal(rep.predicted_row_nnz_ceil, oceil)
        plan = oracle.make_sample_plan(a.rows, 7, 0.05, -1)
        assert np.array_equal(rep.plan.sample_rows, plan[0] if isinstance(plan, tuple) else plan)
        if k == 2:
            P.exact_symbolic()
    for k in range(3):
        ps = P.predict_sampled(11, SamplePolicy(0.05, UNCAPPED))
        o2 = oracle.run_prediction(a, a, 11, 0.05, -1, want_rows=False)[0]
        assert ps.stats.sampled_nnz == o2.sampled_nnz and ps.z2_star == o2.z2_star
    P.close()


@pytest.mark.parametrize("cfg", [1, 2, 3, 4])
def test_repeat_calls_graph_replay_and_cached_heavy_sizes(golden, cfg, monkeypatch):
    """Repeated calls take the sync-free path: heavy-row sizes known in advance
    (no row can be heavy, or the same draw ran before: config 2 has heavy
    rows), captured into a CUDA graph on the second use and replayed after --
    every call's outputs equal the eager path's and the reference's; changing
    the seed, the outputs or the profile drops / re-keys the graph."""
    import torch
    monkeypatch.setenv("SPNNZ_STRICT_SIZES", "1")  # a wrong advance size is an error here
    rec = golden["configs"][str(cfg)] if str(cfg) in golden["configs"] else None
    info = gen.CONFIGS[cfg]
    a, b = gen.make_config(cfg)
    P = Predictor(0)
    P.load(a, None if b is a else b)
    pol = SamplePolicy(info["fraction"], UNCAPPED)
    m = P.local_rows
    out = torch.empty(m, dtype=torch.int64, device="cuda")
    reps, ceils = [], []
    for i in range(5):  # eager (sync), eager (known sizes), capture, replay, replay
        r = P.run_prediction(info["seed"], pol, ceil_out=out, residency=spnnz.DEVICE,
                             want_real=False, want_samples=False)
        reps.append(_rep_tuple(r))
        ceils.append(out.cpu().numpy().copy())
        out.fill_(-7)
    assert all(x == reps[0] for x in reps)
    assert all(np.array_equal(x, ceils[0]) for x in ceils)
    if rec:
        ref = rec["modes"]["uncapped"]
        assert reps[0][2] == ref["z_star"] and digest(ceils[0]) == ref["ceil"]
    # another seed: a new key (its own eager run first)
    r2 = P.run_prediction(info["seed"] + 1, pol, ceil_out=out, residency=1, want_real=False, want_samples=False)
    monkeypatch.setenv("SPNNZ_GRAPH", "0")
    r2e = P.run_prediction(info["seed"] + 1, pol, ceil_out=out, residency=1, want_real=False, want_samples=False)
    assert _rep_tuple(r2) == _rep_tuple(r2e)
    monkeypatch.delenv("SPNNZ_GRAPH")
    # the profile path (run_prediction_with_plan on the resident profile), repeated
    plan = P.make_sample_plan(a.rows, 3, pol)
    w = [_rep_tuple(P.run_prediction_with_plan(plan)) for _ in range(4)]
    assert all(x == w[0] for x in w)
    P.close()


def test_device_residency_matches_host(P):
    import torch
    a, b = gen.make_config(3)
    P.load(a, b)
    host = P.run_prediction(3, SamplePolicy(0.001, UNCAPPED))
    dev = torch.empty(a.rows, dtype=torch.int64, device="cuda")
    rep = P.run_prediction(3, SamplePolicy(0.001, UNCAPPED), ceil_out=dev, want_real=False,
                           want_samples=False)
    assert rep.z2_star == host.z2_star
    assert (dev.cpu().numpy() == host.predicted_row_nnz_ceil).all()
    # device-resident inputs
    ta = type("M", (), dict(rows=a.rows, cols=a.cols, rpt=torch.from_numpy(a.rpt).cuda(),
                            col=torch.from_numpy(a.col).cuda()))()
    P.load(ta, None)
    rep2 = P.run_prediction(3, SamplePolicy(0.001, UNCAPPED))
    assert rep2.z2_star == host.z2_star and (rep2.predicted_row_nnz_ceil == host.predicted_row_nnz_ceil).all()


def test_device_inputs_produced_on_a_side_stream():
    """Device inputs an asynchronous kernel writes on a torch side stream are
    read after it (spnnz_gpu_set_input_stream, set from torch's current
    stream): sample rows, a profile and the matrices themselves, each written
    by a queued kernel right before the call."""
    import torch
    a, b = gen.make_config(4)
    P = Predictor(0)
    P.load(a, b)
    prof = P.compute_flop()
    rows_h = P.make_sample_plan(a.rows, 4, SamplePolicy(0.005, UNCAPPED)).sample_rows
    ref = P.sampled_symbolic(rows_h)
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        torch.cuda._sleep(20_000_000)  # keep the side stream busy
        rows_d = torch.from_numpy(rows_h.astype(np.int64)).cuda(non_blocking=True).to(torch.int32)
        got = P.sampled_symbolic(rows_d)
        assert got.total_nnz == ref.total_nnz
        assert np.array_equal(got.nnz_per_row.cpu().numpy(), ref.nnz_per_row)
        torch.cuda._sleep(20_000_000)
        flop_d = torch.from_numpy(prof.flop_per_row).cuda(non_blocking=True)
        P.set_profile(spnnz.FlopProfile(flop_d, prof.total_flop, prof.max_flop_row))
        assert P.sampled_flop(rows_h) == int(prof.flop_per_row[rows_h.astype(np.int64)].sum())
        torch.cuda._sleep(20_000_000)
        ta = type("M", (), dict(rows=a.rows, cols=a.cols, rpt=torch.from_numpy(a.rpt).cuda(non_blocking=True),
                                col=torch.from_numpy(a.col).cuda(non_blocking=True)))()
        tb = type("M", (), dict(rows=b.rows, cols=b.cols, rpt=torch.from_numpy(b.rpt).cuda(non_blocking=True),
                                col=torch.from_numpy(b.col).cuda(non_blocking=True)))()
        P.load(ta, tb)
        assert P.compute_flop().total_flop == prof.total_flop
    P.close()


def test_cpp_dropin_header():
    """include/spnnz_gpu/spnnz_gpu.hpp: the reference's known answers through
    the C++ mirror (tests/cpp/test_dropin.cpp)."""
    import subprocess
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    exe = os.path.join(root, "build", "test_dropin")
    if not os.path.exists(exe):
        subprocess.run(["make", "-C", root, "build/test_dropin"], check=True, capture_output=True)
    r = subprocess.run([exe], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr


def test_guard_bands_sanitize_cases():
    """compute-sanitizer is closed on the GPU pool, so out-of-bounds writes are
    caught with guard bands instead: every library buffer is followed by 256
    bytes of a known pattern (SPNNZ_GUARD=1), and tools/sanitize_cases.py --
    every kernel family on small inputs, each result checked against the CPU
    oracle -- must leave every band intact."""
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, SPNNZ_GUARD="1")
    r = subprocess.run([sys.executable, os.path.join(root, "tools", "sanitize_cases.py")], env=env,
                       capture_output=True, text=True, timeout=900)
    assert r.returncode == 0 and "guard bands intact" in r.stdout, r.stdout[-2000:] + r.stderr[-2000:]


def test_cpp_dropin_reference_types():
    """The reference's own spnnz::CsrMatrix / FlopProfile / SamplePlan into
    spnnz::gpu::*, every output compared with the unmodified reference function
    (tests/cpp/test_dropin_ref.cpp; built where /root/reference exists)."""
    import subprocess
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    exe = os.path.join(root, "build", "test_dropin_ref")
    if not os.path.exists(exe):
        pytest.skip("build/test_dropin_ref not built (needs the reference headers at build time)")
    r = subprocess.run([exe], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0 and "all checks passed" in r.stdout, r.stdout + r.stderr


# ------------------------------------------------------------------ fuzzing
def _fuzz_matrix(rng, rows, cols, kind):
    """Random CSR with sorted distinct columns: uniform, skewed (a few hub
    rows with thousands of entries) or banded."""
    out = []
    for i in range(rows):
        if kind == "skewed":
            k = int(rng.integers(2000, 6000)) if rng.random() < 0.01 else int(rng.integers(0, 12))
        elif kind == "banded":
            k = int(rng.integers(1, 30))
        else:
            k = int(rng.integers(0, 40))
        k = min(k, cols)
        if kind == "banded":
            c0 = max(0, min(cols - k, i * cols // max(rows, 1) - k // 2))
            out.append(np.arange(c0, c0 + k))
        else:
            out.append(np.sort(rng.choice(cols, size=k, replace=False)))
    return csr(rows, cols, [r.tolist() for r in out])


@pytest.mark.parametrize("case", range(36))
def test_fuzz_pipeline_vs_oracle(oracle, case, monkeypatch):
    """Random shapes (square and rectangular, narrow to 2^26 columns),
    uniform / skewed / banded rows, random heavy-path and pipeline options:
    per-row FLOP, exact NNZ, sampled totals and the ceil view equal the
    oracle's."""
    rng = np.random.default_rng(1000 + case)
    kinds = ["uniform", "skewed", "banded"]
    m = int(rng.integers(200, 3000))
    k = int(rng.integers(200, 3000))
    n = int(rng.choice([64, 3000, 1 << 16, 1 << 21, 1 << 26]))
    a = _fuzz_matrix(rng, m, k, kinds[case % 3])
    b = _fuzz_matrix(rng, k, min(n, 1 << 16) if kinds[(case + 1) % 3] == "banded" else n, kinds[(case + 1) % 3])
    b = csr(b.rows, n, [b.col[b.rpt[i]:b.rpt[i + 1]].tolist() for i in range(b.rows)])
    if case % 4 == 1:
        monkeypatch.setenv("SPNNZ_HEAVY_INTERVALS", "1")
    if case % 4 == 2:
        monkeypatch.setenv("SPNNZ_FUSED_PREDICT", "1")
    if case % 4 == 3:
        monkeypatch.setenv("SPNNZ_HEAVY_BATCH_PRODUCTS", "50000")
    if case % 3 == 0:
        monkeypatch.setenv("SPNNZ_MP_MAX", "98304")    # the opt-in multipass tier below the heavy path
    elif case % 3 == 1:
        monkeypatch.setenv("SPNNZ_MP_MAX", "98304")
        monkeypatch.setenv("SPNNZ_MP_PART", "150000")  # ... with too few passes: redos
    q = Predictor(0)
    q.load(a, b)
    prof = q.compute_flop()
    f, F, mx = oracle.compute_flop(a, b)
    assert (prof.flop_per_row == f).all() and prof.total_flop == F and prof.max_flop_row == mx
    ex = q.exact_symbolic()
    nnz, Z = oracle.exact_symbolic(a, b, f, mx)
    assert (ex.nnz_per_row == nnz).all() and ex.total_nnz == Z
    seed, frac = int(rng.integers(1, 1 << 40)), float(rng.choice([0.01, 0.1, 0.5]))
    rep = q.run_prediction(seed, SamplePolicy(frac, UNCAPPED))
    o, _, oceil, oreal = oracle.run_prediction(a, b, seed, frac, UNCAPPED)
    assert rep.stats.sampled_flop == o.sampled_flop and rep.stats.sampled_nnz == o.sampled_nnz
    assert rep.predicted_cr == o.predicted_cr and rep.z2_star == o.z2_star
    assert (rep.predicted_row_nnz_ceil == oceil).all() and (rep.predicted_row_nnz == oreal).all()
    q.close()


def test_detached_shards_more_ranks_than_heavy_samples(oracle):
    """FLOP-balanced windows when the ranks outnumber the useful samples: a
    matrix whose sampled FLOP sits in one hub row plus empty rows; 8 detached
    ranks still sum to the single-GPU f* and z*."""
    n = 4000
    rows = [list(range(0, n, 3))] + [[] for _ in range(n - 2)] + [[5, 6]]
    a = csr(n, n, rows)
    single = Predictor(0)
    single.load(a)
    ref = single.run_prediction(3, SamplePolicy(0.002, UNCAPPED))
    single.close()
    fs = zs = 0
    for r in range(8):
        q = Predictor(0, r, 8)
        q.load(a)
        rep = q.run_prediction(3, SamplePolicy(0.002, UNCAPPED))
        fs += rep.stats.sampled_flop
        zs += rep.stats.sampled_nnz
        q.close()
    assert (fs, zs) == (ref.stats.sampled_flop, ref.stats.sampled_nnz)


def test_pattern_floor_probe_both_shapes(P):
    # instrumentation (bench.py's roofline.pattern_*): the L2-gather probe for
    # the tile kernels and the shared-table probe for the row streams; neither
    # may disturb the FLOP pass that follows
    a = gen.uniform_len(1 << 14, 1 << 12, 4, 32, 11)   # K = 4096: row streams
    b = gen.geometric(1 << 12, 1 << 14, 12.0, 12)
    P.load(a, b)
    before = P.compute_flop().flop_per_row.copy()
    assert "row streams" in P.last_flop_kernel()
    s_ms, g_ms = P.probe_flop_floor(3)
    assert s_ms > 0 and g_ms > 0
    assert np.array_equal(P.compute_flop().flop_per_row, before)
    r = gen.rmat(17, 1 << 21, 0.57, 0.19, 0.19, 3)     # K = 131072: tiles, L2 gathers
    P.load(r, r)
    before = P.compute_flop().flop_per_row.copy()
    assert "row streams" not in P.last_flop_kernel()
    s_ms, g_ms = P.probe_flop_floor(3)
    assert s_ms > 0 and g_ms > 0
    assert np.array_equal(P.compute_flop().flop_per_row, before)


@pytest.mark.parametrize("part", [None, 7000, 1000000])
def test_multipass_tier_vs_oracle(oracle, part, monkeypatch):
    """Rows of 24576 < FLOP <= 98304 on the opt-in multipass hash tier: nearly all
    distinct, duplicate-heavy, one with more entries than the block (staged
    per pass), and rows just inside / outside the tier's limits; with the
    default part size, many small passes, and a part size that puts the whole
    row in one pass (the table fills: the row is redone with 2x, 4x passes)."""
    monkeypatch.setenv("SPNNZ_MP_MAX", "98304")  # the tier is opt-in
    if part is not None:
        monkeypatch.setenv("SPNNZ_MP_PART", str(part))
    rng = np.random.default_rng(23)
    nb, ncols = 6000, 1 << 22
    b_lens = list(rng.integers(20, 60, nb - 1200)) + [1] * 1200
    b_rows = [np.sort(rng.choice(ncols, size=int(L), replace=False)).tolist() for L in b_lens[:nb - 1200]]
    b_rows += [[int(rng.integers(0, 50))] for _ in range(1200)]  # one-entry rows over 50 columns: duplicates
    b = csr(nb, ncols, b_rows)
    long_ids = np.arange(nb - 1200)
    a_rows = [np.sort(rng.choice(long_ids, size=L, replace=False)).tolist() for L in (700, 1000, 1500, 2300, 620, 2700)]
    # duplicate-heavy: 1100 long rows' products + 1200 products over 50 columns
    a_rows.append(np.sort(np.concatenate([rng.choice(long_ids, size=700, replace=False),
                                          np.arange(nb - 1200, nb)])).tolist())
    a_rows.append([3, 4])
    a = csr(len(a_rows), nb, a_rows)
    q = Predictor(0)
    q.load(a, b)
    prof = q.compute_flop()
    f, F, mx = oracle.compute_flop(a, b)
    assert (prof.flop_per_row == f).all()
    assert ((f > 24576) & (f <= 98304)).sum() >= 5 and (f > 98304).any()
    assert max(len(r) for r in a_rows) > 1024  # an entry list longer than the block
    ex = q.exact_symbolic()
    nnz, Z = oracle.exact_symbolic(a, b, f, mx)
    assert (ex.nnz_per_row == nnz).all() and ex.total_nnz == Z
    rows = np.arange(a.rows, dtype=np.int32)[::-1].copy()
    s2 = q.sampled_symbolic(rows)
    assert (s2.nnz_per_row == nnz[rows]).all() and s2.total_nnz == Z
    ex2 = q.exact_symbolic()  # tickets and bin counters reset per call
    assert (ex2.nnz_per_row == nnz).all()
    q.close()
