"""Shared helpers for the test suites (numpy dense oracles of
proj/tests/oracle.hpp and array digests)."""
import hashlib

import numpy as np


def digest(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()[:32]


def to_dense(m) -> np.ndarray:
    """oracle::to_dense (proj/tests/oracle.hpp:15-25)."""
    d = np.zeros((m.rows, m.cols), dtype=bool)
    r = np.repeat(np.arange(m.rows), np.diff(m.rpt))
    d[r, m.col] = True
    return d


def dense_bool_multiply_row_nnz(a, b) -> np.ndarray:
    """oracle::dense_bool_multiply_row_nnz (oracle.hpp:28-43)."""
    da, db = to_dense(a).astype(np.int64), to_dense(b).astype(np.int64)
    return ((da @ db) > 0).sum(axis=1).astype(np.int64)


def dense_flop_count(a, b) -> int:
    """oracle::dense_flop_count (oracle.hpp:47-60)."""
    da, db = to_dense(a).astype(np.int64), to_dense(b).astype(np.int64)
    return int((da @ db).sum())


def identity(n):
    from paper_2207_13848_b200.spnnz import CsrMatrix
    return CsrMatrix(n, n, np.arange(n + 1, dtype=np.int64), np.arange(n, dtype=np.int32))


def upper_2x2():
    """[[1,1],[0,1]] (test_flop.cpp:20-23)."""
    from paper_2207_13848_b200.spnnz import CsrMatrix
    return CsrMatrix(2, 2, np.array([0, 2, 3], np.int64), np.array([0, 1, 1], np.int32))


def csr(rows, cols, row_lists):
    from paper_2207_13848_b200.spnnz import CsrMatrix
    rpt = np.zeros(rows + 1, np.int64)
    for i, r in enumerate(row_lists):
        rpt[i + 1] = rpt[i] + len(r)
    col = np.array([c for r in row_lists for c in r], np.int32)
    return CsrMatrix(rows, cols, rpt, col)
