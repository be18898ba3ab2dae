"""Synthetic inputs for the five BASELINE.json configurations (structure only).

Binds ``_lib/libspnnz_gen.so`` (csrc/gen/generators.cpp): deterministic,
thread-count invariant, one SplitMix64 substream per row.  Input plumbing,
never on the timed path.
"""
from __future__ import annotations

import ctypes
import os
from ctypes import POINTER, c_double, c_int, c_int32, c_int64, c_uint64

import numpy as np

from .capi import GEN_PATH
from .spnnz import CsrMatrix


class _GenCsr(ctypes.Structure):
    _fields_ = [("rows", c_int32), ("cols", c_int32), ("nnz", c_int64),
                ("rpt", POINTER(c_int64)), ("col", POINTER(c_int32))]


_g = None


def _lib():
    global _g
    if _g is None:
        if not os.path.exists(GEN_PATH):
            raise RuntimeError(f"{GEN_PATH} not built (run `make`)")
        _g = ctypes.CDLL(GEN_PATH)
        _g.spnnz_gen_free.argtypes = [POINTER(_GenCsr)]
        _g.spnnz_gen_poisson_uniform.argtypes = [c_int32, c_int32, c_double, c_int32, c_int32, c_uint64, c_int, POINTER(_GenCsr)]
        _g.spnnz_gen_rmat.argtypes = [c_int, c_int64, c_double, c_double, c_double, c_uint64, c_int, POINTER(_GenCsr)]
        _g.spnnz_gen_stencil27.argtypes = [c_int32, c_int32, c_int32, c_int, POINTER(_GenCsr)]
        _g.spnnz_gen_uniform_len.argtypes = [c_int32, c_int32, c_int32, c_int32, c_uint64, c_int, POINTER(_GenCsr)]
        _g.spnnz_gen_geometric.argtypes = [c_int32, c_int32, c_double, c_uint64, c_int, POINTER(_GenCsr)]
        _g.spnnz_gen_random_pattern.argtypes = [c_int32, c_int32, c_double, POINTER(c_uint64), POINTER(_GenCsr)]
        _g.spnnz_gen_synthetic.argtypes = [c_int, c_int32, c_int32, c_double, c_uint64, c_int32, c_double,
                                           c_int, POINTER(_GenCsr)]
        _g.spnnz_mm_read.argtypes = [ctypes.c_char_p, c_int, POINTER(_GenCsr), ctypes.c_char_p, c_int]
        _g.spnnz_mm_write.argtypes = [ctypes.c_char_p, POINTER(_GenCsr)]
    return _g


def _take(g: _GenCsr, rc: int) -> CsrMatrix:
    if rc != 0:
        raise RuntimeError(f"generator failed ({rc})")
    try:
        rpt = np.ctypeslib.as_array(g.rpt, (g.rows + 1,)).copy()
        col = (np.ctypeslib.as_array(g.col, (g.nnz,)).copy() if g.nnz
               else np.zeros(0, np.int32))
    finally:
        _lib().spnnz_gen_free(ctypes.byref(g))
    return CsrMatrix(g.rows, g.cols, rpt, col)


def poisson_uniform(rows, cols, mean, lo, hi, seed, threads=0) -> CsrMatrix:
    g = _GenCsr()
    return _take(g, _lib().spnnz_gen_poisson_uniform(rows, cols, mean, lo, hi, seed, threads, ctypes.byref(g)))


def rmat(log2n, draws, a, b, c, seed, threads=0) -> CsrMatrix:
    g = _GenCsr()
    return _take(g, _lib().spnnz_gen_rmat(log2n, draws, a, b, c, seed, threads, ctypes.byref(g)))


def stencil27(nx, ny, nz, threads=0) -> CsrMatrix:
    g = _GenCsr()
    return _take(g, _lib().spnnz_gen_stencil27(nx, ny, nz, threads, ctypes.byref(g)))


def uniform_len(rows, cols, lo, hi, seed, threads=0) -> CsrMatrix:
    g = _GenCsr()
    return _take(g, _lib().spnnz_gen_uniform_len(rows, cols, lo, hi, seed, threads, ctypes.byref(g)))


def geometric(rows, cols, mean, seed, threads=0) -> CsrMatrix:
    g = _GenCsr()
    return _take(g, _lib().spnnz_gen_geometric(rows, cols, mean, seed, threads, ctypes.byref(g)))


# --------------------------------------------------------- synthetic corpus
MODELS = {"uniform": 0, "banded": 1, "power-law": 2}


def synthetic(model: str, rows: int, cols: int, target: float, seed: int, bandwidth: int = 0,
              skew: float = 1.0, threads: int = 0) -> CsrMatrix:
    """spnnz::generate_synthetic (synthetic.hpp:92-154): the reference's
    synthetic corpus model, restated row-parallel in csrc/gen/generators.cpp.
    Raises ValueError for an infeasible spec like the reference."""
    g = _GenCsr()
    rc = _lib().spnnz_gen_synthetic(MODELS[model], rows, cols, float(target), seed, bandwidth,
                                    float(skew), threads, ctypes.byref(g))
    if rc == 3:
        raise ValueError(f"generate_synthetic: infeasible spec rows={rows} cols={cols} "
                         f"target_nnz_per_row={target}")
    return _take(g, rc)


def _g6(v: float) -> str:
    """printf("%.6g")."""
    return "%.6g" % v


def synthetic_name(model: str, rows: int, cols: int, target: float, seed: int, bandwidth: int = 0,
                   skew: float = 1.0) -> str:
    """spnnz::synthetic_name (synthetic.hpp:203-215)."""
    name = f"synth:{model}:{rows}x{cols}:nnz={_g6(target)}"
    if model == "banded" and bandwidth > 0:
        name += f":bw={bandwidth}"
    if model == "power-law":
        name += f":skew={_g6(skew)}"
    return name + f":seed={seed}"


def parse_synthetic_spec(text: str) -> dict:
    """spnnz::parse_synthetic_spec (synthetic.hpp:157-200): "synth:<model>:RxC:key=val..."."""
    parts = text.split(":")
    if len(parts) < 3 or parts[0] != "synth":
        raise ValueError(f"invalid synthetic spec '{text}'")
    if parts[1] not in MODELS:
        raise ValueError(f"unknown synthetic model '{parts[1]}'")
    if "x" not in parts[2]:
        raise ValueError(f"invalid dimensions '{parts[2]}' (want RxC)")
    r, c = parts[2].split("x", 1)
    spec = dict(model=parts[1], rows=int(r), cols=int(c), target=0.0, seed=0, bandwidth=0, skew=1.0)
    keys = {"nnz": ("target", float), "seed": ("seed", int), "bw": ("bandwidth", int),
            "skew": ("skew", float)}
    for opt in parts[3:]:
        if "=" not in opt:
            raise ValueError(f"invalid synthetic option '{opt}'")
        k, v = opt.split("=", 1)
        if k not in keys:
            raise ValueError(f"unknown synthetic option '{k}'")
        spec[keys[k][0]] = keys[k][1](v)
    return spec


# ------------------------------------------------------------ Matrix Market
class ParseError(ValueError):
    """spnnz::parse_error: the message ends with " (line N)"."""


def read_matrix_market(path, threads: int = 0) -> CsrMatrix:
    """spnnz::read_matrix_market (matrix_market.hpp:89-196), structure only
    (csrc/gen/mmio.cpp): symmetric kinds mirrored, duplicates collapsed,
    columns sorted."""
    g = _GenCsr()
    err = ctypes.create_string_buffer(512)
    rc = _lib().spnnz_mm_read(str(path).encode(), threads, ctypes.byref(g), err, 512)
    if rc == 4:
        raise ParseError(err.value.decode(errors="replace"))
    if rc:
        raise RuntimeError(err.value.decode(errors="replace") or f"read_matrix_market failed ({rc})")
    return _take(g, 0)


def write_matrix_market(path, m: CsrMatrix) -> None:
    """spnnz::write_matrix_market (matrix_market.hpp:200-211): pattern, general."""
    g = _GenCsr(m.rows, m.cols, int(m.rpt[m.rows]), m.rpt.ctypes.data_as(POINTER(ctypes.c_int64)),
                m.col.ctypes.data_as(POINTER(c_int32)))
    if _lib().spnnz_mm_write(str(path).encode(), ctypes.byref(g)):
        raise RuntimeError(f"cannot write {path}")


# The reference's default corpus (bench.hpp:496-517): 12 specs whose 144
# ordered products span CR ~1 to ~20.  (rows, cols, model, nnz/row, seed,
# bandwidth, skew)
DEFAULT_CORPUS = [
    (20000, 20000, "uniform", 3.0, 101, 0, 1.0),
    (12000, 12000, "uniform", 8.0, 102, 0, 1.0),
    (6000, 6000, "uniform", 25.0, 103, 0, 1.0),
    (4000, 4000, "uniform", 40.0, 104, 0, 1.0),
    (3000, 3000, "uniform", 60.0, 105, 0, 1.0),
    (8000, 2000, "uniform", 50.0, 106, 0, 1.0),
    (8000, 1000, "uniform", 55.0, 107, 0, 1.0),
    (10000, 10000, "banded", 10.0, 110, 50, 1.0),
    (12000, 12000, "banded", 18.0, 113, 30, 1.0),
    (6000, 300, "uniform", 77.0, 109, 0, 1.0),
    (15000, 15000, "power-law", 6.0, 111, 0, 0.9),
    (9000, 9000, "power-law", 15.0, 112, 0, 0.7),
]


class SplitMix64:
    """spnnz::SplitMix64 (rng.hpp:10-41) for driving the reference's test loops."""
    M = (1 << 64) - 1

    def __init__(self, seed: int):
        self.state = seed & self.M

    def next_u64(self) -> int:
        self.state = (self.state + 0x9E3779B97F4A7C15) & self.M
        z = self.state
        z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & self.M
        z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & self.M
        return z ^ (z >> 31)

    def next_double(self) -> float:
        return float(self.next_u64() >> 11) * 2.0 ** -53

    def next_below(self, bound: int) -> int:
        return (self.next_u64() * bound) >> 64


def random_pattern(rows: int, cols: int, density: float, rng: SplitMix64) -> CsrMatrix:
    """oracle::random_pattern (proj/tests/oracle.hpp:63-74); advances rng."""
    st = c_uint64(rng.state)
    g = _GenCsr()
    m = _take(g, _lib().spnnz_gen_random_pattern(rows, cols, density, ctypes.byref(st), ctypes.byref(g)))
    rng.state = st.value
    return m


# The BASELINE.json configurations.  (A, B) with B None for C = A*A.
CONFIGS = {
    1: dict(name="cfg1_poisson4096", fraction=0.01, seed=1,
            desc="A*A, n=4096, Poisson(8) lengths clipped to [1,64], uniform distinct cols"),
    2: dict(name="cfg2_rmat20", fraction=0.003, seed=2,
            desc="A*A, R-MAT 2^20, 16*2^20 draws, (.57,.19,.19,.05), deduplicated"),
    3: dict(name="cfg3_stencil27_128", fraction=0.001, seed=3,
            desc="A*A, 27-point stencil on 128^3"),
    4: dict(name="cfg4_rect", fraction=0.005, seed=4,
            desc="A*B, A 2^20 x 2^16 U[4,32] lengths, B 2^16 x 2^20 Geometric(12) lengths"),
    5: dict(name="cfg5_rmat24", fraction=0.001, seed=5,
            desc="A*A, R-MAT 2^24, 24*2^24 draws, (.45,.22,.22,.11), deduplicated"),
}


def make_config(cfg: int, threads: int = 0):
    """Returns (A, B) host CsrMatrix for BASELINE.json config `cfg` (B is A for A*A)."""
    if cfg == 1:
        a = poisson_uniform(4096, 4096, 8.0, 1, 64, 1, threads)
        return a, a
    if cfg == 2:
        a = rmat(20, 16 << 20, 0.57, 0.19, 0.19, 2, threads)
        return a, a
    if cfg == 3:
        a = stencil27(128, 128, 128, threads)
        return a, a
    if cfg == 4:
        a = uniform_len(1 << 20, 1 << 16, 4, 32, 4, threads)
        b = geometric(1 << 16, 1 << 20, 12.0, 4 ^ 0x5EED, threads)
        return a, b
    if cfg == 5:
        a = rmat(24, 24 << 24, 0.45, 0.22, 0.22, 5, threads)
        return a, a
    raise ValueError(f"unknown config {cfg}")
