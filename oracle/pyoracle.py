"""ctypes binding of the CPU checkers -- TEST INFRASTRUCTURE ONLY.

``Oracle`` wraps oracle/liboracle.so, the plain-C restatement of the
reference hot path (spnnz_oracle.c).  ``Reference`` wraps
oracle/_ref/libspnnz_ref.so, the reference's own headers compiled in place
(ref_shim.cpp), when it was built.  Only tests/, __graft_entry__.smoke() and
bench.py's CPU-baseline legs may import this module; the product path never
does.
"""
from __future__ import annotations

import ctypes
import os
from ctypes import POINTER, byref, c_double, c_int, c_int32, c_int64, c_uint64, c_void_p

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "libspnnz_ref.so")


class _Csr(ctypes.Structure):
    _fields_ = [("rows", c_int32), ("cols", c_int32), ("rpt", c_void_p), ("col", c_void_p)]


class OracleReport(ctypes.Structure):
    _fields_ = [("total_flop", c_int64), ("max_flop_row", c_int64), ("sample_num", c_int64),
                ("p", c_double), ("sampled_flop", c_int64), ("sampled_nnz", c_int64),
                ("sampled_cr", c_double), ("z1_star", c_double), ("z2_star", c_double),
                ("predicted_cr", c_double)]

    def as_dict(self):
        return {k: getattr(self, k) for k, _ in self._fields_}


def _csr(m) -> _Csr:
    return _Csr(m.rows, m.cols, m.rpt.ctypes.data, m.col.ctypes.data)


def build_if_missing():
    if not os.path.exists(ORACLE_SO):
        import subprocess
        subprocess.run(["make", "-C", HERE], check=True, capture_output=True)


class Oracle:
    """The C restatement (always available after `make -C oracle`)."""

    def __init__(self, threads: int = 0):
        build_if_missing()
        self.L = ctypes.CDLL(ORACLE_SO)
        self.threads = threads
        L = self.L
        L.oracle_last_error.restype = ctypes.c_char_p
        L.oracle_splitmix_next.restype = c_uint64
        L.oracle_splitmix_next.argtypes = [POINTER(c_uint64)]
        L.oracle_compute_flop.argtypes = [POINTER(_Csr), POINTER(_Csr), c_int, c_void_p, POINTER(c_int64), POINTER(c_int64)]
        L.oracle_sampled_flop.argtypes = [c_void_p, c_int64, c_void_p, c_int64, POINTER(c_int64)]
        L.oracle_sample_count.argtypes = [c_int32, c_double, c_int64, POINTER(c_int64), POINTER(c_double)]
        L.oracle_make_sample_plan.argtypes = [c_int32, c_uint64, c_double, c_int64, c_void_p, POINTER(c_int64), POINTER(c_double)]
        L.oracle_exact_symbolic.argtypes = [POINTER(_Csr), POINTER(_Csr), c_void_p, c_int64, c_int, c_void_p, POINTER(c_int64)]
        L.oracle_sampled_symbolic.argtypes = [POINTER(_Csr), POINTER(_Csr), c_void_p, c_int64, c_void_p, c_int64, c_int, c_void_p, POINTER(c_int64)]
        L.oracle_sampled_cr.restype = c_double
        L.oracle_sampled_cr.argtypes = [c_int64, c_int64]
        L.oracle_predict_reference.argtypes = [c_int64, c_double, POINTER(c_double)]
        L.oracle_predict_proposed.argtypes = [c_int64, c_int64, c_int64, POINTER(c_double), POINTER(c_double)]
        L.oracle_error_report_compute.argtypes = [c_double, c_double, c_int64, c_int64, c_int64, c_double, c_void_p]
        L.oracle_predict_row_structure.argtypes = [c_void_p, c_int64, c_double, c_void_p]
        L.oracle_predict_row_structure_ceil.argtypes = [c_void_p, c_int64, c_double, c_void_p]
        L.oracle_run_prediction.argtypes = [POINTER(_Csr), POINTER(_Csr), c_uint64, c_double, c_int64, c_int, POINTER(OracleReport), c_void_p, c_void_p, c_void_p]

    def _chk(self, rc):
        if rc == 1:
            raise ValueError(self.L.oracle_last_error().decode())
        if rc:
            raise RuntimeError(self.L.oracle_last_error().decode())

    def splitmix(self, seed: int, n: int):
        st = c_uint64(seed)
        return [self.L.oracle_splitmix_next(byref(st)) for _ in range(n)]

    def compute_flop(self, a, b):
        flop = np.empty(a.rows, np.int64)
        t, m = c_int64(), c_int64()
        self._chk(self.L.oracle_compute_flop(byref(_csr(a)), byref(_csr(b)), self.threads, flop.ctypes.data, byref(t), byref(m)))
        return flop, t.value, m.value

    def sampled_flop(self, flop, rows):
        rows = np.ascontiguousarray(rows, np.int32)
        out = c_int64()
        self._chk(self.L.oracle_sampled_flop(flop.ctypes.data, len(flop), rows.ctypes.data, len(rows), byref(out)))
        return out.value

    def sample_count(self, m, fraction, cap):
        n, p = c_int64(), c_double()
        self._chk(self.L.oracle_sample_count(m, fraction, cap if cap >= 0 else 2**63 - 1, byref(n), byref(p)))
        return n.value, p.value

    def make_sample_plan(self, m, seed, fraction, cap):
        n, _ = self.sample_count(m, fraction, cap)
        rows = np.empty(n, np.int32)
        nn, p = c_int64(), c_double()
        self._chk(self.L.oracle_make_sample_plan(m, seed, fraction, cap if cap >= 0 else 2**63 - 1, rows.ctypes.data, byref(nn), byref(p)))
        return rows, nn.value, p.value

    def exact_symbolic(self, a, b, flop, max_flop):
        out = np.empty(a.rows, np.int64)
        t = c_int64()
        self._chk(self.L.oracle_exact_symbolic(byref(_csr(a)), byref(_csr(b)), flop.ctypes.data, max_flop, self.threads, out.ctypes.data, byref(t)))
        return out, t.value

    def sampled_symbolic(self, a, b, flop, max_flop, rows):
        rows = np.ascontiguousarray(rows, np.int32)
        out = np.empty(len(rows), np.int64)
        t = c_int64()
        self._chk(self.L.oracle_sampled_symbolic(byref(_csr(a)), byref(_csr(b)), flop.ctypes.data, max_flop, rows.ctypes.data, len(rows), self.threads, out.ctypes.data, byref(t)))
        return out, t.value

    def predict_row_structure(self, flop, cr):
        out = np.empty(len(flop), np.float64)
        self._chk(self.L.oracle_predict_row_structure(flop.ctypes.data, len(flop), cr, out.ctypes.data))
        return out

    def predict_row_structure_ceil(self, flop, cr):
        out = np.empty(len(flop), np.int64)
        self._chk(self.L.oracle_predict_row_structure_ceil(flop.ctypes.data, len(flop), cr, out.ctypes.data))
        return out

    def estimators(self, f, z, F, p):
        z1, z2, cr = c_double(), c_double(), c_double()
        self._chk(self.L.oracle_predict_reference(z, p, byref(z1)))
        self.L.oracle_predict_proposed(f, z, F, byref(z2), byref(cr))
        return z1.value, z2.value, cr.value

    def error_report(self, z1, z2, f_star, Z, F, p):
        out = (c_double * 4)()
        self._chk(self.L.oracle_error_report_compute(z1, z2, f_star, Z, F, p, out))
        return tuple(out)

    def run_prediction(self, a, b, seed, fraction, cap, want_rows=True):
        rep = OracleReport()
        flop = np.empty(a.rows, np.int64) if want_rows else None
        ceil = np.empty(a.rows, np.int64) if want_rows else None
        real = np.empty(a.rows, np.float64) if want_rows else None
        self._chk(self.L.oracle_run_prediction(byref(_csr(a)), byref(_csr(b)), seed, fraction,
                                               cap if cap >= 0 else 2**63 - 1, self.threads, byref(rep),
                                               flop.ctypes.data if want_rows else None,
                                               ceil.ctypes.data if want_rows else None,
                                               real.ctypes.data if want_rows else None))
        return rep, flop, ceil, real


class RefReport(ctypes.Structure):
    _fields_ = OracleReport._fields_


class Reference:
    """The reference's own headers compiled in place (oracle/_ref)."""

    @staticmethod
    def available() -> bool:
        return os.path.exists(REF_SO)

    def __init__(self, threads: int = 0):
        self.L = ctypes.CDLL(REF_SO)
        self.threads = threads
        L = self.L
        L.ref_last_error.restype = ctypes.c_char_p
        L.ref_matrix_new.restype = c_void_p
        L.ref_matrix_new.argtypes = [c_int32, c_int32, c_void_p, c_void_p]
        L.ref_matrix_free.argtypes = [c_void_p]
        L.ref_profile_free.argtypes = [c_void_p]
        L.ref_compute_flop.argtypes = [c_void_p, c_void_p, c_int, c_void_p, POINTER(c_int64), POINTER(c_int64), POINTER(c_void_p)]
        L.ref_sampled_flop.argtypes = [c_void_p, c_void_p, c_int64, POINTER(c_int64)]
        L.ref_make_sample_plan.argtypes = [c_int32, c_uint64, c_double, c_int64, c_void_p, POINTER(c_int64), POINTER(c_double)]
        L.ref_exact_symbolic.argtypes = [c_void_p, c_void_p, c_void_p, c_int, c_void_p, POINTER(c_int64)]
        L.ref_sampled_symbolic.argtypes = [c_void_p, c_void_p, c_void_p, c_void_p, c_int64, c_int, c_void_p, POINTER(c_int64)]
        L.ref_predict_row_structure_ceil.argtypes = [c_void_p, c_double, c_void_p]
        L.ref_predict_row_structure.argtypes = [c_void_p, c_double, c_void_p]
        L.ref_run_pipeline.argtypes = [c_void_p, c_void_p, c_uint64, c_double, c_int64, c_int, POINTER(RefReport), c_void_p]
        L.ref_run_pipeline_ceil.argtypes = L.ref_run_pipeline.argtypes
        L.ref_profile_new.restype = c_void_p
        L.ref_profile_new.argtypes = [c_void_p, c_int64, c_int64, c_int64]
        L.ref_run_with_plan.argtypes = [c_void_p, c_void_p, c_void_p, c_void_p, c_int64, c_double, c_uint64,
                                        c_int, POINTER(RefReport), c_void_p, c_void_p]
        L.ref_error_report.argtypes = [c_double, c_double, c_int64, c_int64, c_int64, c_double, c_void_p]
        L.ref_splitmix_seq.argtypes = [c_uint64, c_int64, c_void_p]
        L.ref_matrix_export.argtypes = [c_void_p, POINTER(c_int32), POINTER(c_int32), POINTER(c_int64), c_void_p, c_void_p]
        L.ref_generate_synthetic.argtypes = [c_int, c_int32, c_int32, c_double, c_uint64, c_int32, c_double,
                                             POINTER(c_void_p), ctypes.c_char_p, c_int]
        L.ref_read_matrix_market.argtypes = [ctypes.c_char_p, POINTER(c_void_p)]
        L.ref_write_matrix_market.argtypes = [ctypes.c_char_p, c_void_p]

    def _chk(self, rc):
        if rc == 1:
            raise ValueError(self.L.ref_last_error().decode())
        if rc:
            raise RuntimeError(self.L.ref_last_error().decode())

    def matrix(self, m):
        return self.L.ref_matrix_new(m.rows, m.cols, m.rpt.ctypes.data, m.col.ctypes.data)

    def free_matrix(self, h):
        self.L.ref_matrix_free(h)

    def export(self, h):
        """(rows, cols, rpt, col) of a reference matrix handle."""
        r, c, n = c_int32(), c_int32(), c_int64()
        self.L.ref_matrix_export(h, byref(r), byref(c), byref(n), None, None)
        rpt = np.empty(r.value + 1, np.int64)
        col = np.empty(max(n.value, 1), np.int32)
        self.L.ref_matrix_export(h, byref(r), byref(c), byref(n), rpt.ctypes.data, col.ctypes.data)
        return r.value, c.value, rpt, col[: n.value]

    def generate_synthetic(self, model, rows, cols, target, seed, bandwidth=0, skew=1.0):
        """spnnz::generate_synthetic + synthetic_name -> (rows, cols, rpt, col, name)."""
        h = c_void_p()
        name = ctypes.create_string_buffer(256)
        codes = {"uniform": 0, "banded": 1, "power-law": 2}
        self._chk(self.L.ref_generate_synthetic(codes[model], rows, cols, target, seed, bandwidth, skew,
                                                byref(h), name, 256))
        out = self.export(h)
        self.free_matrix(h)
        return (*out, name.value.decode())

    def read_matrix_market(self, path):
        h = c_void_p()
        self._chk(self.L.ref_read_matrix_market(str(path).encode(), byref(h)))
        out = self.export(h)
        self.free_matrix(h)
        return out

    def write_matrix_market(self, path, m):
        h = self.matrix(m)
        try:
            self._chk(self.L.ref_write_matrix_market(str(path).encode(), h))
        finally:
            self.free_matrix(h)

    def splitmix(self, seed, n):
        out = np.empty(n, np.uint64)
        self.L.ref_splitmix_seq(seed, n, out.ctypes.data)
        return [int(x) for x in out]

    def compute_flop(self, ha, hb, rows, keep_profile=False):
        flop = np.empty(rows, np.int64)
        t, m, prof = c_int64(), c_int64(), c_void_p()
        self._chk(self.L.ref_compute_flop(ha, hb, self.threads, flop.ctypes.data, byref(t), byref(m), byref(prof)))
        if not keep_profile:
            self.L.ref_profile_free(prof)
            prof = None
        return flop, t.value, m.value, prof

    def make_sample_plan(self, m, seed, fraction, cap):
        n, p = c_int64(), c_double()
        cap = cap if cap >= 0 else 2**63 - 1
        self._chk(self.L.ref_make_sample_plan(m, seed, fraction, cap, None, byref(n), byref(p)))
        rows = np.empty(n.value, np.int32)
        self._chk(self.L.ref_make_sample_plan(m, seed, fraction, cap, rows.ctypes.data, byref(n), byref(p)))
        return rows, n.value, p.value

    def exact_symbolic(self, ha, hb, prof, rows):
        out = np.empty(rows, np.int64)
        t = c_int64()
        self._chk(self.L.ref_exact_symbolic(ha, hb, prof, self.threads, out.ctypes.data, byref(t)))
        return out, t.value

    def sampled_symbolic(self, ha, hb, prof, sample_rows):
        sample_rows = np.ascontiguousarray(sample_rows, np.int32)
        out = np.empty(len(sample_rows), np.int64)
        t = c_int64()
        self._chk(self.L.ref_sampled_symbolic(ha, hb, prof, sample_rows.ctypes.data, len(sample_rows), self.threads, out.ctypes.data, byref(t)))
        return out, t.value

    def predict_row_structure_ceil(self, prof, cr, rows):
        out = np.empty(rows, np.int64)
        self._chk(self.L.ref_predict_row_structure_ceil(prof, cr, out.ctypes.data))
        return out

    def predict_row_structure(self, prof, cr, rows):
        out = np.empty(rows, np.float64)
        self._chk(self.L.ref_predict_row_structure(prof, cr, out.ctypes.data))
        return out

    def run_pipeline(self, ha, hb, seed, fraction, cap, rows, want_ceil=True, real_view=True):
        """compute_flop + make_sample_plan + run_prediction_with_plan (which
        also builds the real per-row view) + predict_row_structure_ceil; with
        real_view=False the same functions composed without the real view
        (the outputs the GPU step produces)."""
        rep = RefReport()
        ceil = np.empty(rows, np.int64) if want_ceil else None
        fn = self.L.ref_run_pipeline if real_view else self.L.ref_run_pipeline_ceil
        self._chk(fn(ha, hb, seed, fraction, cap if cap >= 0 else 2**63 - 1,
                     self.threads, byref(rep), ceil.ctypes.data if want_ceil else None))
        return rep, ceil

    def run_with_plan(self, ha, hb, flop, total, mx, rows, p, seed=0):
        """spnnz::run_prediction_with_plan on a hand-built FlopProfile
        {flop, total, mx}: (report, real view, ceil view)."""
        flop = np.ascontiguousarray(flop, np.int64)
        rows = np.ascontiguousarray(rows, np.int32)
        prof = self.L.ref_profile_new(flop.ctypes.data, len(flop), int(total), int(mx))
        rep = RefReport()
        real = np.empty(len(flop), np.float64)
        ceil = np.empty(len(flop), np.int64)
        try:
            self._chk(self.L.ref_run_with_plan(ha, hb, prof, rows.ctypes.data, len(rows), p, seed,
                                               self.threads, byref(rep), real.ctypes.data, ceil.ctypes.data))
        finally:
            self.L.ref_profile_free(prof)
        return rep, real, ceil

    def error_report(self, z1, z2, f_star, Z, F, p):
        out = (c_double * 4)()
        self._chk(self.L.ref_error_report(z1, z2, f_star, Z, F, p, out))
        return tuple(out)
