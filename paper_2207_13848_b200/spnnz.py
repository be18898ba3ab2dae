"""Python mirror of the reference predictor API (namespace ``spnnz``,
/root/reference/proj/include/spnnz/{csr,flop,symbolic,predict}.hpp), computed
on the B200 through the C ABI (include/spnnz_gpu/capi.h).

Same names, argument meaning and error behaviour as the reference: argument
errors raise ``ValueError`` where the reference throws
``std::invalid_argument``.  ``threads`` arguments are accepted for signature
parity and ignored (the GPU grid replaces ``parallel_blocks``).

Two ways in:
  * free functions (``compute_flop(a, b)``, ``run_prediction(a, b, seed)``, ...)
    use a per-process default ``Predictor`` on ``cuda:0`` and (re)upload the
    matrices when they change -- the drop-in for single-call users;
  * ``Predictor`` keeps matrices resident in HBM across calls and, with
    ``world > 1``, owns this rank's nnz-balanced shard of A plus a replica of B
    (one NCCL all-reduce per prediction).
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass, field
from typing import Optional, Sequence

import numpy as np

from . import capi
from .capi import DEVICE, HOST, CsrView, Report, check, lib

NO_CAP = -1  # cap < 0: sample the stated fraction without the 300-row cap


# --------------------------------------------------------------- data model
@dataclass
class CsrMatrix:
    """spnnz::CsrMatrix (csr.hpp:22-35), structure only (val is never read)."""
    rows: int = 0
    cols: int = 0
    rpt: np.ndarray = field(default_factory=lambda: np.zeros(1, np.int64))
    col: np.ndarray = field(default_factory=lambda: np.zeros(0, np.int32))

    def __post_init__(self):
        self.rpt = np.ascontiguousarray(self.rpt, dtype=np.int64)
        self.col = np.ascontiguousarray(self.col, dtype=np.int32)

    def nnz(self) -> int:
        return int(self.rpt[-1]) if len(self.rpt) else 0

    def view(self) -> CsrView:
        return CsrView(self.rows, self.cols, self.rpt.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)),
                       self.col.ctypes.data_as(ctypes.POINTER(ctypes.c_int32)))


def from_triplets(triplets: Sequence[tuple], rows: int, cols: int) -> CsrMatrix:
    """spnnz::from_triplets (csr.hpp:46-100), structure only: duplicates collapse."""
    if rows < 0 or cols < 0:
        raise ValueError("from_triplets: negative dimensions")
    t = np.asarray(triplets, dtype=np.int64).reshape(-1, 2) if len(triplets) else np.zeros((0, 2), np.int64)
    if len(t) and (t[:, 0].min() < 0 or t[:, 0].max() >= rows or t[:, 1].min() < 0 or t[:, 1].max() >= cols):
        raise ValueError("from_triplets: triplet out of bounds")
    key = np.unique(t[:, 0] * max(cols, 1) + t[:, 1])
    r, c = key // max(cols, 1), key % max(cols, 1)
    rpt = np.zeros(rows + 1, np.int64)
    np.add.at(rpt, r + 1, 1)
    return CsrMatrix(rows, cols, np.cumsum(rpt), c.astype(np.int32))


@dataclass
class FlopProfile:
    """spnnz::FlopProfile (flop.hpp:15-19)."""
    flop_per_row: np.ndarray = field(default_factory=lambda: np.zeros(0, np.int64))
    total_flop: int = 0
    max_flop_row: int = 0


@dataclass
class RowNnzResult:
    """spnnz::RowNnzResult (symbolic.hpp:74-77)."""
    nnz_per_row: np.ndarray = field(default_factory=lambda: np.zeros(0, np.int64))
    total_nnz: int = 0


@dataclass
class SamplePolicy:
    """spnnz::SamplePolicy (predict.hpp:20-23); cap < 0 disables the cap."""
    fraction: float = 0.003
    cap: int = 300


@dataclass
class SamplePlan:
    """spnnz::SamplePlan (predict.hpp:27-32)."""
    sample_rows: np.ndarray = field(default_factory=lambda: np.zeros(0, np.int32))
    sample_num: int = 0
    p: float = 0.0
    seed: int = 0


@dataclass
class SampleStats:
    """spnnz::SampleStats (predict.hpp:75-79)."""
    sampled_flop: int = 0
    sampled_nnz: int = 0
    sampled_cr: float = 1.0


@dataclass
class ProposedPrediction:
    """spnnz::ProposedPrediction (predict.hpp:101-104)."""
    z2_star: float = 0.0
    predicted_cr: float = 1.0


@dataclass
class ErrorReport:
    """spnnz::ErrorReport (predict.hpp:156-161)."""
    eps1: float = 0.0
    eps_f: float = 0.0
    eps2: float = 0.0
    identity_residual: float = 0.0


@dataclass
class PredictionReport:
    """spnnz::PredictionReport (predict.hpp:192-200) plus the integer ceil view
    (predict_row_structure_ceil) that allocation consumers use."""
    z1_star: float = 0.0
    z2_star: float = 0.0
    predicted_cr: float = 1.0
    predicted_row_nnz: Optional[np.ndarray] = None
    plan: SamplePlan = field(default_factory=SamplePlan)
    stats: SampleStats = field(default_factory=SampleStats)
    total_flop: int = 0
    predicted_row_nnz_ceil: Optional[np.ndarray] = None
    max_flop_row: int = 0


def _ptr(a) -> int:
    """Device pointer of a torch tensor or host pointer of a numpy array."""
    if a is None:
        return None
    if isinstance(a, np.ndarray):
        return a.ctypes.data
    return a.data_ptr()


def _res(a) -> int:
    if a is None or isinstance(a, np.ndarray):
        return HOST
    return DEVICE if getattr(a, "is_cuda", False) else HOST


# ---------------------------------------------------------------- Predictor
class Predictor:
    """One device context (C ABI ``spnnz_gpu_ctx``) on ``device`` for
    rank ``rank`` of ``world``."""

    def __init__(self, device: int = 0, rank: int = 0, world: int = 1,
                 nccl_id: Optional[bytes] = None):
        self._ctx = ctypes.c_void_p()
        idbuf = ctypes.create_string_buffer(nccl_id, 128) if nccl_id else None
        check(lib().spnnz_gpu_create(device, rank, world, idbuf, ctypes.byref(self._ctx)))
        self.device, self.rank, self.world = device, rank, world
        self.row_lo = self.row_hi = self.a_rows = 0

    @staticmethod
    def nccl_unique_id() -> bytes:
        buf = ctypes.create_string_buffer(128)
        check(lib().spnnz_gpu_nccl_unique_id(buf))
        return buf.raw

    def close(self):
        if self._ctx:
            lib().spnnz_gpu_destroy(self._ctx)
            self._ctx = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def ctx(self):
        return self._ctx

    def _after_torch(self, *objs):
        """Device tensors are read after the work torch queued on its current
        stream (spnnz_gpu_set_input_stream), so a tensor an asynchronous kernel
        just wrote is complete when the context's stream reads it."""
        for o in objs:
            if _res(o) == DEVICE:
                import torch
                h = torch.cuda.current_stream(o.device).cuda_stream
                check(lib().spnnz_gpu_set_input_stream(self._ctx, ctypes.c_void_p(h)))
                return

    # -- matrices
    def load(self, a, b=None, residency: Optional[int] = None):
        """Upload A (this rank's shard) and B (replicated).  ``a``/``b`` are
        CsrMatrix (host) or objects with rows/cols/rpt/col device tensors."""
        res = residency if residency is not None else _res(a.rpt)
        self._after_torch(a.rpt)
        va = CsrView(a.rows, a.cols, ctypes.cast(_ptr(a.rpt), ctypes.POINTER(ctypes.c_int64)),
                     ctypes.cast(_ptr(a.col), ctypes.POINTER(ctypes.c_int32)))
        vb = None
        if b is not None and b is not a:
            vb = CsrView(b.rows, b.cols, ctypes.cast(_ptr(b.rpt), ctypes.POINTER(ctypes.c_int64)),
                         ctypes.cast(_ptr(b.col), ctypes.POINTER(ctypes.c_int32)))
        check(lib().spnnz_gpu_load(self._ctx, ctypes.byref(va), ctypes.byref(vb) if vb else None, res))
        lo, hi, rows = ctypes.c_int32(), ctypes.c_int32(), ctypes.c_int32()
        check(lib().spnnz_gpu_shard(self._ctx, ctypes.byref(lo), ctypes.byref(hi), ctypes.byref(rows)))
        self.row_lo, self.row_hi, self.a_rows = lo.value, hi.value, rows.value
        return self

    def ensure_loaded(self, a, b):
        """Upload (A, B) for a stateless reference-style call.  The reference's
        free functions read their matrices on every call, so this always
        re-uploads: a cache keyed on object ids or buffer addresses can match a
        different matrix once the old one is freed (CPython and the allocator
        reuse both), and it misses in-place edits.  Callers that want the
        matrices to stay resident use a Predictor's methods directly."""
        self.load(a, None if b is a else b)

    @property
    def local_rows(self) -> int:
        return self.row_hi - self.row_lo

    # -- reference functions
    def compute_flop(self, out=None) -> FlopProfile:
        m = self.local_rows
        flop = out if out is not None else np.empty(m, np.int64)
        tot, mx = ctypes.c_int64(), ctypes.c_int64()
        check(lib().spnnz_gpu_compute_flop(self._ctx, _ptr(flop), _res(flop), ctypes.byref(tot),
                                           ctypes.byref(mx)))
        return FlopProfile(flop, tot.value, mx.value)

    def set_profile(self, profile: FlopProfile):
        f = profile.flop_per_row
        if isinstance(f, np.ndarray):
            f = np.ascontiguousarray(f, dtype=np.int64)
        self._after_torch(f)
        check(lib().spnnz_gpu_set_profile(self._ctx, _ptr(f), len(f), _res(f),
                                          int(profile.total_flop), int(profile.max_flop_row)))

    def sampled_flop(self, rows) -> int:
        rows = _rows_arg(rows)
        self._after_torch(rows)
        out = ctypes.c_int64()
        check(lib().spnnz_gpu_sampled_flop(self._ctx, _ptr(rows), len(rows), _res(rows),
                                           ctypes.byref(out)))
        return out.value

    def make_sample_plan(self, num_rows: int, seed: int, policy: SamplePolicy = SamplePolicy(),
                         out=None) -> SamplePlan:
        n, p = ctypes.c_int64(), ctypes.c_double()
        check(lib().spnnz_gpu_make_sample_plan(self._ctx, num_rows, seed, policy.fraction,
                                               policy.cap, None, HOST, ctypes.byref(n), ctypes.byref(p)))
        rows = out if out is not None else np.empty(n.value, np.int32)
        check(lib().spnnz_gpu_make_sample_plan(self._ctx, num_rows, seed, policy.fraction,
                                               policy.cap, _ptr(rows), _res(rows), ctypes.byref(n),
                                               ctypes.byref(p)))
        return SamplePlan(rows, n.value, p.value, seed)

    def sampled_symbolic(self, rows, per_sample: bool = True) -> RowNnzResult:
        rows = _rows_arg(rows)
        out = np.empty(len(rows), np.int64) if per_sample else None
        tot = ctypes.c_int64()
        res = _res(rows)
        self._after_torch(rows)
        if res == DEVICE and per_sample:
            import torch
            out = torch.empty(len(rows), dtype=torch.int64, device=rows.device)
        check(lib().spnnz_gpu_sampled_symbolic(self._ctx, _ptr(rows), len(rows), res, _ptr(out),
                                               ctypes.byref(tot)))
        return RowNnzResult(out, tot.value)

    def exact_symbolic(self, per_row: bool = True) -> RowNnzResult:
        out = np.empty(self.local_rows, np.int64) if per_row else None
        tot = ctypes.c_int64()
        check(lib().spnnz_gpu_exact_symbolic(self._ctx, _ptr(out), HOST, ctypes.byref(tot)))
        return RowNnzResult(out, tot.value)

    def predict_row_structure(self, cr: float, out=None) -> np.ndarray:
        o = out if out is not None else np.empty(self.local_rows, np.float64)
        check(lib().spnnz_gpu_predict_row_structure(self._ctx, cr, _ptr(o), _res(o)))
        return o

    def predict_row_structure_ceil(self, cr: float, out=None) -> np.ndarray:
        o = out if out is not None else np.empty(self.local_rows, np.int64)
        check(lib().spnnz_gpu_predict_row_structure_ceil(self._ctx, cr, _ptr(o), _res(o)))
        return o

    def run_prediction(self, seed: int, policy: SamplePolicy = SamplePolicy(), *, ceil_out=None,
                       real_out=None, samples_out=None, residency: Optional[int] = None,
                       want_real: bool = True, want_ceil: bool = True,
                       want_samples: bool = True) -> PredictionReport:
        """run_prediction (predict.hpp:220-226) + the ceil view, one device pipeline."""
        m = self.local_rows
        res = residency if residency is not None else (
            _res(ceil_out) if ceil_out is not None else _res(real_out) if real_out is not None else HOST)
        if res == HOST:
            if ceil_out is None and want_ceil:
                ceil_out = np.empty(m, np.int64)
            if real_out is None and want_real:
                real_out = np.empty(m, np.float64)
            n, _ = plan_size(self.a_rows, policy)
            if samples_out is None and want_samples:
                samples_out = np.empty(n, np.int32)
        rep = Report()
        check(lib().spnnz_gpu_run_prediction(self._ctx, seed, policy.fraction, policy.cap,
                                             ctypes.byref(rep), _ptr(ceil_out), _ptr(real_out),
                                             _ptr(samples_out), res))
        return _report(rep, real_out, ceil_out, samples_out, seed)

    def run_prediction_with_plan(self, plan: SamplePlan, profile: Optional[FlopProfile] = None, *,
                                 want_real=True, want_ceil=True) -> PredictionReport:
        """run_prediction_with_plan (predict.hpp:202-216) on `profile` (installed
        with set_profile; its flop is each row's table size, f* and the views
        come from it, F is its total_flop).  Without one, the profile of the
        loaded matrices is computed on the device first (nothing copied back)."""
        if profile is not None:
            self.set_profile(profile)
        else:
            t, mx = ctypes.c_int64(), ctypes.c_int64()
            check(lib().spnnz_gpu_compute_flop(self._ctx, None, HOST, ctypes.byref(t), ctypes.byref(mx)))
        m = self.local_rows
        rows = _rows_arg(plan.sample_rows)
        self._after_torch(rows)
        ceil_out = np.empty(m, np.int64) if want_ceil else None
        real_out = np.empty(m, np.float64) if want_real else None
        rep = Report()
        check(lib().spnnz_gpu_run_prediction_with_plan(self._ctx, _ptr(rows), len(rows), plan.p,
                                                       _res(rows), ctypes.byref(rep), _ptr(ceil_out),
                                                       _ptr(real_out), HOST))
        r = _report(rep, real_out, ceil_out, plan.sample_rows, plan.seed)
        r.plan = plan
        r.plan.sample_num = len(rows)
        return r

    def predict_sampled(self, seed: int, policy: SamplePolicy = SamplePolicy()) -> PredictionReport:
        """make_sample_plan + sampled_symbolic + collect_sample_stats +
        predict_reference + predict_proposed on the resident profile, one
        device call (the reference harness's predict task, bench.hpp:187-195);
        no per-row view."""
        n, _ = plan_size(self.a_rows, policy)
        rows = np.empty(n, np.int32)
        rep = Report()
        check(lib().spnnz_gpu_predict_sampled(self._ctx, seed, policy.fraction, policy.cap, ctypes.byref(rep),
                                              rows.ctypes.data))
        return _report(rep, None, None, rows, seed)

    # -- instrumentation
    def set_profiling(self, on: bool):
        check(lib().spnnz_gpu_set_profiling(self._ctx, int(on)))

    def last_timings(self):
        ms = (ctypes.c_double * 5)()
        n = ctypes.c_int64()
        check(lib().spnnz_gpu_last_timings(self._ctx, ms, ctypes.byref(n)))
        return dict(zip(("flop", "sample", "symbolic", "allreduce", "predict"), list(ms))), n.value

    def last_flop_kernel(self) -> str:
        """The kernel the last FLOP pass ran (instrumentation)."""
        return (lib().spnnz_gpu_last_flop_kernel(self._ctx) or b"").decode()

    def probe_flop_floor(self, reps: int = 10):
        """(stream_ms, gather_ms): the FLOP pass's A.col stream alone, and with
        its degree gathers, without the row logic (instrumentation)."""
        a, b = ctypes.c_double(), ctypes.c_double()
        check(lib().spnnz_gpu_probe_flop_floor(self._ctx, reps, ctypes.byref(a), ctypes.byref(b)))
        return a.value, b.value

    def synchronize(self):
        check(lib().spnnz_gpu_synchronize(self._ctx))

    def stream_handle(self) -> int:
        return lib().spnnz_gpu_stream(self._ctx)


def _rows_arg(rows):
    if isinstance(rows, np.ndarray) or not hasattr(rows, "data_ptr"):
        return np.ascontiguousarray(np.asarray(rows, dtype=np.int32))
    return rows


def _report(rep: Report, real, ceil, samples, seed) -> PredictionReport:
    plan = SamplePlan(samples, rep.sample_num, rep.p, seed)
    stats = SampleStats(rep.sampled_flop, rep.sampled_nnz, rep.sampled_cr)
    return PredictionReport(rep.z1_star, rep.z2_star, rep.predicted_cr, real, plan, stats,
                            rep.total_flop, ceil, rep.max_flop_row)


def plan_size(num_rows: int, policy: SamplePolicy):
    n, p = ctypes.c_int64(), ctypes.c_double()
    check(lib().spnnz_gpu_make_sample_plan(None, num_rows, 0, policy.fraction, policy.cap, None,
                                           HOST, ctypes.byref(n), ctypes.byref(p)))
    return n.value, p.value


# ------------------------------------------------- reference free functions
_default: Optional[Predictor] = None


def default_predictor() -> Predictor:
    global _default
    if _default is None:
        _default = Predictor(0)
    return _default


def compute_flop(a: CsrMatrix, b: CsrMatrix, threads: int = 0) -> FlopProfile:
    """spnnz::compute_flop (flop.hpp:25-60)."""
    P = default_predictor()
    P.ensure_loaded(a, b)
    return P.compute_flop()


_profile_ctx: Optional[Predictor] = None


def _profile_only(profile: FlopProfile) -> Predictor:
    """A context that never holds matrices: sampled_flop and the
    predict_row_structure views depend on the profile alone."""
    global _profile_ctx
    if _profile_ctx is None:
        _profile_ctx = Predictor(0)
    _profile_ctx.set_profile(profile)
    _profile_ctx.row_lo, _profile_ctx.row_hi = 0, len(profile.flop_per_row)
    return _profile_ctx


def sampled_flop(profile: FlopProfile, sample_rows) -> int:
    """spnnz::sampled_flop (flop.hpp:64-74)."""
    return _profile_only(profile).sampled_flop(sample_rows)


def make_sample_plan(num_rows: int, seed: int, policy: SamplePolicy = SamplePolicy()) -> SamplePlan:
    """spnnz::make_sample_plan (predict.hpp:34-56), drawn on the device."""
    return default_predictor().make_sample_plan(num_rows, seed, policy)


def exhaustive_plan(num_rows: int) -> SamplePlan:
    """spnnz::exhaustive_plan (predict.hpp:60-70)."""
    if num_rows < 1:
        raise ValueError("exhaustive_plan: M must be >= 1")
    return SamplePlan(np.arange(num_rows, dtype=np.int32), num_rows, 1.0, 0)


def _check_profile(a: CsrMatrix, b: CsrMatrix, profile: FlopProfile):
    if a.cols != b.rows:
        raise ValueError("symbolic: A.cols != B.rows")
    if len(profile.flop_per_row) != a.rows:
        raise ValueError("symbolic: profile does not match A")


def sampled_symbolic(a: CsrMatrix, b: CsrMatrix, profile: FlopProfile, sample_rows,
                     threads: int = 0) -> RowNnzResult:
    """spnnz::sampled_symbolic (symbolic.hpp:122-154)."""
    _check_profile(a, b, profile)
    P = default_predictor()
    P.ensure_loaded(a, b)
    P.set_profile(profile)
    return P.sampled_symbolic(sample_rows)


def exact_symbolic(a: CsrMatrix, b: CsrMatrix, profile: FlopProfile, threads: int = 0) -> RowNnzResult:
    """spnnz::exact_symbolic (symbolic.hpp:94-118)."""
    _check_profile(a, b, profile)
    P = default_predictor()
    P.ensure_loaded(a, b)
    P.set_profile(profile)
    return P.exact_symbolic()


def collect_sample_stats(profile: FlopProfile, plan: SamplePlan, sampled: RowNnzResult) -> SampleStats:
    """spnnz::collect_sample_stats (predict.hpp:81-91)."""
    f = sampled_flop(profile, plan.sample_rows)
    z = int(sampled.total_nnz)
    return SampleStats(f, z, lib().spnnz_sampled_cr(f, z))


def predict_reference(stats: SampleStats, plan: SamplePlan) -> float:
    """spnnz::predict_reference (predict.hpp:94-99)."""
    out = ctypes.c_double()
    check(lib().spnnz_predict_reference(int(stats.sampled_nnz), float(plan.p), ctypes.byref(out)))
    return out.value


def predict_proposed(stats: SampleStats, total_flop: int) -> ProposedPrediction:
    """spnnz::predict_proposed (predict.hpp:109-123)."""
    z2, cr = ctypes.c_double(), ctypes.c_double()
    check(lib().spnnz_predict_proposed(int(stats.sampled_flop), int(stats.sampled_nnz),
                                       int(total_flop), ctypes.byref(z2), ctypes.byref(cr)))
    return ProposedPrediction(z2.value, cr.value)


def predict_row_structure(profile: FlopProfile, predicted_cr: float) -> np.ndarray:
    """spnnz::predict_row_structure (predict.hpp:126-136)."""
    if not predicted_cr > 0.0:
        raise ValueError("predict_row_structure: predicted_cr must be positive")
    return _profile_only(profile).predict_row_structure(predicted_cr)


def predict_row_structure_ceil(profile: FlopProfile, predicted_cr: float) -> np.ndarray:
    """spnnz::predict_row_structure_ceil (predict.hpp:140-151)."""
    if not predicted_cr > 0.0:
        raise ValueError("predict_row_structure_ceil: predicted_cr must be positive")
    return _profile_only(profile).predict_row_structure_ceil(predicted_cr)


def error_report(z1_star: float, z2_star: float, f_star: int, exact_nnz: int, total_flop: int,
                 p: float) -> ErrorReport:
    """spnnz::error_report (predict.hpp:163-188)."""
    out = (ctypes.c_double * 4)()
    check(lib().spnnz_error_report(z1_star, z2_star, int(f_star), int(exact_nnz), int(total_flop),
                                   p, out))
    return ErrorReport(*list(out))


def run_prediction_with_plan(a: CsrMatrix, b: CsrMatrix, profile: FlopProfile, plan: SamplePlan,
                             threads: int = 0) -> PredictionReport:
    """spnnz::run_prediction_with_plan (predict.hpp:202-216)."""
    _check_profile(a, b, profile)
    P = default_predictor()
    P.ensure_loaded(a, b)
    return P.run_prediction_with_plan(plan, profile)


def run_prediction(a: CsrMatrix, b: CsrMatrix, seed: int, policy: SamplePolicy = SamplePolicy(),
                   threads: int = 0) -> PredictionReport:
    """spnnz::run_prediction (predict.hpp:220-226)."""
    P = default_predictor()
    P.ensure_loaded(a, b)
    return P.run_prediction(seed, policy)
