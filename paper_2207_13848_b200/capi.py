"""ctypes binding of the C ABI in include/spnnz_gpu/capi.h.

Loads the in-tree ``_lib/libspnnz_gpu.so`` (built by ``make`` /
``__graft_entry__.build()``).  There is no fallback: if the library is missing
or a device call fails, a ``SpnnzError`` (or ``ValueError`` where the reference
throws ``std::invalid_argument``) is raised.
"""
from __future__ import annotations

import ctypes
import os
from ctypes import POINTER, c_double, c_int, c_int32, c_int64, c_size_t, c_uint64, c_void_p

_HERE = os.path.dirname(os.path.abspath(__file__))
# SPNNZ_GPU_LIB: an alternative build of the same library (A/B experiments,
# tools/variants.sh); the in-tree build otherwise.
LIB_PATH = os.environ.get("SPNNZ_GPU_LIB") or os.path.join(_HERE, "_lib", "libspnnz_gpu.so")
GEN_PATH = os.path.join(_HERE, "_lib", "libspnnz_gen.so")

OK, EINVAL, ECUDA, ENCCL, ENOMEM, ESTATE = 0, 1, 2, 3, 4, 5
HOST, DEVICE = 0, 1


class SpnnzError(RuntimeError):
    """Non-argument failure of the GPU path (CUDA, NCCL, memory, call order)."""

    def __init__(self, code: int, msg: str):
        super().__init__(f"[spnnz_gpu code {code}] {msg}")
        self.code = code


class CsrView(ctypes.Structure):
    _fields_ = [("rows", c_int32), ("cols", c_int32),
                ("rpt", POINTER(c_int64)), ("col", POINTER(c_int32))]


class Report(ctypes.Structure):
    """spnnz_report: the scalars of spnnz::PredictionReport (predict.hpp:192-200)."""
    _fields_ = [("total_flop", c_int64), ("max_flop_row", c_int64), ("sample_num", c_int64),
                ("p", c_double), ("seed", c_uint64), ("sampled_flop", c_int64),
                ("sampled_nnz", c_int64), ("sampled_cr", c_double), ("z1_star", c_double),
                ("z2_star", c_double), ("predicted_cr", c_double)]

    def as_dict(self) -> dict:
        return {k: getattr(self, k) for k, _ in self._fields_}


# name -> (restype, argtypes)
_SIGS = {
    "spnnz_gpu_abi_version": (c_int, []),
    "spnnz_gpu_last_error": (ctypes.c_char_p, []),
    "spnnz_gpu_nccl_unique_id": (c_int, [c_void_p]),
    "spnnz_gpu_create": (c_int, [c_int, c_int, c_int, c_void_p, POINTER(c_void_p)]),
    "spnnz_gpu_destroy": (c_int, [c_void_p]),
    "spnnz_gpu_synchronize": (c_int, [c_void_p]),
    "spnnz_gpu_host_alloc": (c_int, [c_size_t, POINTER(c_void_p)]),
    "spnnz_gpu_host_free": (c_int, [c_void_p]),
    "spnnz_gpu_partition_rows": (c_int, [c_void_p, c_int32, c_int, c_void_p]),
    "spnnz_gpu_load": (c_int, [c_void_p, POINTER(CsrView), POINTER(CsrView), c_int]),
    "spnnz_gpu_shard": (c_int, [c_void_p, POINTER(c_int32), POINTER(c_int32), POINTER(c_int32)]),
    "spnnz_gpu_compute_flop": (c_int, [c_void_p, c_void_p, c_int, POINTER(c_int64),
                                       POINTER(c_int64)]),
    "spnnz_gpu_set_profile": (c_int, [c_void_p, c_void_p, c_int64, c_int, c_int64, c_int64]),
    "spnnz_gpu_sampled_flop": (c_int, [c_void_p, c_void_p, c_int64, c_int, POINTER(c_int64)]),
    "spnnz_gpu_make_sample_plan": (c_int, [c_void_p, c_int32, c_uint64, c_double, c_int64,
                                           c_void_p, c_int, POINTER(c_int64), POINTER(c_double)]),
    "spnnz_gpu_sampled_symbolic": (c_int, [c_void_p, c_void_p, c_int64, c_int, c_void_p,
                                           POINTER(c_int64)]),
    "spnnz_gpu_exact_symbolic": (c_int, [c_void_p, c_void_p, c_int, POINTER(c_int64)]),
    "spnnz_gpu_predict_row_structure": (c_int, [c_void_p, c_double, c_void_p, c_int]),
    "spnnz_gpu_predict_row_structure_ceil": (c_int, [c_void_p, c_double, c_void_p, c_int]),
    "spnnz_gpu_run_prediction": (c_int, [c_void_p, c_uint64, c_double, c_int64, POINTER(Report),
                                         c_void_p, c_void_p, c_void_p, c_int]),
    "spnnz_gpu_run_prediction_with_plan": (c_int, [c_void_p, c_void_p, c_int64, c_double, c_int,
                                                   POINTER(Report), c_void_p, c_void_p, c_int]),
    "spnnz_sampled_cr": (c_double, [c_int64, c_int64]),
    "spnnz_predict_reference": (c_int, [c_int64, c_double, POINTER(c_double)]),
    "spnnz_predict_proposed": (c_int, [c_int64, c_int64, c_int64, POINTER(c_double),
                                       POINTER(c_double)]),
    "spnnz_error_report": (c_int, [c_double, c_double, c_int64, c_int64, c_int64, c_double,
                                   c_void_p]),
    "spnnz_gpu_set_profiling": (c_int, [c_void_p, c_int]),
    "spnnz_gpu_last_timings": (c_int, [c_void_p, c_void_p, POINTER(c_int64)]),
    "spnnz_gpu_last_flop_kernel": (ctypes.c_char_p, [c_void_p]),
    "spnnz_gpu_stream": (c_void_p, [c_void_p]),
    "spnnz_gpu_set_input_stream": (c_int, [c_void_p, c_void_p]),
    "spnnz_gpu_predict_sampled": (c_int, [c_void_p, c_uint64, c_double, c_int64, POINTER(Report), c_void_p]),
    "spnnz_gpu_probe_flop_floor": (c_int, [c_void_p, c_int, POINTER(c_double), POINTER(c_double)]),
    "spnnz_gpu_check_guards": (c_int, [POINTER(c_int64), POINTER(c_int64)]),
}

EXPORTED = tuple(_SIGS)

_lib = None


def _default_nccl() -> None:
    """Points SPNNZ_NCCL_LIB at the pip-installed NCCL (the one torch loads),
    so a communicator created before `import torch` does not pin an older
    system libnccl.so.2 into the process."""
    if os.environ.get("SPNNZ_NCCL_LIB"):
        return
    try:
        import importlib.util
        spec = importlib.util.find_spec("nvidia.nccl")
    except (ImportError, ValueError):
        return
    for d in (spec.submodule_search_locations or []) if spec else []:
        p = os.path.join(d, "lib", "libnccl.so.2")
        if os.path.exists(p):
            os.environ["SPNNZ_NCCL_LIB"] = p
            return


def lib() -> ctypes.CDLL:
    """The loaded product library; raises if it was not built."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise SpnnzError(ECUDA, f"{LIB_PATH} not built (run `make` or "
                                    "__graft_entry__.build()); there is no CPU fallback")
        _default_nccl()
        L = ctypes.CDLL(LIB_PATH, mode=ctypes.RTLD_GLOBAL)
        for name, (res, args) in _SIGS.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib


def check(rc: int) -> None:
    if rc == OK:
        return
    msg = lib().spnnz_gpu_last_error().decode(errors="replace")
    if rc == EINVAL:
        raise ValueError(msg)
    raise SpnnzError(rc, msg)
