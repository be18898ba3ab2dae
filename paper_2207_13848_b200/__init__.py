"""B200-native SpGEMM output-structure predictor (arXiv 2207.13848).

GPU drop-in for the reference's ``spnnz`` predictor API: per-row FLOP,
seeded row sample, sampled symbolic NNZ, compression ratio and predicted
per-row NNZ, all as sm_100a CUDA kernels behind the C ABI in
``include/spnnz_gpu/capi.h``.  ``spnnz`` mirrors the reference functions,
``gen`` builds the benchmark configurations.
"""
from . import capi  # noqa: F401

__all__ = ["capi", "spnnz", "gen"]
