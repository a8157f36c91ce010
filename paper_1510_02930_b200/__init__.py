"""B200-native (sm_100a) TNRD/TRDPD Poisson-denoising inference (arXiv 1510.02930).

The product is libtnrd.so (C ABI, include/tnrd.h): fused CUDA stage kernels
plus the host stage loop, row-slab halo exchange (NCCL) and instrumentation.
This package is its thin ctypes binding; see DESIGN.md.
"""
from ._binding import *  # noqa: F401,F403
from ._binding import EXPORTED, LIB_PATH, TNRD, TNRDError, lib  # noqa: F401

__all__ = list(EXPORTED) + ["TNRD", "TNRDError", "lib", "LIB_PATH"]
