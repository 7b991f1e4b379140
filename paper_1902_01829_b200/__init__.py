"""B200-native H^2-matrix hot path (arXiv 1902.01829): mat-vec + compression.

Public API mirrors the reference h2kit library (see api.py); the compute path
is libh2b.so (hand-written sm_100a CUDA behind the C-ABI in include/h2b.h).
"""
from .host import HostMatrix  # noqa: F401
from .api import (H2Matrix, HmvContext, HmvGraph, CompressionReport, compress, crc32, dense_mv, device_count,  # noqa: F401
                  downsweep, hmv, hmv_multi, orthogonalize_basis, release_cached_memory,
                  tree_multiply, upsweep, validate_sampled)
from ._lib import H2bError, H2bInvalidArgument, H2bIOError, H2bNoDevice  # noqa: F401

__all__ = ["HostMatrix", "H2Matrix", "CompressionReport", "compress", "dense_mv",
           "device_count", "downsweep", "hmv", "hmv_multi", "orthogonalize_basis", "release_cached_memory",
           "tree_multiply", "upsweep", "validate_sampled", "H2bError", "H2bInvalidArgument", "H2bIOError",
           "H2bNoDevice", "crc32"]
