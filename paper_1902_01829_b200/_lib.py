"""ctypes binding of libh2b.so (include/h2b.h).

The library is built in-tree (``make -C paper_1902_01829_b200``); importing this
module without it raises immediately -- there is no CPU fallback.
"""
from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libh2b.so")

H2B_OK = 0
H2B_INVALID_ARGUMENT = 1
H2B_CUDA_ERROR = 2
H2B_OUT_OF_MEMORY = 3
H2B_UNSUPPORTED = 4
H2B_NO_DEVICE = 5
H2B_INTERNAL = 6
H2B_IO_ERROR = 7

PTR_AUTO, PTR_HOST, PTR_DEVICE, PTR_HOST_ASYNC = 0, 1, 2, 3
WS_XHAT, WS_YHAT, WS_XC, WS_PERM = 0, 1, 2, 3
CUDA_STREAM_LEGACY = 1  # cudaStreamLegacy


class H2bError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"[h2b status {code}] {msg}")
        self.code = code


class H2bInvalidArgument(H2bError, ValueError):
    """The reference's std::invalid_argument (include/h2kit/defs.hpp:20-22)."""


class H2bIOError(H2bError, OSError):
    """h2kit::IOError (io.hpp:19-21): container open / format / checksum errors."""


class H2bNoDevice(H2bError):
    pass


class MatrixDesc(C.Structure):
    _fields_ = [("n", C.c_int32), ("m", C.c_int32), ("depth", C.c_int32), ("symmetric", C.c_int32),
                ("perm", C.c_void_p), ("ranks", C.c_void_p), ("leaf", C.c_void_p),
                ("transfer", C.c_void_p), ("cpl_row_ptr", C.c_void_p), ("cpl_col_idx", C.c_void_p),
                ("cpl_values", C.c_void_p), ("dense_row_ptr", C.c_void_p),
                ("dense_col_idx", C.c_void_p), ("dense_values", C.c_void_p),
                ("col_ranks", C.c_void_p), ("col_leaf", C.c_void_p), ("col_transfer", C.c_void_p)]


class BuildInfo(C.Structure):
    _fields_ = [("dim", C.c_int32), ("seed", C.c_uint64), ("perturbation", C.c_double),
                ("ell", C.c_double), ("eta", C.c_double), ("grid_order", C.c_int32)]


class BuildConfig(C.Structure):
    _fields_ = [("dim", C.c_int32), ("n", C.c_int32), ("leaf_size", C.c_int32),
                ("grid_order", C.c_int32), ("eta", C.c_double), ("ell", C.c_double),
                ("perturbation", C.c_double), ("seed", C.c_uint64)]


class MatrixInfo(C.Structure):
    _fields_ = [("n", C.c_int32), ("m", C.c_int32), ("depth", C.c_int32), ("symmetric", C.c_int32),
                ("ranks", C.c_int32 * 32), ("cpl_blocks", C.c_int64 * 32),
                ("cpl_max_row", C.c_int32 * 32), ("dense_blocks", C.c_int64),
                ("dense_max_row", C.c_int32), ("footprint_bytes", C.c_uint64),
                ("device_bytes", C.c_uint64), ("hmv_flops", C.c_double),
                ("global_footprint_bytes", C.c_uint64), ("part_log2", C.c_int32),
                ("part_index", C.c_int32), ("col_ranks", C.c_int32 * 32)]


class CompressReport(C.Structure):
    _fields_ = [("old_ranks", C.c_int32 * 32), ("new_ranks", C.c_int32 * 32),
                ("bytes_before", C.c_uint64), ("bytes_after", C.c_uint64),
                ("frobenius_error", C.c_double), ("frobenius_norm", C.c_double),
                ("time_orthogonalize_ms", C.c_double), ("time_project_orth_ms", C.c_double),
                ("time_weights_ms", C.c_double), ("time_truncate_ms", C.c_double),
                ("time_project_trunc_ms", C.c_double), ("flops_orthogonalize", C.c_double),
                ("flops_project_orth", C.c_double), ("flops_weights", C.c_double),
                ("flops_truncate", C.c_double), ("flops_project_trunc", C.c_double)]


# h2b_comm (include/h2b.h): host communicator callbacks of h2b_part_compress
ALLGATHER_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_void_p, C.c_int64)
ALLREDUCE_I32_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.POINTER(C.c_int32), C.c_int)
ALLREDUCE_F64_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.POINTER(C.c_double), C.c_int)


class Comm(C.Structure):
    _fields_ = [("ctx", C.c_void_p), ("allgather", ALLGATHER_FN),
                ("allreduce_max_i32", ALLREDUCE_I32_FN), ("allreduce_sum_f64", ALLREDUCE_F64_FN)]


# h2b_dcomm (include/h2b.h): stream-ordered device all-gather of the
# partitioned mat-vec (h2b_part_hmv / h2b_part_hmv_multi)
DALLGATHER_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p)


class DComm(C.Structure):
    _fields_ = [("ctx", C.c_void_p), ("allgather", DALLGATHER_FN)]


Y_REPLICATED, Y_OWNED = 0, 1

# name -> (restype, argtypes)
_SIGS = {
    "h2b_last_error": (C.c_char_p, []),
    "h2b_version": (C.c_char_p, []),
    "h2b_device_count": (C.c_int, []),
    "h2b_release_cached_memory": (C.c_int, [C.c_int]),
    "h2b_matrix_create": (C.c_int, [C.POINTER(MatrixDesc), C.c_int, C.POINTER(C.c_void_p)]),
    "h2b_matrix_build": (C.c_int, [C.POINTER(BuildConfig), C.c_int, C.POINTER(C.c_void_p)]),
    "h2b_matrix_destroy": (C.c_int, [C.c_void_p]),
    "h2b_matrix_info_get": (C.c_int, [C.c_void_p, C.POINTER(MatrixInfo)]),
    "h2b_matrix_export": (C.c_int, [C.c_void_p] + [C.c_void_p] * 9),
    "h2b_matrix_export_col": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p]),
    "h2b_matrix_footprint": (C.c_uint64, [C.c_void_p]),
    "h2b_matrix_save": (C.c_int, [C.c_void_p, C.c_char_p, C.c_void_p]),
    "h2b_matrix_load": (C.c_int, [C.c_char_p, C.c_int, C.POINTER(C.c_void_p), C.c_void_p]),
    "h2b_crc32": (C.c_uint32, [C.c_void_p, C.c_uint64]),
    "h2b_hmv": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_double, C.c_double, C.c_int,
                          C.c_void_p]),
    "h2b_hmv_multi": (C.c_int, [C.c_void_p, C.c_int, C.c_void_p, C.c_int64, C.c_void_p, C.c_int64,
                                C.c_double, C.c_double, C.c_int, C.c_void_p]),
    "h2b_upsweep": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int]),
    "h2b_tree_multiply": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int]),
    "h2b_downsweep": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int]),
    "h2b_dense_mv": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_double, C.c_double, C.c_int]),
    "h2b_compress": (C.c_int, [C.c_void_p, C.c_double, C.POINTER(CompressReport)]),
    "h2b_part_compress": (C.c_int, [C.c_void_p, C.c_double, C.POINTER(Comm), C.POINTER(CompressReport)]),
    "h2b_orthogonalize": (C.c_int, [C.c_void_p, C.c_void_p]),
    "h2b_orthogonalize_col": (C.c_int, [C.c_void_p, C.c_void_p]),
    "h2b_last_hmv_timing": (C.c_int, [C.c_void_p, C.POINTER(C.c_double)]),
    "h2b_matrix_build_part": (C.c_int, [C.POINTER(BuildConfig), C.c_int, C.c_int, C.c_int,
                                        C.POINTER(C.c_void_p)]),
    "h2b_workspace": (C.c_int, [C.c_void_p, C.c_int, C.POINTER(C.c_void_p), C.POINTER(C.c_int64)]),
    "h2b_part_upsweep": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p]),
    "h2b_part_finish": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p]),
    "h2b_hmv_graph_create": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_double, C.c_double,
                                       C.POINTER(C.c_void_p)]),
    "h2b_hmv_graph_launch": (C.c_int, [C.c_void_p, C.c_void_p]),
    "h2b_hmv_graph_destroy": (C.c_int, [C.c_void_p]),
    "h2b_part_hmv": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_double, C.c_double, C.c_int,
                               C.POINTER(DComm), C.c_void_p]),
    "h2b_part_hmv_multi": (C.c_int, [C.c_void_p, C.c_int, C.c_void_p, C.c_int64, C.c_void_p, C.c_int64,
                                     C.c_double, C.c_double, C.c_int, C.POINTER(DComm), C.c_void_p]),
    "h2b_validate_sampled": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int, C.c_double, C.c_double,
                                       C.c_uint64, C.POINTER(C.c_double)]),
    "h2b_set_phase_timing": (C.c_int, [C.c_void_p, C.c_int]),
    "h2b_context_create": (C.c_int, [C.c_void_p, C.POINTER(C.c_void_p)]),
    "h2b_context_destroy": (C.c_int, [C.c_void_p]),
    "h2b_hmv_ctx": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_double, C.c_double,
                              C.c_int, C.c_void_p]),
}

EXPORTED_SYMBOLS = tuple(_SIGS)

_lib = None


def load(path: str = LIB_PATH):
    """Load libh2b.so (raises OSError if it has not been built)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise OSError(f"libh2b.so not built at {path}; run `make -C paper_1902_01829_b200` "
                      "(the product has no CPU fallback)")
    lib = C.CDLL(path)
    for name, (res, args) in _SIGS.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


def check(status: int):
    if status == H2B_OK:
        return
    msg = load().h2b_last_error().decode(errors="replace")
    if status == H2B_INVALID_ARGUMENT:
        raise H2bInvalidArgument(status, msg)
    if status == H2B_IO_ERROR:
        raise H2bIOError(status, msg)
    if status == H2B_NO_DEVICE:
        raise H2bNoDevice(status, msg)
    raise H2bError(status, msg)
