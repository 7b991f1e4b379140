"""Python mirror of the reference h2kit operator API for the hot path.

Same names, argument meaning and error behaviour as the reference C++ templates
(include/h2kit/hmv.hpp, compression.hpp, construction.hpp), over the B200
C-ABI (include/h2b.h).  Invalid arguments raise ``H2bInvalidArgument`` (a
``ValueError``), the Python face of the reference's ``std::invalid_argument``.

Vectors may be numpy arrays (host; copies happen inside the call) or CUDA
tensors / any object exposing ``data_ptr()`` on the matrix's device.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import numpy as np

from . import _lib
from .host import HostMatrix


def _ptr(a):
    if a is None:
        return None, _lib.PTR_AUTO
    if isinstance(a, np.ndarray):
        if a.dtype not in (np.float64, np.int32) or not a.flags.c_contiguous:
            raise ValueError("arrays must be C-contiguous float64/int32")
        return a.ctypes.data, _lib.PTR_HOST
    if hasattr(a, "data_ptr"):
        return a.data_ptr(), (_lib.PTR_DEVICE if getattr(a, "is_cuda", False) else _lib.PTR_HOST)
    raise TypeError(f"unsupported array type {type(a)}")


def _bad(msg: str) -> Exception:
    """The Python face of the reference's std::invalid_argument."""
    return _lib.H2bInvalidArgument(_lib.H2B_INVALID_ARGUMENT, msg)


def _vec(a, n: int, name: str, writable: bool = False):
    """(pointer, kind) of a float64 vector of exactly n entries: a C-contiguous
    numpy array (host) or a contiguous torch tensor (host or CUDA).  The C side
    copies exactly n doubles from / to the pointer, so anything else is a
    ValueError here (the reference's std::invalid_argument), never an
    out-of-bounds access."""
    if isinstance(a, np.ndarray):
        if a.dtype != np.float64 or not a.flags.c_contiguous:
            raise _bad(f"{name}: must be a C-contiguous float64 array")
        if writable and not a.flags.writeable:
            raise _bad(f"{name}: must be writable")
        if a.size != n:
            raise _bad(f"{name}: has {a.size} entries, expected {n}")
        return a.ctypes.data, _lib.PTR_HOST
    if hasattr(a, "data_ptr"):
        import torch
        if a.dtype != torch.float64 or not a.is_contiguous():
            raise _bad(f"{name}: must be a contiguous float64 tensor")
        if a.numel() != n:
            raise _bad(f"{name}: has {a.numel()} entries, expected {n}")
        return a.data_ptr(), (_lib.PTR_DEVICE if a.is_cuda else _lib.PTR_HOST)
    raise TypeError(f"{name}: unsupported array type {type(a)}")


def _host_vec(a, n: int, name: str) -> np.ndarray:
    """A float64 host copy-or-view of exactly n entries (input vectors)."""
    a = np.ascontiguousarray(a, dtype=np.float64)
    if a.size != n:
        raise _bad(f"{name}: has {a.size} entries, expected {n}")
    return a


@dataclass
class MatrixInfo:
    n: int
    m: int
    depth: int
    ranks: list
    cpl_blocks: list
    cpl_max_row: list
    dense_blocks: int
    dense_max_row: int
    footprint_bytes: int
    device_bytes: int
    hmv_flops: float
    symmetric: int = 1
    col_ranks: list = None  # column basis ranks (== ranks when symmetric)


class H2Matrix:
    """Device-resident H^2 matrix (the reference's H2Matrix<double>,
    h2_matrix.hpp:62-80, plus its HmvContext workspace, hmv.hpp:161-172);
    symmetric, or with a separate column basis (from_host / load)."""

    def __init__(self, handle: int, device: int):
        self._h = C.c_void_p(handle)
        self.device = device

    # -- construction -------------------------------------------------
    @classmethod
    def from_host(cls, hm: HostMatrix, device: int = 0) -> "H2Matrix":
        lib = _lib.load()
        hm.validate()
        keep = [np.ascontiguousarray(a) for a in (hm.perm, hm.ranks.astype(np.int32), hm.leaf,
                                                    hm.transfer, hm.cpl_row_ptr, hm.cpl_col_idx,
                                                    hm.cpl_values, hm.dense_row_ptr,
                                                    hm.dense_col_idx, hm.dense_values)]
        col = [None, None, None]
        if not hm.symmetric:  # column basis V / F (h2_matrix.hpp:69)
            keep += [np.ascontiguousarray(hm.col_ranks.astype(np.int32)),
                     np.ascontiguousarray(hm.col_leaf), np.ascontiguousarray(hm.col_transfer)]
            col = [a.ctypes.data for a in keep[-3:]]
        d = _lib.MatrixDesc(hm.n, hm.m, hm.depth, 1 if hm.symmetric else 0,
                            *[a.ctypes.data for a in keep[:10]], *col)
        out = C.c_void_p()
        _lib.check(lib.h2b_matrix_create(C.byref(d), device, C.byref(out)))
        return cls(out.value, device)

    @classmethod
    def construct(cls, dim: int, n: int, leaf_size: int = 64, grid_order: int | None = None,
                  eta: float = 2.0, ell: float | None = None, perturbation: float = 0.25,
                  seed: int = 1, device: int = 0) -> "H2Matrix":
        """construct<double>(generate_perturbed_grid(dim, n, perturbation, seed),
        KernelSpec{ell}, ConstructionConfig{leaf_size, grid_order, eta}) built on the
        device (construction.hpp:179-200; defaults of tools/h2kit.cpp:55-58)."""
        lib = _lib.load()
        if grid_order is None:
            grid_order = 8 if dim == 2 else 4
        if ell is None:
            ell = 0.1 if dim == 2 else 0.2
        cfg = _lib.BuildConfig(dim, n, leaf_size, grid_order, eta, ell, perturbation, seed)
        out = C.c_void_p()
        _lib.check(lib.h2b_matrix_build(C.byref(cfg), device, C.byref(out)))
        A = cls(out.value, device)
        A.build_config = dict(dim=dim, n=n, leaf_size=leaf_size, grid_order=grid_order, eta=eta,
                              ell=ell, perturbation=perturbation, seed=seed)
        return A

    @classmethod
    def load(cls, path: str, device: int = 0) -> "H2Matrix":
        """h2kit::load<double>(path) (io.hpp:247-282) straight into HBM; the stored
        BuildInfo is available as .build_info."""
        out = C.c_void_p()
        bi = _lib.BuildInfo()
        _lib.check(_lib.load().h2b_matrix_load(os.fspath(path).encode(), device, C.byref(out),
                                               C.byref(bi)))
        A = cls(out.value, device)
        A.build_info = {k: getattr(bi, k) for k, _ in bi._fields_}
        return A

    def save(self, path: str, build_info: dict | None = None):
        """h2kit::save(A, path) (io.hpp:183-229): the reference's container, byte for
        byte.  build_info overrides the stored BuildInfo (dim, seed, perturbation,
        ell, eta, grid_order)."""
        bi = None
        if build_info is not None:
            bi = _lib.BuildInfo(**build_info)
        _lib.check(_lib.load().h2b_matrix_save(self._h, os.fspath(path).encode(),
                                               C.byref(bi) if bi is not None else None))

    def close(self):
        if self._h and self._h.value:
            _lib.check(_lib.load().h2b_matrix_destroy(self._h))
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    # -- queries --------------------------------------------------------
    def info(self) -> MatrixInfo:
        inf = _lib.MatrixInfo()
        _lib.check(_lib.load().h2b_matrix_info_get(self._h, C.byref(inf)))
        q = inf.depth
        return MatrixInfo(inf.n, inf.m, q, list(inf.ranks[:q + 1]), list(inf.cpl_blocks[:q + 1]),
                          list(inf.cpl_max_row[:q + 1]), inf.dense_blocks, inf.dense_max_row,
                          inf.footprint_bytes, inf.device_bytes, inf.hmv_flops, inf.symmetric,
                          list(inf.col_ranks[:q + 1]))

    @property
    def n(self) -> int:
        if getattr(self, "_n", None) is None:
            self._n = self.info().n  # fixed for the handle's lifetime
        return self._n

    def memory_footprint(self) -> int:
        """memory_footprint(A).total() (h2_matrix.hpp:90-102)."""
        return int(_lib.load().h2b_matrix_footprint(self._h))

    def to_host(self) -> HostMatrix:
        inf = self.info()
        q = inf.depth
        sym = bool(inf.symmetric)
        hm = HostMatrix.empty(inf.n, inf.m, q, list(inf.ranks)[:q + 1], list(inf.cpl_blocks)[:q + 1],
                              inf.dense_blocks, None if sym else list(inf.col_ranks)[:q + 1])
        _lib.check(_lib.load().h2b_matrix_export(self._h, *[a.ctypes.data for a in hm.arrays()]))
        if not sym:
            _lib.check(_lib.load().h2b_matrix_export_col(self._h, hm.col_leaf.ctypes.data,
                                                         hm.col_transfer.ctypes.data))
        return hm

    def vec_size(self) -> int:
        """Length of y^ (row basis, LevelVectors::resize(A.row_basis))."""
        inf = self.info()
        return sum((1 << l) * r for l, r in enumerate(inf.ranks))

    def col_vec_size(self) -> int:
        """Length of x^ (LevelVectors::resize(A.col_basis()), hmv.hpp:166)."""
        inf = self.info()
        return sum((1 << l) * r for l, r in enumerate(inf.col_ranks))

    # -- hot path -------------------------------------------------------
    def set_phase_timing(self, on: bool = True):
        _lib.check(_lib.load().h2b_set_phase_timing(self._h, int(on)))

    def last_hmv_timing(self):
        buf = (C.c_double * 4)()
        _lib.check(_lib.load().h2b_last_hmv_timing(self._h, buf))
        return list(buf)


class HmvContext:
    """HmvContext<double> (hmv.hpp:159-172): a per-caller device workspace.
    Concurrent hmv calls on one matrix are safe with one context each (calls
    sharing a context are serialised in device order)."""

    def __init__(self, A: H2Matrix):
        out = C.c_void_p()
        _lib.check(_lib.load().h2b_context_create(A._h, C.byref(out)))
        self._c = out

    def close(self):
        if self._c and self._c.value:
            _lib.check(_lib.load().h2b_context_destroy(self._c))
            self._c = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class HmvGraph:
    """One mat-vec y <- alpha A x + beta y on fixed CUDA tensors x, y captured
    as a CUDA graph (h2b_hmv_graph_create) and replayed by launch(): for small
    matrices whose launch sequence costs as much as the work."""

    def __init__(self, A: H2Matrix, x, y, alpha: float = 1.0, beta: float = 0.0, ctx: HmvContext | None = None):
        px, kx = _vec(x, A.n, "hmv: x")
        py, ky = _vec(y, A.n, "hmv: y", writable=True)
        if not kx == ky == _lib.PTR_DEVICE:
            raise _bad("HmvGraph: x and y must be CUDA tensors")
        out = C.c_void_p()
        _lib.check(_lib.load().h2b_hmv_graph_create(A._h, ctx._c if ctx is not None else None, px, py,
                                                    float(alpha), float(beta), C.byref(out)))
        self._g, self._keep = out, (A, x, y, ctx)

    def launch(self, stream=None):
        if stream is None:
            from .dist import torch_stream_handle
            stream = torch_stream_handle()
        _lib.check(_lib.load().h2b_hmv_graph_launch(self._g, C.c_void_p(stream)))

    def close(self):
        if self._g and self._g.value:
            _lib.check(_lib.load().h2b_hmv_graph_destroy(self._g))
            self._g = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def hmv(A: H2Matrix, x, y=None, alpha: float = 1.0, beta: float = 0.0, stream=None,
        ctx: HmvContext | None = None, asynchronous: bool = False):
    """y <- alpha (A_D + A_LR) x + beta y (hmv.hpp:175-194). Returns y.
    asynchronous: x and y are PINNED host arrays; the copies and the mat-vec
    are enqueued on `stream` and the call returns at once (H2B_PTR_HOST_ASYNC):
    synchronise the stream before reading y.  With one HmvContext and one
    stream per in-flight call, the copies of one call overlap another's
    kernels."""
    if y is None:
        if isinstance(x, np.ndarray):
            y = np.zeros_like(x)
        else:
            import torch
            y = torch.zeros_like(x)
    n = A.n
    px, kx = _vec(x, n, "hmv: x")
    py, ky = _vec(y, n, "hmv: y", writable=True)
    kind = _lib.PTR_DEVICE if (kx == ky == _lib.PTR_DEVICE) else (
        _lib.PTR_HOST if (kx == ky == _lib.PTR_HOST) else _lib.PTR_AUTO)
    if asynchronous:
        if not kx == ky == _lib.PTR_HOST:
            raise _bad("hmv: asynchronous calls take pinned host arrays")
        kind = _lib.PTR_HOST_ASYNC
    if stream is None and _lib.PTR_DEVICE in (kx, ky):
        # device tensors: run on torch's current stream (NULL would mean the
        # matrix's own non-blocking stream, unordered with torch's work)
        from .dist import torch_stream_handle
        stream = torch_stream_handle()
    st = None if stream is None else C.c_void_p(stream)
    if ctx is None:
        _lib.check(_lib.load().h2b_hmv(A._h, px, py, float(alpha), float(beta), kind, st))
    else:
        _lib.check(_lib.load().h2b_hmv_ctx(A._h, ctx._c, px, py, float(alpha), float(beta), kind, st))
    return y


def hmv_multi(A: H2Matrix, X: np.ndarray, alpha: float = 1.0, beta: float = 0.0, Y=None):
    """Column-wise hmv of X (n x nvec, column-major i.e. X[:, v] contiguous when
    passed as a (nvec, n) C array)."""
    X = np.ascontiguousarray(X, dtype=np.float64)
    if X.ndim != 2 or X.shape[1] != A.n:
        raise _bad(f"hmv_multi: bad leading dimension (X must be (nvec, {A.n}))")
    nvec, n = X.shape
    if Y is None:
        Y = np.zeros_like(X)
    elif (not isinstance(Y, np.ndarray) or Y.dtype != np.float64 or Y.shape != X.shape
          or not Y.flags.c_contiguous or not Y.flags.writeable):
        raise _bad(f"hmv_multi: Y must be a writable C-contiguous float64 {X.shape} array")
    _lib.check(_lib.load().h2b_hmv_multi(A._h, nvec, X.ctypes.data, n, Y.ctypes.data, n,
                                         float(alpha), float(beta), _lib.PTR_HOST, None))
    return Y


def upsweep(A: H2Matrix, xc: np.ndarray) -> np.ndarray:
    """upsweep(V, xc, n, xhat) (hmv.hpp:79-111); xc in cluster order."""
    xc = _host_vec(xc, A.n, "upsweep: xc")
    out = np.zeros(A.col_vec_size(), np.float64)
    _lib.check(_lib.load().h2b_upsweep(A._h, xc.ctypes.data, out.ctypes.data, _lib.PTR_HOST))
    return out


def tree_multiply(A: H2Matrix, xhat: np.ndarray) -> np.ndarray:
    """tree_multiply(S, xhat, yhat) (hmv.hpp:114-125)."""
    xhat = _host_vec(xhat, A.col_vec_size(), "tree_multiply: xhat")
    out = np.zeros(A.vec_size(), np.float64)
    _lib.check(_lib.load().h2b_tree_multiply(A._h, xhat.ctypes.data, out.ctypes.data,
                                             _lib.PTR_HOST))
    return out


def downsweep(A: H2Matrix, yhat: np.ndarray, yc: np.ndarray) -> np.ndarray:
    """downsweep(U, yhat, yc, n) (hmv.hpp:129-157): returns yc + the U-expansion.
    Like the reference's LevelVectors, yhat is updated in place
    (y^l += E y^{l-1}) when it is a writable float64 array of the right size."""
    nv = A.vec_size()
    inplace = (isinstance(yhat, np.ndarray) and yhat.dtype == np.float64 and yhat.flags.c_contiguous
               and yhat.flags.writeable)
    yh = yhat if inplace else np.array(_host_vec(yhat, nv, "downsweep: yhat"), copy=True)
    if yh.size != nv:
        raise _bad(f"downsweep: yhat has {yh.size} entries, expected {nv}")
    yc = np.array(_host_vec(yc, A.n, "downsweep: yc"), copy=True)
    _lib.check(_lib.load().h2b_downsweep(A._h, yh.ctypes.data, yc.ctypes.data, _lib.PTR_HOST))
    return yc


def dense_mv(A: H2Matrix, xc: np.ndarray) -> np.ndarray:
    """block_sparse_mv(A.dense, xc, yc, 1, 0) (bsr.hpp:79-82)."""
    xc = _host_vec(xc, A.n, "dense_mv: xc")
    out = np.zeros_like(xc)
    _lib.check(_lib.load().h2b_dense_mv(A._h, xc.ctypes.data, out.ctypes.data, 1.0, 0.0,
                                        _lib.PTR_HOST))
    return out


@dataclass
class CompressionReport:
    """CompressionReport (compression.hpp:422-441)."""
    old_ranks: list
    new_ranks: list
    bytes_before: int
    bytes_after: int
    frobenius_error: float
    frobenius_norm: float
    time_orthogonalize_ms: float
    time_project_orth_ms: float
    time_weights_ms: float
    time_truncate_ms: float
    time_project_trunc_ms: float
    flops_orthogonalize: float
    flops_project_orth: float
    flops_weights: float
    flops_truncate: float
    flops_project_trunc: float

    def total_flops(self) -> float:
        return (self.flops_orthogonalize + self.flops_project_orth + self.flops_weights
                + self.flops_truncate + self.flops_project_trunc)

    def total_ms(self) -> float:
        return (self.time_orthogonalize_ms + self.time_project_orth_ms + self.time_weights_ms
                + self.time_truncate_ms + self.time_project_trunc_ms)


def report_from_c(rep, depth: int) -> CompressionReport:
    return CompressionReport(
        list(rep.old_ranks[:depth + 1]), list(rep.new_ranks[:depth + 1]), rep.bytes_before,
        rep.bytes_after, rep.frobenius_error, rep.frobenius_norm, rep.time_orthogonalize_ms,
        rep.time_project_orth_ms, rep.time_weights_ms, rep.time_truncate_ms,
        rep.time_project_trunc_ms, rep.flops_orthogonalize, rep.flops_project_orth,
        rep.flops_weights, rep.flops_truncate, rep.flops_project_trunc)


def compress(A: H2Matrix, eps: float) -> CompressionReport:
    """compress(A, eps) (compression.hpp:466-551), in place on the device."""
    depth = A.info().depth
    rep = _lib.CompressReport()
    _lib.check(_lib.load().h2b_compress(A._h, float(eps), C.byref(rep)))
    return report_from_c(rep, depth)


def orthogonalize_basis(A: H2Matrix, basis: str = "row") -> np.ndarray:
    """orthogonalize_basis(B) (compression.hpp:69-126) on B = A.row_basis
    (basis="row") or A.col_basis() (basis="col"; the same tree when A is
    symmetric): the basis is orthogonalized in place, the coupling is not
    projected.  Returns the projection tree (level-concatenated k_l x k_l
    blocks, k = that basis' ranks)."""
    if basis not in ("row", "col"):
        raise ValueError("basis must be 'row' or 'col'")
    inf = A.info()
    ranks = inf.ranks if basis == "row" else inf.col_ranks
    out = np.zeros(sum((1 << l) * int(ranks[l]) ** 2 for l in range(inf.depth + 1)), np.float64)
    lib = _lib.load()
    f = lib.h2b_orthogonalize if basis == "row" else lib.h2b_orthogonalize_col
    _lib.check(f(A._h, out.ctypes.data))
    return out


def validate_sampled(A: H2Matrix, fraction: float, seed: int = 1, points=None, dim: int = 0,
                     ell: float = 0.0) -> float:
    """validate_sampled(A, points, spec, fraction, seed) (validate.hpp:26-62) on the
    device; points default to the ones construct() generated on the device."""
    pp = None
    if points is not None:
        points = np.ascontiguousarray(points, dtype=np.float64)
        if points.ndim != 2 or points.shape[0] != A.n or points.shape[1] not in (2, 3):
            raise _bad(f"validate_sampled: points must be ({A.n}, 2|3)")
        dim = points.shape[1]
        pp = points.ctypes.data
    err = C.c_double()
    _lib.check(_lib.load().h2b_validate_sampled(A._h, pp, int(dim), float(ell), float(fraction),
                                                int(seed), C.byref(err)))
    return err.value


def device_count() -> int:
    return int(_lib.load().h2b_device_count())


def release_cached_memory(device: int = 0) -> None:
    """Hand the memory compress() cached in the device's stream-ordered pool back
    to the device (h2b_release_cached_memory)."""
    _lib.check(_lib.load().h2b_release_cached_memory(int(device)))


def crc32(data) -> int:
    """h2kit::crc32 (crc32.cpp:6-20) of a bytes-like object (host)."""
    mv = memoryview(data).cast("B")
    buf = (C.c_char * len(mv)).from_buffer_copy(mv) if mv.readonly else (C.c_char * len(mv)).from_buffer(mv)
    return int(_lib.load().h2b_crc32(C.addressof(buf), len(mv)))
