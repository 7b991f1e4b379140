"""TEST INFRASTRUCTURE ONLY -- CPU oracles for the H^2 hot path.

Two backends with the same interface:

* ``restated()`` -- oracle/liboracle.so, the from-scratch CPU restatement
  (oracle/h2oracle.cpp), always buildable from this repo;
* ``reference()`` -- oracle/_ref/libh2ref.so, the UNMODIFIED reference h2kit
  compiled from /root/reference by oracle/Makefile (absent when the
  reference tree was never available to build it).

Only tests/, __graft_entry__.smoke() and bench.py's CPU legs may import this
package, and only as the checker / CPU baseline -- never as the product path.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

from paper_1902_01829_b200.host import HostMatrix

_HERE = os.path.dirname(os.path.abspath(__file__))
RESTATED_PATH = os.path.join(_HERE, "liboracle.so")
REF_PATH = os.path.join(_HERE, "_ref", "libh2ref.so")

_P = C.c_void_p
_I = C.c_int
_D = C.c_double


class OracleError(RuntimeError):
    pass


class OracleInvalidArgument(OracleError, ValueError):
    pass


class Backend:
    def __init__(self, path: str, prefix: str, name: str):
        if not os.path.exists(path):
            raise OSError(f"oracle library missing: {path} (run `make -C oracle`)")
        self.lib = C.CDLL(path)
        self.prefix = prefix
        self.name = name
        sig = {
            "last_error": (C.c_char_p, []),
            "points": (_I, [_I, _I, _D, C.c_uint64, _P]),
            "random_vector": (_I, [_I, C.c_uint64, _P]),
            "construct": (_I, [_I, _I, _I, _I, _D, _D, _D, C.c_uint64, C.POINTER(_P)]),
            "destroy": (None, [_P]),
            "clone": (_P, [_P]),
            "shape": (None, [_P, _P]),
            "layout": (None, [_P, _P, _P, _P, _P, _P]),
            "export": (None, [_P] * 10),
            "import": (_I, [_I, _I, _I] + [_P] * 10 + [C.POINTER(_P)]),
            "footprint": (C.c_uint64, [_P]),
            "flops_reset": (None, []),
            "flops_total": (_D, []),
            "hmv": (_I, [_P, _P, _P, _D, _D]),
            "upsweep": (_I, [_P, _P, _P]),
            "tree_multiply": (_I, [_P, _P, _P]),
            "downsweep": (_I, [_P, _P, _P]),
            "dense_mv": (_I, [_P, _P, _P, _D, _D]),
            "compress": (_I, [_P, _D, _P]),
            "orthogonalize": (_I, [_P, _P]),
            "orth_project_weights": (_I, [_P, _P]),
        }
        for k, (res, args) in sig.items():
            fn = getattr(self.lib, prefix + k)
            fn.restype = res
            fn.argtypes = args
        if prefix == "ref_":
            self.lib.ref_set_threads.argtypes = [_I]
            self.lib.ref_set_threads.restype = None
            self.lib.ref_max_threads.restype = _I
            self.lib.ref_hmv_reps.argtypes = [_P, _P, _P, _I]
            self.lib.ref_hmv_reps.restype = _I
            self.lib.ref_expand_dense.argtypes = [_P, _P]
            self.lib.ref_expand_dense.restype = _I
            self.lib.ref_validate_sampled.argtypes = [_P, _D, C.c_uint64, _P]
            self.lib.ref_validate_sampled.restype = _I
        else:
            self.lib.h2o_qr.argtypes = [_I, _I, _P, _P]
            self.lib.h2o_qr.restype = _I
            self.lib.h2o_svd.argtypes = [_I, _I, _P, _D, _P, _P]
            self.lib.h2o_svd.restype = _I
            self.lib.h2o_cluster.argtypes = [_I, _I, _I, _D, C.c_uint64, _P, _P, _P]
            self.lib.h2o_cluster.restype = _I

    def fn(self, name):
        return getattr(self.lib, self.prefix + name)

    def check(self, st):
        if st == 0:
            return
        msg = self.fn("last_error")().decode(errors="replace")
        if st == 1:
            raise OracleInvalidArgument(msg)
        raise OracleError(msg)

    # -- free functions ----------------------------------------------------
    def points(self, dim, n, pert=0.25, seed=1):
        out = np.zeros(n * dim, np.float64)
        self.check(self.fn("points")(dim, n, pert, seed, out.ctypes.data))
        return out.reshape(n, dim)

    def random_vector(self, n, seed):
        out = np.zeros(n, np.float64)
        self.check(self.fn("random_vector")(n, seed, out.ctypes.data))
        return out

    def construct(self, dim, n, leaf_size=64, grid_order=None, eta=2.0, ell=None,
                  perturbation=0.25, seed=1) -> "OracleMatrix":
        if grid_order is None:
            grid_order = 8 if dim == 2 else 4
        if ell is None:
            ell = 0.1 if dim == 2 else 0.2
        h = _P()
        self.check(self.fn("construct")(dim, n, leaf_size, grid_order, eta, ell, perturbation,
                                        seed, C.byref(h)))
        return OracleMatrix(self, h.value)

    def from_host(self, hm: HostMatrix) -> "OracleMatrix":
        h = _P()
        if not hm.symmetric:  # column basis: the reference backend only
            if self.prefix != "ref_":
                raise OracleError("non-symmetric matrices need the reference backend")
            arrs = [np.ascontiguousarray(a) for a in (
                hm.ranks.astype(np.int32), hm.col_ranks.astype(np.int32), hm.perm, hm.leaf,
                hm.transfer, hm.col_leaf, hm.col_transfer, hm.cpl_row_ptr, hm.cpl_col_idx,
                hm.cpl_values, hm.dense_row_ptr, hm.dense_col_idx, hm.dense_values)]
            f = self.lib.ref_import_ns
            f.argtypes = [C.c_int] * 3 + [C.c_void_p] * 13 + [C.POINTER(_P)]
            f.restype = C.c_int
            self.check(f(hm.n, hm.m, hm.depth, *[a.ctypes.data for a in arrs], C.byref(h)))
            return OracleMatrix(self, h.value)
        arrs = [np.ascontiguousarray(a) for a in (hm.ranks.astype(np.int32), hm.perm, hm.leaf,
                                                    hm.transfer, hm.cpl_row_ptr, hm.cpl_col_idx,
                                                    hm.cpl_values, hm.dense_row_ptr,
                                                    hm.dense_col_idx, hm.dense_values)]
        self.check(self.fn("import")(hm.n, hm.m, hm.depth, *[a.ctypes.data for a in arrs],
                                     C.byref(h)))
        return OracleMatrix(self, h.value)

    # -- container I/O (reference backend only: h2kit::save / load, crc32) --
    def load(self, path: str) -> "OracleMatrix":
        h = _P()
        self.lib.ref_load.argtypes = [C.c_char_p, C.POINTER(_P)]
        self.check(self.lib.ref_load(path.encode(), C.byref(h)))
        return OracleMatrix(self, h.value)

    def crc32(self, data: bytes) -> int:
        self.lib.ref_crc32.argtypes = [C.c_char_p, C.c_uint64]
        self.lib.ref_crc32.restype = C.c_uint32
        return int(self.lib.ref_crc32(data, len(data)))

    def set_threads(self, n):
        if self.prefix == "ref_":
            self.lib.ref_set_threads(int(n))

    def max_threads(self):
        return self.lib.ref_max_threads() if self.prefix == "ref_" else 1


class OracleMatrix:
    def __init__(self, be: Backend, h: int):
        self.be = be
        self.h = _P(h)

    def __del__(self):
        try:
            if self.h and self.h.value:
                self.be.fn("destroy")(self.h)
        except Exception:
            pass

    def save(self, path: str):
        self.be.lib.ref_save.argtypes = [_P, C.c_char_p]
        self.be.check(self.be.lib.ref_save(self.h, path.encode()))

    def clone(self) -> "OracleMatrix":
        return OracleMatrix(self.be, self.be.fn("clone")(self.h))

    def shape(self):
        out = np.zeros(4, np.int32)
        self.be.fn("shape")(self.h, out.ctypes.data)
        return [int(v) for v in out]

    def layout(self):
        n, m, q, _ = self.shape()
        ranks = np.zeros(q + 1, np.int32)
        nb = np.zeros(q + 1, np.int64)
        br = np.zeros(q + 1, np.int32)
        bc = np.zeros(q + 1, np.int32)
        nd = np.zeros(1, np.int64)
        self.be.fn("layout")(self.h, ranks.ctypes.data, nb.ctypes.data, br.ctypes.data,
                             bc.ctypes.data, nd.ctypes.data)
        return ranks, nb, int(nd[0])

    def to_host(self) -> HostMatrix:
        n, m, q, sym = self.shape()
        ranks, nb, nd = self.layout()
        cr = None
        if not sym:
            cr = np.zeros(q + 1, np.int32)
            self.be.lib.ref_col_ranks.argtypes = [_P, C.c_void_p]
            self.be.lib.ref_col_ranks(self.h, cr.ctypes.data)
        hm = HostMatrix.empty(n, m, q, ranks, nb, nd, cr)
        self.be.fn("export")(self.h, *[a.ctypes.data for a in hm.arrays()])
        if not sym:
            self.be.lib.ref_export_col.argtypes = [_P, C.c_void_p, C.c_void_p]
            self.be.lib.ref_export_col(self.h, hm.col_leaf.ctypes.data, hm.col_transfer.ctypes.data)
        return hm

    @property
    def n(self):
        return self.shape()[0]

    def footprint(self) -> int:
        return int(self.be.fn("footprint")(self.h))

    def vec_size(self):
        ranks, _, _ = self.layout()
        return int(sum((1 << l) * int(r) for l, r in enumerate(ranks)))

    def col_vec_size(self):
        n, m, q, sym = self.shape()
        if sym:
            return self.vec_size()
        cr = np.zeros(q + 1, np.int32)
        self.be.lib.ref_col_ranks.argtypes = [_P, C.c_void_p]
        self.be.lib.ref_col_ranks(self.h, cr.ctypes.data)
        return int(sum((1 << l) * int(r) for l, r in enumerate(cr)))

    def hmv(self, x, y=None, alpha=1.0, beta=0.0):
        x = np.ascontiguousarray(x, dtype=np.float64)
        y = np.zeros_like(x) if y is None else np.array(y, dtype=np.float64, copy=True)
        self.be.check(self.be.fn("hmv")(self.h, x.ctypes.data, y.ctypes.data, alpha, beta))
        return y

    def hmv_flops(self, x=None):
        if x is None:
            x = np.ones(self.n)
        self.be.fn("flops_reset")()
        self.hmv(x)
        return float(self.be.fn("flops_total")())

    def upsweep(self, xc):
        xc = np.ascontiguousarray(xc, dtype=np.float64)
        out = np.zeros(self.col_vec_size(), np.float64)
        self.be.check(self.be.fn("upsweep")(self.h, xc.ctypes.data, out.ctypes.data))
        return out

    def tree_multiply(self, xh):
        xh = np.ascontiguousarray(xh, dtype=np.float64)
        out = np.zeros(self.vec_size(), np.float64)
        self.be.check(self.be.fn("tree_multiply")(self.h, xh.ctypes.data, out.ctypes.data))
        return out

    def downsweep(self, yh, yc):
        yh = np.ascontiguousarray(yh, dtype=np.float64)
        yc = np.array(yc, dtype=np.float64, copy=True)
        self.be.check(self.be.fn("downsweep")(self.h, yh.ctypes.data, yc.ctypes.data))
        return yc

    def dense_mv(self, xc):
        xc = np.ascontiguousarray(xc, dtype=np.float64)
        out = np.zeros_like(xc)
        self.be.check(self.be.fn("dense_mv")(self.h, xc.ctypes.data, out.ctypes.data, 1.0, 0.0))
        return out

    def compress(self, eps):
        """In place. Returns the report dict (CompressionReport fields)."""
        r = np.zeros(14, np.float64)
        old = [int(v) for v in self.layout()[0]]
        self.be.check(self.be.fn("compress")(self.h, eps, r.ctypes.data))
        keys = ["frobenius_error", "frobenius_norm", "bytes_before", "bytes_after",
                "time_orthogonalize_ms", "time_project_orth_ms", "time_weights_ms",
                "time_truncate_ms", "time_project_trunc_ms", "flops_orthogonalize",
                "flops_project_orth", "flops_weights", "flops_truncate", "flops_project_trunc"]
        rep = dict(zip(keys, (float(v) for v in r)))
        rep["old_ranks"] = old
        rep["new_ranks"] = [int(v) for v in self.layout()[0]]
        rep["total_flops"] = sum(rep[k] for k in keys[9:])
        rep["total_ms"] = sum(rep[k] for k in keys[4:9])
        return rep

    def orthogonalize(self):
        ranks, _, _ = self.layout()
        out = np.zeros(int(sum((1 << l) * int(r) ** 2 for l, r in enumerate(ranks))), np.float64)
        self.be.check(self.be.fn("orthogonalize")(self.h, out.ctypes.data))
        return out

    def orthogonalize_col(self):
        """orthogonalize_basis(A.col_basis()) (reference backend only)."""
        n, m, q, sym = self.shape()
        cr = np.zeros(q + 1, np.int32)
        self.be.lib.ref_col_ranks.argtypes = [_P, C.c_void_p]
        self.be.lib.ref_col_ranks(self.h, cr.ctypes.data)
        out = np.zeros(int(sum((1 << l) * int(r) ** 2 for l, r in enumerate(cr))), np.float64)
        f = self.be.lib.ref_orthogonalize_col
        f.argtypes, f.restype = [_P, _P], _I
        self.be.check(f(self.h, out.ctypes.data))
        return out

    def orth_project_weights(self):
        ranks, _, _ = self.layout()
        out = np.zeros(int(sum((1 << l) * int(r) ** 2 for l, r in enumerate(ranks))), np.float64)
        self.be.check(self.be.fn("orth_project_weights")(self.h, out.ctypes.data))
        return out

    def expand_dense(self):
        n = self.n
        out = np.zeros(n * n, np.float64)
        self.be.check(self.be.lib.ref_expand_dense(self.h, out.ctypes.data))
        return out.reshape(n, n).T  # column-major -> D[i, j]


_cache = {}


def restated() -> Backend:
    if "o" not in _cache:
        _cache["o"] = Backend(RESTATED_PATH, "h2o_", "restated")
    return _cache["o"]


def reference_available() -> bool:
    return os.path.exists(REF_PATH)


def reference() -> Backend:
    if "r" not in _cache:
        _cache["r"] = Backend(REF_PATH, "ref_", "reference")
    return _cache["r"]


def best() -> Backend:
    """The real reference when built, else the restatement."""
    return reference() if reference_available() else restated()
