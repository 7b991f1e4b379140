"""Subtree-partitioned multi-GPU H^2 mat-vec.

One process per GPU (torch.distributed, NCCL).  Each rank builds only its
partition of the matrix in HBM (h2b_matrix_build_part: its top-level
subtree's leaves, basis nodes and coupling/dense block rows, plus the
replicated levels above the split), so an n = 2^22 matrix takes 1/P of the
memory per GPU.  One mat-vec (DistributedH2Matrix.hmv) is ONE library call,
h2b_part_hmv, which runs every step in libh2b.so on the caller's stream:

  1. owned leaves -> x^ of the owned nodes, up to level s (dataflow launch)
  2. pack the owned x^ of every level >= s into one buffer, ONE stream-ordered
     all-gather through the communicator (NCCL: ncclAllGather in place),
     unpack the other ranks' slices
  3. replicated top upsweep, coupling + dense rows of the owned subtree,
     downsweep, leaf expansion
  4. Y_REPLICATED: all-gather of the cluster-order y slices and the fused
     owner-row scatter y[perm] = a y_c + b y[perm]; Y_OWNED: each rank writes
     its own rows of y directly (no y collective)

No torch compute op runs on this path; torch.distributed only provides the
NCCL communicator (TorchComm).  A C++ host drives the same call with its own
ncclComm_t (examples/part_hmv_nccl.cpp).  x^ crossing the partition boundary
is < 1 % of the matrix bytes at n = 2^22.
"""
from __future__ import annotations

import ctypes as C

from . import _lib
from .partition import PartitionPlan


class _CudaView:
    """Zero-copy torch view of a libh2b device buffer."""

    def __init__(self, ptr: int, count: int, typestr: str, device: int):
        self.__cuda_array_interface__ = {"shape": (int(count),), "typestr": typestr,
                                         "data": (int(ptr), False), "version": 3, "strides": None}
        self.device = device


def device_view(handle, which: int, device: int):
    import torch
    ptr, cnt = C.c_void_p(), C.c_int64()
    _lib.check(_lib.load().h2b_workspace(handle, which, C.byref(ptr), C.byref(cnt)))
    typestr = "<i4" if which == _lib.WS_PERM else "<f8"
    if cnt.value == 0:
        return torch.empty(0, dtype=torch.int32 if which == _lib.WS_PERM else torch.float64,
                           device=f"cuda:{device}")
    return torch.as_tensor(_CudaView(ptr.value, cnt.value, typestr, device), device=f"cuda:{device}")


def torch_stream_handle() -> int:
    """The current torch stream as a cudaStream_t (legacy default stream = 0x1,
    since NULL means "the matrix's own stream" in the C-ABI)."""
    import torch
    h = torch.cuda.current_stream().cuda_stream
    return h if h else _lib.CUDA_STREAM_LEGACY


def _stream_of(handle: int):
    """torch stream object for a cudaStream_t handed back by the library."""
    import torch
    if handle in (0, _lib.CUDA_STREAM_LEGACY):
        return torch.cuda.default_stream()
    return torch.cuda.ExternalStream(handle)


def gather_xhat(plan: PartitionPlan, xhat, allgather):
    """All-gather the owned x^ slices of every level >= s, in place in the
    level-concatenated pool `xhat` (any tensor type the callback accepts)."""
    for l in plan.gather_levels():
        off, length, chunk = plan.level_slice(l)
        level = xhat[off:off + length]
        # the owned slice is copied out first: no reliance on in-place
        # all-gather semantics of the backend (the slice is <= 1/P of a level)
        allgather(level, level[plan.part * chunk:(plan.part + 1) * chunk].clone())


# ------------------------------------------------------------------ communicators
def _wrap(ptr: int, count: int, device):
    """Zero-copy torch view of `count` doubles at `ptr` (device memory when
    `device` is an int, host memory when None)."""
    import numpy as np
    import torch
    if device is None:
        arr = np.ctypeslib.as_array((C.c_double * int(count)).from_address(int(ptr)))
        return torch.from_numpy(arr)
    return torch.as_tensor(_CudaView(ptr, count, "<f8", device), device=f"cuda:{device}")


class Communicator:
    """Host side of h2b_comm (include/h2b.h) for h2b_part_compress: the library
    calls allgather / allreduce at fixed points of the compression, in the
    same order on every rank.  Subclasses implement the three collectives on
    torch tensors:
      allgather(buf)     buf holds nparts equal slices (device memory); slice
                         `part` is this rank's; fill the others in place
      allreduce_max(t)   element-wise, in place (host int32 tensor)
      allreduce_sum(t)   element-wise, in place (host float64 tensor)"""

    def __init__(self, nparts: int, part: int, device):
        self.nparts, self.part, self.device = nparts, part, device
        self._c = None

    def allgather(self, buf):
        raise NotImplementedError

    def allreduce_max(self, t):
        raise NotImplementedError

    def allreduce_sum(self, t):
        raise NotImplementedError

    def allgather_stream(self, buf, stream: int):
        """Stream-ordered form used by h2b_part_hmv: the all-gather must be
        complete, in stream order, before the stream's next operation.  Default:
        synchronise the stream, then the blocking allgather."""
        _stream_of(stream).synchronize()
        self.allgather(buf)

    def as_dcomm(self) -> "_lib.DComm":
        """ctypes h2b_dcomm (the partitioned mat-vec's device all-gather)."""

        def ag(ctx, ptr, count, stream):
            try:
                self.allgather_stream(_wrap(ptr, int(count) * self.nparts, self.device), int(stream or 0))
                return 0
            except Exception as e:  # noqa: BLE001  (cannot propagate through C)
                self.error = e
                return 1

        self.error = None
        self._dfn = _lib.DALLGATHER_FN(ag)
        self._dc = _lib.DComm(None, self._dfn)
        return self._dc

    def as_c(self) -> "_lib.Comm":
        """ctypes h2b_comm whose callbacks call this object (kept alive by it)."""
        import numpy as np
        import torch

        def ag(ctx, ptr, count):
            try:
                self.allgather(_wrap(ptr, int(count) * self.nparts, self.device))
                return 0
            except Exception as e:  # noqa: BLE001  (cannot propagate through C)
                self.error = e
                return 1

        def mx(ctx, v, n):
            try:
                t = torch.from_numpy(np.ctypeslib.as_array(v, shape=(int(n),)))
                self.allreduce_max(t)
                return 0
            except Exception as e:  # noqa: BLE001
                self.error = e
                return 1

        def sm(ctx, v, n):
            try:
                t = torch.from_numpy(np.ctypeslib.as_array(v, shape=(int(n),)))
                self.allreduce_sum(t)
                return 0
            except Exception as e:  # noqa: BLE001
                self.error = e
                return 1

        self.error = None
        self._fns = (_lib.ALLGATHER_FN(ag), _lib.ALLREDUCE_I32_FN(mx), _lib.ALLREDUCE_F64_FN(sm))
        self._c = _lib.Comm(None, *self._fns)
        return self._c


class TorchComm(Communicator):
    """torch.distributed collectives (NCCL over NVLink for the device
    all-gathers; the small host all-reduces go through the same group)."""

    def __init__(self, group=None, device=None):
        import torch.distributed as dist
        super().__init__(dist.get_world_size(group), dist.get_rank(group), device)
        self.group = group
        self.nccl = dist.get_backend(group) == "nccl"

    def allgather(self, buf):
        import torch
        import torch.distributed as dist
        chunk = buf.numel() // self.nparts
        mine = buf[self.part * chunk:(self.part + 1) * chunk].clone()
        if buf.is_cuda:
            dist.all_gather_into_tensor(buf, mine, group=self.group)
            torch.cuda.synchronize()
        else:
            parts = [torch.empty_like(mine) for _ in range(self.nparts)]
            dist.all_gather(parts, mine, group=self.group)
            buf.copy_(torch.cat(parts))

    def allgather_stream(self, buf, stream: int):
        """NCCL: enqueue the in-place all-gather on `stream` (no host sync);
        the rank's own slice of buf is the send buffer."""
        if not (self.nccl and buf.is_cuda):
            return super().allgather_stream(buf, stream)
        import torch
        import torch.distributed as dist
        chunk = buf.numel() // self.nparts
        with torch.cuda.stream(_stream_of(stream)):
            dist.all_gather_into_tensor(buf, buf.narrow(0, self.part * chunk, chunk), group=self.group)

    def _allreduce(self, t, op):
        import torch
        import torch.distributed as dist
        if self.nccl:
            d = t.to(f"cuda:{self.device}")
            dist.all_reduce(d, op=op, group=self.group)
            t.copy_(d.cpu())
        else:
            dist.all_reduce(t, op=op, group=self.group)

    def allreduce_max(self, t):
        import torch.distributed as dist
        self._allreduce(t, dist.ReduceOp.MAX)

    def allreduce_sum(self, t):
        import torch.distributed as dist
        self._allreduce(t, dist.ReduceOp.SUM)


class ThreadComm:
    """In-process communicator for P partitions driven by P threads (one GPU
    emulating P ranks): rank(part) returns the Communicator of one thread."""

    def __init__(self, nparts: int, device=0):
        import threading
        self.nparts, self.device = nparts, device
        self.barrier = threading.Barrier(nparts)
        self.slots = [None] * nparts

    def rank(self, part: int) -> Communicator:
        outer = self

        class _R(Communicator):
            def _exchange(self, value):
                outer.slots[self.part] = value
                outer.barrier.wait()
                vals = list(outer.slots)
                outer.barrier.wait()
                return vals

            def allgather(self, buf):
                import torch
                chunk = buf.numel() // outer.nparts
                vals = self._exchange(buf[self.part * chunk:(self.part + 1) * chunk].clone())
                for g, v in enumerate(vals):
                    if g != self.part:
                        buf[g * chunk:(g + 1) * chunk].copy_(v)
                if buf.is_cuda:
                    torch.cuda.synchronize()

            def allreduce_max(self, t):
                import torch
                vals = self._exchange(t.clone())
                t.copy_(torch.stack(vals).max(dim=0).values)

            def allreduce_sum(self, t):
                vals = self._exchange(t.clone())
                acc = vals[0].clone()
                for v in vals[1:]:  # fixed order: identical sums on every rank
                    acc += v
                t.copy_(acc)

        return _R(self.nparts, part, self.device)


class DistributedH2Matrix:
    """Rank-local partition of construct<double>(...) (construction.hpp:179-200)."""

    def __init__(self, dim: int, n: int, leaf_size: int = 64, grid_order: int | None = None,
                 eta: float = 2.0, ell: float | None = None, perturbation: float = 0.25,
                 seed: int = 1, group=None, device: int | None = None,
                 nparts: int | None = None, part: int | None = None):
        import torch
        import torch.distributed as dist
        self.group = group
        if nparts is None:
            nparts = dist.get_world_size(group)
            part = dist.get_rank(group)
        self.nparts, self.part = nparts, part
        self.device = torch.cuda.current_device() if device is None else device
        if grid_order is None:
            grid_order = 8 if dim == 2 else 4
        if ell is None:
            ell = 0.1 if dim == 2 else 0.2
        cfg = _lib.BuildConfig(dim, n, leaf_size, grid_order, eta, ell, perturbation, seed)
        h = C.c_void_p()
        _lib.check(_lib.load().h2b_matrix_build_part(C.byref(cfg), self.device, nparts, part,
                                                     C.byref(h)))
        self._h = h
        inf = _lib.MatrixInfo()
        _lib.check(_lib.load().h2b_matrix_info_get(h, C.byref(inf)))
        self.info = inf
        q = inf.depth
        self.n, self.m, self.depth = inf.n, inf.m, q
        self.ranks = list(inf.ranks[:q + 1])
        self.plan = PartitionPlan(q, self.ranks, self.m, nparts, part)
        self.xhat = device_view(h, _lib.WS_XHAT, self.device)
        self.perm = device_view(h, _lib.WS_PERM, self.device).long()
        a, b = self.plan.y_slice()
        self.y_slice = torch.empty(b - a, dtype=torch.float64, device=f"cuda:{self.device}")
        self.y_cluster = torch.empty(self.n, dtype=torch.float64, device=f"cuda:{self.device}")

    @property
    def footprint_local(self) -> int:
        return int(self.info.footprint_bytes)

    @property
    def footprint_global(self) -> int:
        return int(self.info.global_footprint_bytes)

    def close(self):
        if self._h and self._h.value:
            _lib.check(_lib.load().h2b_matrix_destroy(self._h))
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _refresh(self):
        """Re-read shapes and workspace views (compression changes the ranks)."""
        import torch
        inf = _lib.MatrixInfo()
        _lib.check(_lib.load().h2b_matrix_info_get(self._h, C.byref(inf)))
        self.info = inf
        self.ranks = list(inf.ranks[:self.depth + 1])
        self.plan = PartitionPlan(self.depth, self.ranks, self.m, self.nparts, self.part)
        self.xhat = device_view(self._h, _lib.WS_XHAT, self.device)

    def compress(self, eps: float, comm: Communicator | None = None):
        """compress(A, eps) (compression.hpp:466-551) of the whole partitioned
        matrix: every rank calls it with the same eps; the collectives go through
        `comm` (default: TorchComm over this matrix's process group).  Returns
        the global CompressionReport (identical on every rank)."""
        from .api import report_from_c
        if comm is None:
            comm = TorchComm(self.group, self.device)
        rep = _lib.CompressReport()
        cs = comm.as_c()
        st = _lib.load().h2b_part_compress(self._h, float(eps), C.byref(cs), C.byref(rep))
        if st != _lib.H2B_OK and getattr(comm, "error", None) is not None:
            raise RuntimeError(f"communicator failed: {comm.error!r}")
        _lib.check(st)
        self._refresh()
        return report_from_c(rep, self.depth)

    def hmv(self, x, y=None, alpha: float = 1.0, beta: float = 0.0, comm: Communicator | None = None,
            y_mode: int = _lib.Y_REPLICATED, stream: int | None = None):
        """y <- alpha A x + beta y (hmv.hpp:175-188) with x, y full vectors in
        original order (CUDA float64).  One library call (h2b_part_hmv): the
        upsweep, the packed x^ all-gather (comm, default NCCL through this
        matrix's process group), the coupling / dense rows, the downsweep and the
        owner-row scatter all run in libh2b.so; y_mode Y_REPLICATED all-gathers
        the cluster-order y slices so every rank ends with all of y, Y_OWNED
        writes only this rank's rows."""
        import torch
        if comm is None:
            comm = self._default_comm()
        if y is None:
            y = torch.zeros_like(x)
            beta = 0.0
        st = torch_stream_handle() if stream is None else stream
        dc = comm.as_dcomm()
        status = _lib.load().h2b_part_hmv(self._h, C.c_void_p(x.data_ptr()), C.c_void_p(y.data_ptr()),
                                          float(alpha), float(beta), int(y_mode), C.byref(dc), C.c_void_p(st))
        self._check_comm(status, comm)
        return y

    def hmv_multi(self, X, Y=None, alpha: float = 1.0, beta: float = 0.0, comm: Communicator | None = None,
                  y_mode: int = _lib.Y_REPLICATED, stream: int | None = None):
        """Y <- alpha A X + beta Y for the columns of X (n x nvec, column-major:
        a (nvec, n) row-major CUDA tensor), 16 per pass on the FP64 tensor cores
        (h2b_part_hmv_multi)."""
        import torch
        if comm is None:
            comm = self._default_comm()
        if Y is None:
            Y = torch.zeros_like(X)
            beta = 0.0
        nvec, n = X.shape
        st = torch_stream_handle() if stream is None else stream
        dc = comm.as_dcomm()
        status = _lib.load().h2b_part_hmv_multi(self._h, int(nvec), C.c_void_p(X.data_ptr()), n,
                                                C.c_void_p(Y.data_ptr()), n, float(alpha), float(beta),
                                                int(y_mode), C.byref(dc), C.c_void_p(st))
        self._check_comm(status, comm)
        return Y

    def _default_comm(self):
        if not hasattr(self, "_comm"):
            self._comm = TorchComm(self.group, self.device)
        return self._comm

    @staticmethod
    def _check_comm(status, comm):
        if status != _lib.H2B_OK and getattr(comm, "error", None) is not None:
            raise RuntimeError(f"communicator failed: {comm.error!r}")
        _lib.check(status)
