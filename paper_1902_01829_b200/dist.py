"""Subtree-partitioned multi-GPU H^2 mat-vec.

One process per GPU (torch.distributed, NCCL).  Each rank builds only its
partition of the matrix in HBM (h2b_matrix_build_part: its top-level
subtree's leaves, basis nodes and coupling/dense block rows, plus the
replicated levels above the split), so an n = 2^22 matrix takes 1/P of the
memory per GPU.  One mat-vec (DistributedH2Matrix.hmv):

  1. h2b_part_upsweep   local leaves -> x^ of the owned nodes, up to level s
  2. all-gather x^      one NCCL all-gather per level >= s (the owned slice of a
                        level is contiguous in the level-concatenated pool;
                        in-place, nothing is copied)
  3. h2b_part_finish    replicated top upsweep, coupling + dense rows of the
                        owned subtree, downsweep, leaf expansion -> y slice
  4. all-gather y       cluster-order slices, then y[perm] = a y_c + b y[perm]

x̂ crossing the partition boundary is < 1 % of the matrix bytes at n = 2^22,
so the collectives are a small fraction of the step.
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


def gather_xhat(plan: PartitionPlan, xhat, allgather):
    """All-gather the owned x^ slices of every level >= s, in place in the
    level-concatenated pool `xhat` (any tensor type the callback accepts)."""
    for l in plan.gather_levels():
        off, length, chunk = plan.level_slice(l)
        level = xhat[off:off + length]
        # the owned slice is copied out first: no reliance on in-place
        # all-gather semantics of the backend (the slice is <= 1/P of a level)
        allgather(level, level[plan.part * chunk:(plan.part + 1) * chunk].clone())


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

    def gather_xhat(self, allgather):
        gather_xhat(self.plan, self.xhat, allgather)

    def hmv(self, x, y=None, alpha: float = 1.0, beta: float = 0.0, allgather=None):
        """y <- alpha A x + beta y for the full vectors x, y (original order,
        replicated on every rank, CUDA float64)."""
        import torch
        import torch.distributed as dist
        if allgather is None:
            def allgather(out, inp):
                dist.all_gather_into_tensor(out, inp, group=self.group)
        st = torch_stream_handle()
        lib = _lib.load()
        _lib.check(lib.h2b_part_upsweep(self._h, C.c_void_p(x.data_ptr()), C.c_void_p(st)))
        self.gather_xhat(allgather)
        _lib.check(lib.h2b_part_finish(self._h, C.c_void_p(self.y_slice.data_ptr()), C.c_void_p(st)))
        allgather(self.y_cluster, self.y_slice)
        if y is None:
            y = torch.empty_like(x)
            beta = 0.0
        if beta == 0.0:
            y[self.perm] = alpha * self.y_cluster
        else:
            y[self.perm] = alpha * self.y_cluster + beta * y[self.perm]
        return y
