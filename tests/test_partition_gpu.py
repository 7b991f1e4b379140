"""GPU: the subtree-partitioned mat-vec path (h2b_matrix_build_part,
h2b_part_upsweep / h2b_part_finish) against the single-GPU mat-vec.  P
partitions are emulated on one device; the all-gathers are slice copies."""
import numpy as np
import pytest
import torch

from conftest import rel_err

import paper_1902_01829_b200 as h2
from paper_1902_01829_b200.dist import DistributedH2Matrix

pytestmark = pytest.mark.gpu


def run_partitioned(dim, n, order, nparts, x, alpha=1.0, beta=0.0, y0=None):
    parts = [DistributedH2Matrix(dim, n, grid_order=order, nparts=nparts, part=g, device=0)
             for g in range(nparts)]
    xt = torch.from_numpy(x).cuda()
    st = torch.cuda.current_stream().cuda_stream or 1
    import ctypes as C
    from paper_1902_01829_b200 import _lib
    lib = _lib.load()
    for P in parts:
        _lib.check(lib.h2b_part_upsweep(P._h, C.c_void_p(xt.data_ptr()), C.c_void_p(st)))
    # emulated all-gather of x^ levels >= s: copy every owner's slice to every rank
    plan = parts[0].plan
    for l in plan.gather_levels():
        off, length, chunk = plan.level_slice(l)
        for src in parts:
            piece = src.xhat[off + src.part * chunk: off + (src.part + 1) * chunk].clone()
            for dst in parts:
                dst.xhat[off + src.part * chunk: off + (src.part + 1) * chunk] = piece
    ycl = torch.empty(n, dtype=torch.float64, device="cuda")
    for P in parts:
        _lib.check(lib.h2b_part_finish(P._h, C.c_void_p(P.y_slice.data_ptr()), C.c_void_p(st)))
        a, b = P.plan.y_slice()
        ycl[a:b] = P.y_slice
    y = torch.zeros(n, dtype=torch.float64, device="cuda") if y0 is None else torch.from_numpy(y0).cuda()
    perm = parts[0].perm
    y[perm] = alpha * ycl + (beta * y[perm] if beta != 0.0 else 0.0)
    torch.cuda.synchronize()
    fp = [P.footprint_local for P in parts]
    return y.cpu().numpy(), fp, parts[0].footprint_global


@pytest.mark.parametrize("dim,n,order,nparts", [(2, 1 << 12, 8, 2), (2, 1 << 14, 8, 4),
                                                (3, 1 << 14, 4, 8), (2, 1 << 16, 6, 8),
                                                (2, 1 << 12, 8, 1)])
def test_partitioned_matches_single(gpu, dim, n, order, nparts):
    A = h2.H2Matrix.construct(dim, n, grid_order=order)
    x = np.random.default_rng(4).random(n)
    y_ref = h2.hmv(A, x)
    y, fp, fpg = run_partitioned(dim, n, order, nparts, x)
    assert rel_err(y, y_ref) <= 1e-12
    assert fpg == A.memory_footprint()
    # partitions together hold the matrix once plus the replicated top levels
    assert sum(fp) >= fpg and sum(fp) <= fpg * 1.05 + 1e6


def test_partitioned_alpha_beta(gpu):
    n = 1 << 13
    A = h2.H2Matrix.construct(2, n)
    rng = np.random.default_rng(6)
    x, y0 = rng.random(n), rng.random(n)
    y_ref = h2.hmv(A, x, y0.copy(), 2.0, -0.5)
    y, _, _ = run_partitioned(2, n, 8, 4, x, 2.0, -0.5, y0.copy())
    assert rel_err(y, y_ref) <= 1e-12


def test_partition_handles_refuse_whole_matrix_calls(gpu):
    P = DistributedH2Matrix(2, 1 << 12, nparts=2, part=1, device=0)
    import ctypes as C
    from paper_1902_01829_b200 import _lib
    x = np.zeros(1 << 12)
    st = _lib.load().h2b_hmv(P._h, x.ctypes.data, x.ctypes.data, 1.0, 0.0, 1, None)
    assert st == _lib.H2B_INVALID_ARGUMENT
    with pytest.raises(h2.H2bInvalidArgument):
        DistributedH2Matrix(2, 1 << 12, nparts=3, part=0, device=0)
