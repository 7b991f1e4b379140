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


def compress_partitioned(dim, n, order, eps, nparts):
    """Compress P partition handles on one GPU, one thread per partition,
    collectives through ThreadComm (the same h2b_comm callbacks NCCL drives)."""
    import threading
    from paper_1902_01829_b200.dist import ThreadComm
    parts = [DistributedH2Matrix(dim, n, grid_order=order, nparts=nparts, part=g, device=0)
             for g in range(nparts)]
    tc = ThreadComm(nparts, device=0)
    reps, errs = [None] * nparts, []

    def run(g):
        try:
            torch.cuda.set_device(0)
            reps[g] = parts[g].compress(eps, tc.rank(g))
        except Exception as e:  # noqa: BLE001
            errs.append(e)
            tc.barrier.abort()

    th = [threading.Thread(target=run, args=(g,)) for g in range(nparts)]
    for t in th:
        t.start()
    for t in th:
        t.join(600)
    assert not errs, errs
    return parts, reps


def partitioned_hmv(parts, x):
    import ctypes as C
    from paper_1902_01829_b200 import _lib
    n = parts[0].n
    xt = torch.from_numpy(x).cuda()
    st = torch.cuda.current_stream().cuda_stream or 1
    lib = _lib.load()
    for P in parts:
        _lib.check(lib.h2b_part_upsweep(P._h, C.c_void_p(xt.data_ptr()), C.c_void_p(st)))
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
    y = torch.zeros(n, dtype=torch.float64, device="cuda")
    y[parts[0].perm] = ycl
    torch.cuda.synchronize()
    return y.cpu().numpy()


@pytest.mark.parametrize("dim,n,order,eps,nparts", [(2, 1 << 14, 8, 1e-7, 2), (3, 1 << 14, 4, 1e-6, 4),
                                                    (2, 1 << 16, 6, 1e-7, 8), (2, 1 << 12, 8, 1e-7, 1)])
def test_partitioned_compress_matches_single(gpu, dim, n, order, eps, nparts):
    """Subtree-partitioned compression (h2b_part_compress) == single-GPU compress:
    same truncated ranks per level, same discarded energy and footprints (global
    sums over the ranks), and the compressed partitions' mat-vec equals the
    single-GPU compressed mat-vec."""
    A = h2.H2Matrix.construct(dim, n, grid_order=order)
    ref = h2.compress(A, eps)
    x = np.random.default_rng(9).random(n)
    y_ref = h2.hmv(A, x)
    parts, reps = compress_partitioned(dim, n, order, eps, nparts)
    for r in reps:
        assert r.new_ranks == ref.new_ranks
        assert r.old_ranks == ref.old_ranks
        assert r.bytes_before == ref.bytes_before and r.bytes_after == ref.bytes_after
        assert abs(r.frobenius_norm - ref.frobenius_norm) <= 1e-12 * ref.frobenius_norm
        assert abs(r.frobenius_error - ref.frobenius_error) <= 1e-9 * max(ref.frobenius_error, 1e-300)
        assert abs(r.total_flops() - ref.total_flops()) <= 1e-9 * ref.total_flops()
    assert [P.ranks for P in parts] == [ref.new_ranks] * nparts
    assert all(P.footprint_global == ref.bytes_after for P in parts if nparts > 1)
    y = partitioned_hmv(parts, x)
    assert rel_err(y, y_ref) <= 1e-12
