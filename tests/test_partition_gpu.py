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


# ---------------------------------------------------------------------------
# One-call partitioned mat-vec (h2b_part_hmv / h2b_part_hmv_multi): P ranks
# emulated by P threads on one GPU, each on its own stream, the x^ / y
# all-gathers through ThreadComm's stream-ordered h2b_dcomm callback (the
# same callback NCCL's in-place all-gather fills on a real node).
def run_ranks(parts, fn):
    import threading
    errs, out = [], [None] * len(parts)

    def body(g):
        try:
            torch.cuda.set_device(0)
            st = torch.cuda.Stream()
            with torch.cuda.stream(st):
                out[g] = fn(g, parts[g], st)
            st.synchronize()
        except Exception as e:  # noqa: BLE001
            errs.append(e)

    th = [threading.Thread(target=body, args=(g,)) for g in range(len(parts))]
    for t in th:
        t.start()
    for t in th:
        t.join(600)
    assert not errs, errs
    return out


def make_parts(dim, n, order, nparts):
    return [DistributedH2Matrix(dim, n, grid_order=order, nparts=nparts, part=g, device=0)
            for g in range(nparts)]


@pytest.mark.parametrize("dim,n,order,nparts", [(2, 1 << 12, 8, 2), (2, 1 << 14, 8, 4), (3, 1 << 14, 4, 8),
                                                (2, 1 << 12, 8, 1)])
@pytest.mark.parametrize("y_mode", [0, 1])
def test_part_hmv_one_call(gpu, dim, n, order, nparts, y_mode):
    from paper_1902_01829_b200.dist import ThreadComm
    A = h2.H2Matrix.construct(dim, n, grid_order=order)
    rng = np.random.default_rng(11)
    x, y0 = rng.random(n), rng.random(n)
    y_ref = h2.hmv(A, x, y0.copy(), 1.5, -0.25)
    parts = make_parts(dim, n, order, nparts)
    tc = ThreadComm(nparts, device=0)
    xt = torch.from_numpy(x).cuda()

    def fn(g, P, st):
        y = torch.from_numpy(y0).cuda()
        P.hmv(xt, y, 1.5, -0.25, comm=tc.rank(g), y_mode=y_mode, stream=st.cuda_stream)
        st.synchronize()
        return y.cpu().numpy()

    ys = run_ranks(parts, fn)
    perm = parts[0].perm.cpu().numpy()
    for g, y in enumerate(ys):
        if y_mode == 0 or nparts == 1:  # replicated: all of y on every rank
            assert rel_err(y, y_ref) <= 1e-12
        else:  # owned: this rank's rows are exact, the others untouched (y0)
            a, b = parts[g].plan.y_slice()
            mine = perm[a:b]
            assert rel_err(y[mine], y_ref[mine]) <= 1e-12
            rest = np.setdiff1d(np.arange(n), mine)
            assert np.array_equal(y[rest], y0[rest])


@pytest.mark.parametrize("nvec,nparts,y_mode", [(16, 4, 0), (20, 2, 0), (5, 8, 1), (16, 1, 0)])
def test_part_hmv_multi_one_call(gpu, nvec, nparts, y_mode):
    from paper_1902_01829_b200.dist import ThreadComm
    dim, n, order = (3, 1 << 14, 4) if nparts == 8 else (2, 1 << 14, 8)
    A = h2.H2Matrix.construct(dim, n, grid_order=order)
    rng = np.random.default_rng(12)
    X, Y0 = rng.random((nvec, n)), rng.random((nvec, n))
    Y_ref = h2.hmv_multi(A, X, 2.0, 0.5, Y0.copy())
    parts = make_parts(dim, n, order, nparts)
    tc = ThreadComm(nparts, device=0)
    Xt = torch.from_numpy(X).cuda()

    def fn(g, P, st):
        Y = torch.from_numpy(Y0).cuda()
        P.hmv_multi(Xt, Y, 2.0, 0.5, comm=tc.rank(g), y_mode=y_mode, stream=st.cuda_stream)
        st.synchronize()
        return Y.cpu().numpy()

    Ys = run_ranks(parts, fn)
    perm = parts[0].perm.cpu().numpy()
    for g, Y in enumerate(Ys):
        rows = np.arange(n)
        if y_mode == 1 and nparts > 1:
            a, b = parts[g].plan.y_slice()
            rows = perm[a:b]
        for v in range(nvec):
            assert rel_err(Y[v, rows], Y_ref[v, rows]) <= 1e-12, (g, v)


def test_part_hmv_c4_two_partitions(gpu, orc):
    """C4 (2D n = 2^22, k = 64) split in 2: each partition's coupling pool is
    3.2e9 elements (> 2^31), checked against the reference's y (golden)."""
    import json
    import os
    from conftest import GOLDEN_DIR
    from paper_1902_01829_b200.dist import ThreadComm
    with open(os.path.join(GOLDEN_DIR, "config", "C4.json")) as f:
        meta = json.load(f)
    arr = np.load(os.path.join(GOLDEN_DIR, "config", "C4.npz"))
    n = meta["n"]
    parts = make_parts(2, n, 8, 2)
    assert sum(P.footprint_local for P in parts) >= meta["footprint"]
    tc = ThreadComm(2, device=0)
    xt = torch.from_numpy(orc.random_vector(n, 1)).cuda()

    def fn(g, P, st):
        y = torch.zeros_like(xt)
        P.hmv(xt, y, comm=tc.rank(g), stream=st.cuda_stream)
        st.synchronize()
        return y.cpu().numpy()

    ys = run_ranks(parts, fn)
    for y in ys:
        assert rel_err(y[arr["idx"]], arr["y"]) <= 1e-12
        assert float(np.linalg.norm(y)) == pytest.approx(meta["y_norm2"], rel=1e-12)
    for P in parts:
        P.close()


def test_partitioned_compress_c3_two_partitions(gpu, orc):
    """C3 (3D n = 2^20, k = 64, eps 1e-6) compressed as 2 subtree partitions
    (each coupling pool ~2.8e9 elements, > 2^31) through the partitioned
    protocol: the global report equals the REFERENCE's C3 compression (golden
    from the reference on the GPU host), and the compressed partitions' mat-vec
    matches the reference's compressed operator at the golden indices."""
    import json
    import os
    from conftest import GOLDEN_DIR
    with open(os.path.join(GOLDEN_DIR, "config", "C3.json")) as f:
        meta = json.load(f)
    arr = np.load(os.path.join(GOLDEN_DIR, "config", "C3.npz"))
    g = meta["compress"]
    parts, reps = compress_partitioned(meta["dim"], meta["n"], meta["grid_order"], meta["eps"], 2)
    for r in reps:
        assert r.new_ranks == g["new_ranks"]
        assert r.bytes_before == int(g["bytes_before"]) and r.bytes_after == int(g["bytes_after"])
        assert r.frobenius_error == pytest.approx(g["frobenius_error"], rel=1e-6)
        assert r.total_flops() == pytest.approx(g["total_flops"], rel=1e-12)
    x = orc.random_vector(meta["n"], 1)
    y = partitioned_hmv(parts, x)
    assert rel_err(y[arr["idx"]], arr["yc"]) <= 10 * meta["eps"]
    for P in parts:
        P.close()
