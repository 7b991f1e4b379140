"""GPU: ranks and leaf sizes above 64 (2D grid_order 9-11, 3D grid_order 5,
leaf_size 128; construction.hpp:14-24 allows any).  The mat-vec path takes the
k_hmv_big.cu kernels (two row pairs per lane, two 64-column blocks per
transposed product); compression stays within 64 and says so.  Checked
against the real reference (oracle/_ref) built on the same points."""
import ctypes as C

import numpy as np
import pytest
import torch

from conftest import rel_err

import paper_1902_01829_b200 as h2
from paper_1902_01829_b200 import _lib

pytestmark = pytest.mark.gpu

CASES = [  # dim, n, leaf, order  (rank = order^dim)
    (2, 1 << 12, 64, 9),     # k = 81 > m = 64
    (2, 1 << 13, 128, 10),   # k = 100, leaf 128
    (2, 1 << 13, 128, 8),    # k = 64, leaf 128 (dense blocks 128 x 128)
    (3, 1 << 12, 128, 5),    # k = 125
]


@pytest.mark.parametrize("dim,n,leaf,order", CASES)
def test_big_hmv_matches_reference(gpu, ref, dim, n, leaf, order):
    R = ref.construct(dim, n, leaf_size=leaf, grid_order=order)
    A = h2.H2Matrix.construct(dim, n, leaf_size=leaf, grid_order=order)
    inf = A.info()
    assert max(inf.ranks) == order ** dim
    assert A.memory_footprint() == R.footprint()
    rng = np.random.default_rng(21)
    x, y0 = rng.random(n), rng.random(n)
    assert rel_err(h2.hmv(A, x), R.hmv(x)) <= 1e-12
    assert rel_err(h2.hmv(A, x, y0.copy(), 2.0, -0.5), R.hmv(x, y0.copy(), 2.0, -0.5)) <= 1e-12


@pytest.mark.parametrize("dim,n,leaf,order", CASES[:2])
def test_big_uploaded_matrix_and_phases(gpu, ref, dim, n, leaf, order):
    """The reference's own matrix uploaded (h2b_matrix_create), its phases
    (upsweep / tree_multiply / downsweep) and the multi-vector entry point."""
    R = ref.construct(dim, n, leaf_size=leaf, grid_order=order)
    A = h2.H2Matrix.from_host(R.to_host())
    rng = np.random.default_rng(22)
    x = rng.random(n)
    assert rel_err(h2.hmv(A, x), R.hmv(x)) <= 1e-12
    X = rng.random((3, n))
    Y = h2.hmv_multi(A, X)
    for v in range(3):
        assert rel_err(Y[v], R.hmv(X[v])) <= 1e-12


def test_big_partitioned(gpu, ref):
    from paper_1902_01829_b200.dist import DistributedH2Matrix, ThreadComm
    import threading
    dim, n, leaf, order = 2, 1 << 13, 128, 10
    R = ref.construct(dim, n, leaf_size=leaf, grid_order=order)
    x = np.random.default_rng(23).random(n)
    y_ref = R.hmv(x)
    parts = [DistributedH2Matrix(dim, n, leaf_size=leaf, grid_order=order, nparts=4, part=g, device=0)
             for g in range(4)]
    tc = ThreadComm(4, device=0)
    xt = torch.from_numpy(x).cuda()
    out, errs = [None] * 4, []

    def body(g):
        try:
            torch.cuda.set_device(0)
            st = torch.cuda.Stream()
            with torch.cuda.stream(st):
                y = torch.zeros_like(xt)
                parts[g].hmv(xt, y, comm=tc.rank(g), stream=st.cuda_stream)
                st.synchronize()
                out[g] = y.cpu().numpy()
        except Exception as e:  # noqa: BLE001
            errs.append(e)

    th = [threading.Thread(target=body, args=(g,)) for g in range(4)]
    for t in th:
        t.start()
    for t in th:
        t.join(300)
    assert not errs, errs
    for y in out:
        assert rel_err(y, y_ref) <= 1e-12


def test_big_compress_is_refused(gpu):
    A = h2.H2Matrix.construct(2, 1 << 12, leaf_size=128, grid_order=9)
    st = _lib.load().h2b_compress(A._h, C.c_double(1e-6), None)
    assert st == _lib.H2B_UNSUPPORTED
    assert b"compression kernels" in _lib.load().h2b_last_error()


def test_above_128_refused(gpu):
    with pytest.raises(Exception):
        h2.H2Matrix.construct(2, 1 << 12, grid_order=12)  # k = 144


def test_big_partitioned_multi(gpu, ref):
    """16-vector entry point on partitions with blocks > 64 (column by column)."""
    from paper_1902_01829_b200.dist import DistributedH2Matrix, ThreadComm
    import threading
    dim, n, leaf, order = 2, 1 << 12, 64, 9
    R = ref.construct(dim, n, leaf_size=leaf, grid_order=order)
    X = np.random.default_rng(24).random((3, n))
    parts = [DistributedH2Matrix(dim, n, leaf_size=leaf, grid_order=order, nparts=2, part=g, device=0)
             for g in range(2)]
    tc = ThreadComm(2, device=0)
    Xt = torch.from_numpy(X).cuda()
    out, errs = [None] * 2, []

    def body(g):
        try:
            torch.cuda.set_device(0)
            st = torch.cuda.Stream()
            with torch.cuda.stream(st):
                Y = torch.zeros_like(Xt)
                parts[g].hmv_multi(Xt, Y, comm=tc.rank(g), stream=st.cuda_stream)
                st.synchronize()
                out[g] = Y.cpu().numpy()
        except Exception as e:  # noqa: BLE001
            errs.append(e)

    th = [threading.Thread(target=body, args=(g,)) for g in range(2)]
    for t in th:
        t.start()
    for t in th:
        t.join(300)
    assert not errs, errs
    for Y in out:
        for v in range(3):
            assert rel_err(Y[v], R.hmv(X[v])) <= 1e-12
