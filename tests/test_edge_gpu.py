"""GPU edge cases the reference handles: depth-0 and tiny trees,
empty coupling levels, rank-0 levels after compression, small leaves, 3D
grids with non-cubic sides, error parity."""
import numpy as np
import pytest

from conftest import rel_err

import paper_1902_01829_b200 as h2

pytestmark = pytest.mark.gpu
TOL = 1e-12


@pytest.mark.parametrize("dim,n,leaf,order", [
    (2, 64, 64, 8),      # depth 0: one leaf, dense only
    (2, 128, 64, 8),     # depth 1
    (2, 256, 32, 4),     # leaf 32
    (2, 1024, 16, 4),    # leaf 16 = rank 16
    (3, 512, 64, 3),     # 3D, rank 27 (odd)
    (3, 2048, 32, 2),    # 3D non-cubic sides, rank 8
    (2, 4096, 64, 7),    # rank 49 (odd)
    (2, 1 << 12, 64, 1), # rank 1
])
def test_shapes_match_oracle(gpu, orc, dim, n, leaf, order):
    O = orc.construct(dim, n, leaf_size=leaf, grid_order=order)
    A = h2.H2Matrix.construct(dim, n, leaf_size=leaf, grid_order=order)
    x = np.random.default_rng(n).random(n)
    assert rel_err(h2.hmv(A, x), O.hmv(x)) <= TOL
    U = h2.H2Matrix.from_host(O.to_host())
    assert rel_err(h2.hmv(U, x), O.hmv(x)) <= TOL
    if order ** dim <= leaf:  # orthogonalize requires m >= k (compression.hpp:80)
        ro = O.compress(1e-8)
        rg = h2.compress(U, 1e-8)
        assert all(abs(a - b) <= 1 for a, b in zip(rg.new_ranks, ro["new_ranks"]))
        assert rel_err(h2.hmv(U, x), O.hmv(x)) <= 1e-7


def test_leaf_rank_above_leaf_size_is_rejected(gpu, orc):
    # orthogonalize_basis: leaf_dim must be >= leaf rank (compression.hpp:80)
    A = h2.H2Matrix.construct(2, 1024, leaf_size=16, grid_order=8)
    with pytest.raises(h2.H2bInvalidArgument, match="leaf_dim must be >= leaf rank"):
        h2.compress(A, 1e-7)


def test_all_zero_rank_matrix(gpu, orc):
    # n = 256 compresses to ranks [0, 0, 0] (no coupling blocks): pure dense
    O = orc.construct(2, 256)
    A = h2.H2Matrix.from_host(O.to_host())
    rep = h2.compress(A, 1e-7)
    O.compress(1e-7)
    assert rep.new_ranks == [0, 0, 0]
    x = np.random.default_rng(1).random(256)
    assert rel_err(h2.hmv(A, x), O.hmv(x)) <= TOL
    # and a second compression of the rank-0 matrix is a no-op
    rep2 = h2.compress(A, 1e-7)
    assert rep2.new_ranks == [0, 0, 0] and rep2.frobenius_error == 0.0


def test_invalid_arguments(gpu):
    with pytest.raises(h2.H2bInvalidArgument, match="n must be leaf_size"):
        h2.H2Matrix.construct(2, 900)
    with pytest.raises(h2.H2bInvalidArgument, match="perturbation"):
        h2.H2Matrix.construct(2, 1024, perturbation=0.5)
    with pytest.raises(h2.H2bError):
        h2.H2Matrix.construct(2, 1024, grid_order=12)  # rank 144 > 128: outside the kernel envelope
    A = h2.H2Matrix.construct(2, 1024)
    with pytest.raises(h2.H2bInvalidArgument, match="leading dimension"):
        h2.hmv_multi(A, np.zeros((2, 512)))  # columns shorter than n


def test_validate_sampled_matches_reference(gpu, ref):
    """validate_sampled on the device == the reference's (acceptance c1:
    2D n=2^14 fraction 0.1 -> 3.44e-8; 3D -> 5.16e-5)."""
    for dim, n in [(2, 1 << 14), (3, 1 << 14)]:
        R = ref.construct(dim, n)
        import ctypes as C
        err_ref = C.c_double()
        assert ref.lib.ref_validate_sampled(R.h, 0.1, 1, C.byref(err_ref)) == 0
        A = h2.H2Matrix.construct(dim, n)
        err = h2.validate_sampled(A, 0.1, 1)
        assert err == pytest.approx(err_ref.value, rel=1e-6), (dim, err, err_ref.value)
        pts = ref.points(dim, n)
        assert h2.validate_sampled(A, 0.1, 1, points=pts, ell=0.1 if dim == 2 else 0.2) == pytest.approx(err, rel=1e-12)
