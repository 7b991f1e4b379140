"""GPU parity of the B200 H^2 mat-vec against the CPU oracle / reference.

Bar (BASELINE.json north_star): relative 2-norm error <= 1e-12 in FP64.
Every call goes through the C-ABI (include/h2b.h) via paper_1902_01829_b200.
"""
import numpy as np
import pytest

from conftest import rel_err

import paper_1902_01829_b200 as h2

pytestmark = pytest.mark.gpu
TOL = 1e-12


def _cases(golden):
    return sorted(golden.items())


def test_device_construct_matches_reference(gpu, golden):
    """h2b_matrix_build == construct(): structure and bases bit-identical,
    kernel-evaluated blocks within a few ulp (device exp)."""
    import oracle
    for name, (meta, _) in _cases(golden):
        A = h2.H2Matrix.construct(meta["dim"], meta["n"], grid_order=meta["grid_order"])
        d = A.to_host()
        r = oracle.restated().construct(meta["dim"], meta["n"], grid_order=meta["grid_order"]).to_host()
        for fld in ("perm", "cpl_row_ptr", "cpl_col_idx", "dense_row_ptr", "dense_col_idx", "ranks"):
            assert np.array_equal(getattr(d, fld), getattr(r, fld)), (name, fld)
        assert np.array_equal(d.leaf, r.leaf), name
        assert np.array_equal(d.transfer, r.transfer), name
        for fld in ("cpl_values", "dense_values"):
            a, b = getattr(d, fld), getattr(r, fld)
            assert a.shape == b.shape, (name, fld)
            if b.size:
                assert np.max(np.abs(a - b)) <= 4e-16 * max(1.0, np.max(np.abs(b))), (name, fld)
        assert A.memory_footprint() == meta["footprint"]
        assert A.info().hmv_flops == pytest.approx(meta["hmv_flops"], rel=1e-15)


def test_hmv_golden_device_built(gpu, golden):
    for name, (meta, arr) in _cases(golden):
        A = h2.H2Matrix.construct(meta["dim"], meta["n"], grid_order=meta["grid_order"])
        assert rel_err(h2.hmv(A, arr["x"]), arr["y"]) <= TOL, name
        assert rel_err(h2.hmv(A, arr["x"], arr["y0"].copy(), 2.0, 3.0), arr["y2"]) <= TOL, name


def test_hmv_uploaded_matches_oracle(gpu, golden, orc):
    for name, (meta, arr) in _cases(golden):
        O = orc.construct(meta["dim"], meta["n"], grid_order=meta["grid_order"])
        A = h2.H2Matrix.from_host(O.to_host())
        y = h2.hmv(A, arr["x"])
        assert rel_err(y, arr["y"]) <= TOL, name
        assert rel_err(y, O.hmv(arr["x"])) <= 1e-14, name


def test_beta_zero_never_reads_y(gpu, orc):
    O = orc.construct(2, 1024)
    A = h2.H2Matrix.from_host(O.to_host())
    x = np.random.default_rng(3).random(1024)
    y = np.full(1024, np.nan)
    h2.hmv(A, x, y, 1.0, 0.0)
    assert np.all(np.isfinite(y))
    assert rel_err(y, O.hmv(x)) <= TOL


def test_alpha_beta_semantics(gpu, orc):
    # test_hmv.cpp:91-101
    n = 256
    O = orc.construct(2, n)
    A = h2.H2Matrix.from_host(O.to_host())
    x = np.ones(n)
    base = h2.hmv(A, x)
    y = np.arange(n, dtype=np.float64)
    h2.hmv(A, x, y, 2.0, 3.0)
    assert np.allclose(y, 2.0 * base + 3.0 * np.arange(n), rtol=1e-13, atol=0)


def test_compressed_variable_ranks(gpu, golden, orc):
    """Odd and zero per-level ranks (post-compression layout) through the
    padded device pools."""
    for name, (meta, arr) in _cases(golden):
        O = orc.construct(meta["dim"], meta["n"], grid_order=meta["grid_order"])
        O.compress(meta["eps"])
        hm = O.to_host()
        assert list(hm.ranks) == meta["compress"]["new_ranks"]
        A = h2.H2Matrix.from_host(hm)
        assert rel_err(h2.hmv(A, arr["x"]), arr["yc"]) <= TOL, name
        back = A.to_host()
        for a, b in zip(back.arrays(), hm.arrays()):
            assert np.array_equal(a, b), name  # padded pools round-trip exactly


def test_phases_match_oracle(gpu, orc):
    for dim, n, order in [(2, 4096, 8), (3, 4096, 4), (2, 4096, 6), (3, 2048, 3)]:
        O = orc.construct(dim, n, grid_order=order)
        hm = O.to_host()
        A = h2.H2Matrix.from_host(hm)
        xc = np.random.default_rng(5).standard_normal(n)
        xh = h2.upsweep(A, xc)
        assert rel_err(xh, O.upsweep(xc)) <= TOL
        yh = h2.tree_multiply(A, xh)
        assert rel_err(yh, O.tree_multiply(xh)) <= TOL
        yd = h2.dense_mv(A, xc)
        assert rel_err(yd, O.dense_mv(xc)) <= TOL
        yh_in = yh.copy()
        yc = h2.downsweep(A, yh, yd)
        assert rel_err(yc, O.downsweep(yh_in, yd)) <= TOL
        # the reference's downsweep leaves y^l += E y^{l-1} in its LevelVectors
        # (hmv.hpp:136-146); so does h2b_downsweep
        exp = yh_in.copy()
        off = hm.vec_offsets()
        for l in range(1, hm.depth + 1):
            kc, kp = int(hm.ranks[l]), int(hm.ranks[l - 1])
            E = hm.transfer_level(l)
            par = exp[off[l - 1]:off[l]].reshape(1 << (l - 1), kp)
            ch = exp[off[l]:off[l + 1]].reshape(1 << l, kc)
            if kc and kp:
                ch += np.einsum("cij,cj->ci", E, par[np.arange(1 << l) >> 1])
        assert rel_err(yh, exp) <= TOL


def test_linearity_and_self_adjoint(gpu):
    # test_hmv.cpp:103-142 at a size the dense oracle cannot reach.
    A = h2.H2Matrix.construct(2, 1 << 16)
    rng = np.random.default_rng(23)
    n = 1 << 16
    u, v = rng.uniform(-1, 1, n), rng.uniform(-1, 1, n)
    yu, yv, yw = h2.hmv(A, u), h2.hmv(A, v), h2.hmv(A, 2.0 * u - 0.5 * v)
    assert rel_err(yw, 2.0 * yu - 0.5 * yv) <= TOL
    assert np.dot(v, yu) == pytest.approx(np.dot(u, yv), rel=1e-12)


def test_device_pointers_and_streams(gpu, orc):
    import torch
    O = orc.construct(2, 4096)
    A = h2.H2Matrix.from_host(O.to_host())
    x = np.random.default_rng(1).random(4096)
    xt = torch.from_numpy(x).cuda()
    yt = torch.full_like(xt, float("nan"))
    h2.hmv(A, xt, yt)
    torch.cuda.synchronize()
    assert rel_err(yt.cpu().numpy(), O.hmv(x)) <= TOL
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        h2.hmv(A, xt, yt, 1.0, 0.0, stream=s.cuda_stream)
    s.synchronize()
    assert rel_err(yt.cpu().numpy(), O.hmv(x)) <= TOL


def test_hmv_multi_columnwise(gpu, orc):
    O = orc.construct(2, 1024)
    A = h2.H2Matrix.from_host(O.to_host())
    X = np.random.default_rng(2).random((4, 1024))
    Y = h2.hmv_multi(A, X)
    for v in range(4):
        assert rel_err(Y[v], O.hmv(X[v])) <= TOL


def test_large_matches_reference(gpu, ref):
    """2D n = 2^18 (k = 64): device-built matrix vs the reference CPU hmv on
    the reference's own construct()."""
    n = 1 << 18
    R = ref.construct(2, n)
    x = ref.random_vector(n, 1)
    A = h2.H2Matrix.construct(2, n)
    assert A.memory_footprint() == R.footprint()
    assert rel_err(h2.hmv(A, x), R.hmv(x)) <= TOL


def test_hmv_multi_16_and_ragged(gpu, orc):
    """16-vector FP64-MMA path (k_hmv_mv.cu): every column equals the oracle's
    single-vector hmv; 20 vectors exercise a full pass + a ragged one; alpha/beta."""
    for dim, n, order in [(2, 4096, 8), (3, 4096, 4), (2, 4096, 6)]:
        O = orc.construct(dim, n, grid_order=order)
        A = h2.H2Matrix.from_host(O.to_host())
        rng = np.random.default_rng(8)
        X = rng.random((20, n))
        Y0 = rng.random((20, n))
        Y = h2.hmv_multi(A, X, 2.0, 0.5, Y0.copy())
        for v in range(20):
            assert rel_err(Y[v], O.hmv(X[v], Y0[v], 2.0, 0.5)) <= TOL, (dim, order, v)


def test_hmv_multi_device_pointers(gpu, orc):
    import ctypes as C
    import torch
    from paper_1902_01829_b200 import _lib
    O = orc.construct(2, 4096)
    A = h2.H2Matrix.from_host(O.to_host())
    X = torch.rand(16, 4096, dtype=torch.float64, device="cuda")
    Y = torch.zeros_like(X)
    _lib.check(_lib.load().h2b_hmv_multi(A._h, 16, C.c_void_p(X.data_ptr()), 4096,
                                         C.c_void_p(Y.data_ptr()), 4096, 1.0, 0.0, _lib.PTR_DEVICE,
                                         C.c_void_p(torch.cuda.current_stream().cuda_stream or 1)))
    torch.cuda.synchronize()
    Xn, Yn = X.cpu().numpy(), Y.cpu().numpy()
    for v in range(16):
        assert rel_err(Yn[v], O.hmv(Xn[v])) <= TOL


def test_fused_sweeps_repeat_bitwise(gpu, orc):
    """The up/down sweeps run as persistent dataflow launches whose per-node
    flags carry an epoch and are never reset: many back-to-back calls (device
    pointers, no host sync in between), alternating with the phase API and a
    compress (new ranks, same tree), give bitwise the same results."""
    import torch
    n = 1 << 14
    A = h2.H2Matrix.construct(2, n, grid_order=8)
    rng = np.random.default_rng(31)
    x = rng.random(n)
    y0 = h2.hmv(A, x)
    xt = torch.from_numpy(x).cuda()
    ys = [torch.empty_like(xt) for _ in range(64)]
    for yt in ys:
        h2.hmv(A, xt, yt)
    torch.cuda.synchronize()
    for yt in ys:
        assert np.array_equal(yt.cpu().numpy(), y0)
    xc = rng.random(n)
    xh = h2.upsweep(A, xc)  # per-level phase kernels in between
    assert np.array_equal(h2.hmv(A, x), y0)
    assert xh.size == A.col_vec_size()
    h2.compress(A, 1e-7)
    y1 = h2.hmv(A, x)
    assert rel_err(y1, y0) <= 1e-6
    for _ in range(8):
        assert np.array_equal(h2.hmv(A, x), y1)


def test_hmv_multi_compressed_ranks(gpu):
    """The 16-vector pass (TMA-fed coupling kernel) on compressed layouts: odd,
    small and zero ranks per level, rectangular ld / rank blocks; every column
    equals the single-vector mat-vec of the same handle."""
    for dim, n, order, eps in [(3, 4096, 4, 1e-4), (2, 4096, 8, 1e-2), (2, 1 << 14, 8, 0.5)]:
        A = h2.H2Matrix.construct(dim, n, grid_order=order)
        h2.compress(A, eps)
        X = np.random.default_rng(9).uniform(-1.0, 1.0, (16, n))
        Y = h2.hmv_multi(A, X)
        for v in (0, 5, 15):
            assert rel_err(Y[v], h2.hmv(A, X[v])) <= TOL, (dim, order, eps, A.info().ranks)


def test_tree_multiply_misaligned_device_pointers(gpu):
    """tree_multiply (the coupling product, hmv.hpp:114-125) on device x^ / y^
    pointers that are 8 bytes off a 16-byte boundary: the TMA-streamed kernel
    needs aligned tensor-map bases, so such calls take the register-fed
    kernel -- same result as the aligned call."""
    import ctypes as C
    import torch
    from paper_1902_01829_b200 import _lib
    A = h2.H2Matrix.construct(2, 1 << 14)
    nx, ny = A.col_vec_size(), A.vec_size()
    xh = np.random.default_rng(5).random(nx)
    ref = h2.tree_multiply(A, xh)
    xb = torch.zeros(nx + 1, dtype=torch.float64, device="cuda")
    yb = torch.zeros(ny + 1, dtype=torch.float64, device="cuda")
    xb[1:] = torch.from_numpy(xh)
    _lib.check(_lib.load().h2b_tree_multiply(A._h, C.c_void_p(xb[1:].data_ptr()), C.c_void_p(yb[1:].data_ptr()),
                                             _lib.PTR_DEVICE))
    torch.cuda.synchronize()
    assert rel_err(yb[1:].cpu().numpy(), ref) <= 1e-14
