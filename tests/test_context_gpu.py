"""Per-caller workspaces (HmvContext, hmv.hpp:159-172): the reference allows
concurrent hmv on one immutable matrix with one context each.
Two threads x two contexts x two CUDA streams on one device matrix must give
results bitwise equal to a sequential mat-vec; calls sharing a context (or the
handle's own workspace) from several streams are serialised, not raced."""
import threading

import numpy as np
import pytest

import paper_1902_01829_b200 as h2

pytestmark = pytest.mark.gpu


def _run_threads(fns):
    errs = []

    def wrap(f):
        try:
            f()
        except Exception as e:  # noqa: BLE001
            errs.append(e)

    ts = [threading.Thread(target=wrap, args=(f,)) for f in fns]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    if errs:
        raise errs[0]


def test_two_threads_two_contexts_two_streams_bitwise(gpu):
    import torch
    A = h2.H2Matrix.construct(2, 1 << 16)
    n = A.n
    xs = [torch.rand(n, dtype=torch.float64, device="cuda", generator=torch.Generator("cuda").manual_seed(s))
          for s in (1, 2)]
    ref = [h2.hmv(A, x) for x in xs]
    torch.cuda.synchronize()
    ctxs = [h2.HmvContext(A), h2.HmvContext(A)]
    streams = [torch.cuda.Stream(), torch.cuda.Stream()]
    reps = 20
    outs = [[torch.empty(n, dtype=torch.float64, device="cuda") for _ in range(reps)] for _ in range(2)]

    def worker(i):
        def f():
            with torch.cuda.stream(streams[i]):
                for r in range(reps):
                    h2.hmv(A, xs[i], outs[i][r], ctx=ctxs[i], stream=streams[i].cuda_stream)
        return f

    _run_threads([worker(0), worker(1)])
    torch.cuda.synchronize()
    for i in range(2):
        for r in range(reps):
            assert torch.equal(outs[i][r], ref[i]), (i, r)
    for c in ctxs:
        c.close()
    A.close()


def test_shared_workspace_across_streams_is_serialised(gpu):
    """No context: both threads use the handle's workspace from their own
    streams; the device-order hand-off keeps every result exact."""
    import torch
    A = h2.H2Matrix.construct(2, 1 << 15)
    n = A.n
    xs = [torch.rand(n, dtype=torch.float64, device="cuda") for _ in range(2)]
    ref = [h2.hmv(A, x) for x in xs]
    torch.cuda.synchronize()
    streams = [torch.cuda.Stream(), torch.cuda.Stream()]
    reps = 15
    outs = [[torch.empty(n, dtype=torch.float64, device="cuda") for _ in range(reps)] for _ in range(2)]

    def worker(i):
        def f():
            for r in range(reps):
                h2.hmv(A, xs[i], outs[i][r], stream=streams[i].cuda_stream)
        return f

    _run_threads([worker(0), worker(1)])
    torch.cuda.synchronize()
    for i in range(2):
        for r in range(reps):
            assert torch.equal(outs[i][r], ref[i]), (i, r)
    A.close()


def test_context_follows_compress(gpu, orc):
    """A context created before compress() re-sizes itself for the new ranks
    (the reference's context would be invalid, App. C of SURVEY.md)."""
    A = h2.H2Matrix.construct(2, 4096)
    ctx = h2.HmvContext(A)
    x = orc.random_vector(4096, 1)
    y0 = h2.hmv(A, x, ctx=ctx)
    h2.compress(A, 1e-7)
    y1 = h2.hmv(A, x, ctx=ctx)
    y2 = h2.hmv(A, x)
    assert np.array_equal(y1, y2)
    assert np.linalg.norm(y1 - y0) / np.linalg.norm(y0) <= 1e-6
    ctx.close()


def test_host_pointer_hmv_with_context(gpu, orc):
    O = orc.construct(2, 2048)
    A = h2.H2Matrix.from_host(O.to_host())
    ctx = h2.HmvContext(A)
    x = orc.random_vector(2048, 3)
    y0 = orc.random_vector(2048, 4)
    y = h2.hmv(A, x, y0.copy(), 2.0, 3.0, ctx=ctx)
    yr = O.hmv(x, y0, 2.0, 3.0)
    assert np.linalg.norm(y - yr) / np.linalg.norm(yr) <= 1e-12


def test_python_argument_checks(gpu):
    A = h2.H2Matrix.construct(2, 1024)
    with pytest.raises(ValueError):
        h2.hmv(A, np.zeros(1000))
    with pytest.raises(ValueError):
        h2.hmv(A, np.zeros(1024, np.float32))
    with pytest.raises(ValueError):
        h2.hmv(A, np.zeros(1024), np.zeros(1023))
    with pytest.raises(ValueError):
        h2.upsweep(A, np.zeros(10))
    with pytest.raises(ValueError):
        h2.tree_multiply(A, np.zeros(3))
    with pytest.raises(ValueError):
        h2.downsweep(A, np.zeros(A.vec_size() + 1), np.zeros(1024))
    with pytest.raises(ValueError):
        h2.validate_sampled(A, 0.1, points=np.zeros((1000, 2)))


def test_async_pinned_host_calls(gpu, orc):
    """H2B_PTR_HOST_ASYNC: pinned host vectors, stream-ordered, two calls in
    flight on two contexts / streams; pageable host memory is refused."""
    import torch
    n = 4096
    A = h2.H2Matrix.construct(2, n)
    x = orc.random_vector(n, 1)
    y_ref = h2.hmv(A, x)
    xh = torch.from_numpy(x).pin_memory()
    ys = [torch.zeros(n, dtype=torch.float64).pin_memory() for _ in range(2)]
    ctxs = [h2.HmvContext(A), h2.HmvContext(A)]
    sts = [torch.cuda.Stream(), torch.cuda.Stream()]
    for i in range(6):
        k = i & 1
        h2.hmv(A, xh.numpy(), ys[k].numpy(), stream=sts[k].cuda_stream, ctx=ctxs[k], asynchronous=True)
    torch.cuda.synchronize()
    for y in ys:
        assert np.array_equal(y.numpy(), y_ref)
    with pytest.raises(h2.H2bInvalidArgument):
        h2.hmv(A, x, np.zeros(n), ctx=ctxs[0], asynchronous=True)  # pageable


def test_hmv_graph_replay(gpu, orc):
    """h2b_hmv_graph_*: a captured mat-vec replays bitwise equal to the direct
    call (the sweep epoch advances on the device, so replays stay ordered),
    on a context and on the matrix's own workspace, and refuses to run after
    compress() changed the layout."""
    import torch
    for dim, n, order in [(2, 4096, 8), (2, 8192, 10)]:  # 64 and 100 (k_hmv_big.cu)
        A = h2.H2Matrix.construct(dim, n, grid_order=order)
        x = torch.from_numpy(orc.random_vector(n, 1)).cuda()
        y0 = torch.rand(n, dtype=torch.float64, device="cuda")
        y_ref = y0.clone()
        h2.hmv(A, x, y_ref, 1.5, 0.5)
        ctx = h2.HmvContext(A)
        for c in (ctx, None):
            y = y0.clone()
            g = h2.HmvGraph(A, x, y, 1.5, 0.0, ctx=c)
            for _ in range(5):
                g.launch()
            torch.cuda.synchronize()
            assert torch.equal(y, h2.hmv(A, x, torch.zeros_like(x), 1.5, 0.0))
            g.close()
        y = y0.clone()
        g = h2.HmvGraph(A, x, y, 1.5, 0.5, ctx=ctx)
        g.launch()
        torch.cuda.synchronize()
        assert torch.equal(y, y_ref)
        if order == 8:
            h2.compress(A, 1e-6)
            with pytest.raises(h2.H2bInvalidArgument, match="layout changed"):
                g.launch()
        g.close()
        ctx.close()


def test_async_pinned_host_alpha_beta(gpu, orc):
    """H2B_PTR_HOST_ASYNC with beta != 0 reads the pinned y (stream-ordered)."""
    import torch
    n = 4096
    A = h2.H2Matrix.construct(2, n)
    x = orc.random_vector(n, 2)
    y0 = np.random.default_rng(3).random(n)
    y_ref = h2.hmv(A, x, y0.copy(), 2.0, -0.5)
    xh = torch.from_numpy(x).pin_memory()
    yh = torch.from_numpy(y0.copy()).pin_memory()
    st = torch.cuda.Stream()
    h2.hmv(A, xh.numpy(), yh.numpy(), 2.0, -0.5, stream=st.cuda_stream, asynchronous=True)
    st.synchronize()
    assert np.array_equal(yh.numpy(), y_ref)
