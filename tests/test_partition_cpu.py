"""CPU (gloo, world_size 2 and 4): the subtree-partitioned mat-vec protocol.

Each rank executes ONLY its partition of the mat-vec (numpy restatement of
the per-rank work of h2b_part_upsweep / h2b_part_finish, restricted to the
rows PartitionPlan assigns it), exchanges x^ with the same gather_xhat()
the GPU path uses over a real torch.distributed gloo group, all-gathers the
cluster-order y slices, and the result is compared with the oracle's hmv.
This pins the partition arithmetic and the collective protocol; the kernels
themselves are pinned by tests/test_partition_gpu.py."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1902_01829_b200.dist import gather_xhat
from paper_1902_01829_b200.partition import PartitionPlan, owned_range


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def local_hmv(hm, plan, x, xhat_t, allgather):
    """Per-rank work of the partitioned mat-vec on host arrays; xhat_t is a
    torch CPU tensor (exchanged with gather_xhat), xhat its numpy view."""
    xhat = xhat_t.numpy()
    q, m, r = hm.depth, hm.m, [int(v) for v in hm.ranks]
    off = plan.off
    s, g = plan.s, plan.part
    xc = x[hm.perm]
    U = hm.leaves()
    # (1) owned leaves -> x^q, then owned parents down to level s
    l0, l1 = plan.leaf_range()
    for i in range(l0, l1):
        xhat[off[q] + i * r[q]: off[q] + (i + 1) * r[q]] = U[i].T @ xc[i * m:(i + 1) * m]

    def up(l, p0, p1):
        F = hm.transfer_level(l)
        for p in range(p0, p1):
            acc = np.zeros(r[l - 1])
            for c in (2 * p, 2 * p + 1):
                acc += F[c].T @ xhat[off[l] + c * r[l]: off[l] + (c + 1) * r[l]]
            xhat[off[l - 1] + p * r[l - 1]: off[l - 1] + (p + 1) * r[l - 1]] = acc

    for l in range(q, s, -1):
        up(l, *owned_range(l - 1, s, g))
    # (2) exchange: the same protocol code as the GPU path
    gather_xhat(plan, xhat_t, allgather)
    # (3) replicated top upsweep
    for l in range(s, 0, -1):
        up(l, 0, 1 << (l - 1))
    # coupling rows of the owned subtree (all rows above level s)
    yhat = np.zeros_like(xhat)
    for l in range(q + 1):
        rp, ci, S = hm.level_row_ptr(l), hm.level_col_idx(l), hm.level_values(l)
        a, b = owned_range(l, s, g)
        for row in range(a, b):
            acc = np.zeros(r[l])
            for blk in range(rp[row], rp[row + 1]):
                j = ci[blk]
                acc += S[blk] @ xhat[off[l] + j * r[l]: off[l] + (j + 1) * r[l]]
            yhat[off[l] + row * r[l]: off[l] + (row + 1) * r[l]] = acc
    # downsweep over owned children
    for l in range(1, q + 1):
        E = hm.transfer_level(l)
        a, b = owned_range(l, s, g)
        for c in range(a, b):
            pa = off[l - 1] + (c // 2) * r[l - 1]
            yhat[off[l] + c * r[l]: off[l] + (c + 1) * r[l]] += E[c] @ yhat[pa:pa + r[l - 1]]
    # dense rows + leaf expansion -> owned cluster-order y slice
    D = hm.dense_values.reshape(-1, m, m).transpose(0, 2, 1)
    ys = np.zeros((l1 - l0) * m)
    for i in range(l0, l1):
        acc = U[i] @ yhat[off[q] + i * r[q]: off[q] + (i + 1) * r[q]]
        for blk in range(hm.dense_row_ptr[i], hm.dense_row_ptr[i + 1]):
            j = hm.dense_col_idx[blk]
            acc += D[blk] @ xc[j * m:(j + 1) * m]
        ys[(i - l0) * m:(i - l0 + 1) * m] = acc
    return ys


def _worker(rank, world, port, dim, n, order, out_q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import oracle
        O = oracle.restated().construct(dim, n, grid_order=order)
        hm = O.to_host()
        x = np.random.default_rng(12).random(n)
        plan = PartitionPlan(hm.depth, hm.ranks, hm.m, world, rank)
        xhat_t = torch.zeros(plan.off[-1], dtype=torch.float64)

        def allgather(out, inp):
            parts = [torch.empty_like(inp) for _ in range(world)]
            dist.all_gather(parts, inp.clone())
            out.copy_(torch.cat(parts))

        ys = local_hmv(hm, plan, x, xhat_t, allgather)
        ycl = torch.zeros(n, dtype=torch.float64)
        allgather(ycl, torch.from_numpy(ys))
        y = np.zeros(n)
        y[hm.perm] = ycl.numpy()
        ref = O.hmv(x)
        out_q.put((rank, float(np.linalg.norm(y - ref) / np.linalg.norm(ref))))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,dim,n,order", [(2, 2, 1 << 12, 8), (4, 3, 1 << 12, 4)])
def test_partitioned_protocol_gloo(world, dim, n, order):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, dim, n, order, q)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(240)
        assert p.exitcode == 0
    errs = [q.get(timeout=5) for _ in range(world)]
    assert all(e <= 1e-12 for _, e in errs), errs


def test_plan_matches_device_partition_arithmetic():
    """PartitionPlan mirrors Matrix::own_begin/own_end (csrc/h2b_internal.hpp)."""
    plan = PartitionPlan(10, [64] * 11, 64, 8, 5)
    assert plan.leaf_range() == (5 << 7, 6 << 7)
    assert owned_range(2, 3, 5) == (0, 4)        # above the split: replicated
    assert owned_range(3, 3, 5) == (5, 6)
    off, length, chunk = plan.level_slice(10)
    assert length == (1 << 10) * 64 and chunk == length // 8
    assert plan.gather_levels() == list(range(3, 11))
    with pytest.raises(ValueError):
        PartitionPlan(2, [64] * 3, 64, 8, 0)
    with pytest.raises(ValueError):
        PartitionPlan(5, [64] * 6, 64, 3, 0)
