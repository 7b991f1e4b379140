"""CPU (gloo, world_size 2): the host communicator of the partitioned
compression (h2b_comm, include/h2b.h).  Each rank builds TorchComm, takes its
ctypes h2b_comm and invokes the three callbacks exactly as libh2b does from
h2b_part_compress -- in-place all-gather of per-level slices (host buffers
here; device buffers under NCCL), all-reduce MAX of the per-level truncated
rank + non-finite flag, all-reduce SUM of ||A||_F^2 / energy / footprints --
and checks the results; plus the ThreadComm used by the one-GPU emulation."""
import ctypes as C
import os
import socket
import threading

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1902_01829_b200.dist import ThreadComm, TorchComm


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _exercise(comm, world, rank):
    cs = comm.as_c()
    # level slices of a "T tree": rank r owns chunk r of each level
    out = {}
    for chunk in (1, 7, 4096):
        buf = np.full(world * chunk, -1.0)
        buf[rank * chunk:(rank + 1) * chunk] = np.arange(chunk) + 1000.0 * rank
        assert cs.allgather(None, buf.ctypes.data, chunk) == 0
        out[chunk] = buf.copy()
    v = np.array([3 + rank, 0 if rank else 1], dtype=np.int32)
    assert cs.allreduce_max_i32(None, v.ctypes.data_as(C.POINTER(C.c_int32)), 2) == 0
    d = np.array([1.5 * (rank + 1), 2.0 ** -40, 7.0])
    assert cs.allreduce_sum_f64(None, d.ctypes.data_as(C.POINTER(C.c_double)), 3) == 0
    return out, v, d


def _check(out, v, d, world):
    for chunk, buf in out.items():
        ref = np.concatenate([np.arange(chunk) + 1000.0 * r for r in range(world)])
        assert np.array_equal(buf, ref)
    assert list(v) == [3 + world - 1, 1]
    assert np.allclose(d, [1.5 * world * (world + 1) / 2, world * 2.0 ** -40, 7.0 * world], rtol=0, atol=0)


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        comm = TorchComm(device=None)
        assert (comm.nparts, comm.part) == (world, rank)
        out, v, d = _exercise(comm, world, rank)
        _check(out, v, d, world)
        q.put((rank, "ok"))
    except Exception as e:  # noqa: BLE001
        q.put((rank, repr(e)))
    finally:
        dist.destroy_process_group()


def test_torchcomm_callbacks_gloo():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(240)
        assert p.exitcode == 0
    res = sorted(q.get(timeout=5) for _ in range(world))
    assert res == [(0, "ok"), (1, "ok")], res


@pytest.mark.parametrize("world", [2, 4])
def test_threadcomm_callbacks(world):
    tc = ThreadComm(world, device=None)
    results, errs = [None] * world, []

    def run(r):
        try:
            results[r] = _exercise(tc.rank(r), world, r)
        except Exception as e:  # noqa: BLE001
            errs.append(e)
            tc.barrier.abort()

    th = [threading.Thread(target=run, args=(r,)) for r in range(world)]
    for t in th:
        t.start()
    for t in th:
        t.join(60)
    assert not errs, errs
    for out, v, d in results:
        _check(out, v, d, world)


def test_callback_errors_are_reported():
    tc = ThreadComm(1, device=None)
    c = tc.rank(0)
    c.allgather = lambda buf: (_ for _ in ()).throw(RuntimeError("boom"))
    cs = c.as_c()
    buf = np.zeros(4)
    assert cs.allgather(None, buf.ctypes.data, 4) == 1
    assert isinstance(c.error, RuntimeError)
