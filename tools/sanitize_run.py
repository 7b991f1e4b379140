"""Small end-to-end workload for compute-sanitizer (memcheck / racecheck /
synccheck): device construction, hmv (fused sweeps), 16-vector pass, phase
API, compress (orth / project / weights / truncation / compaction), a
non-symmetric matrix and its compress; round 2: blocks > 64 (k_hmv_big.cu),
the one-call partitioned mat-vec (pack / unpack / scatter, 16-vector
partitions) with an in-process communicator, the asynchronous host path.
    compute-sanitizer --tool memcheck python tools/sanitize_run.py"""
import sys

sys.path.insert(0, ".")
sys.path.insert(0, "tests")
import numpy as np

import paper_1902_01829_b200 as h2

n = 1 << 12
A = h2.H2Matrix.construct(2, n, grid_order=6)
x = np.random.default_rng(1).random(n)
y = h2.hmv(A, x)
Y = h2.hmv_multi(A, np.random.default_rng(2).random((16, n)))
xh = h2.upsweep(A, x)
yh = h2.tree_multiply(A, xh)
rep = h2.compress(A, 1e-6)
y2 = h2.hmv(A, x)
B = h2.H2Matrix.construct(3, n, grid_order=3)
h2.compress(B, 1e-5)
from nonsym import scaled  # noqa: E402

hm = A.to_host()
N = h2.H2Matrix.from_host(scaled(hm))
h2.hmv(N, x)
h2.compress(N, 1e-5)
# blocks of 81 and 128 rows / columns
G = h2.H2Matrix.construct(2, 1 << 13, leaf_size=128, grid_order=9)
xg = np.random.default_rng(3).random(1 << 13)
yg = h2.hmv(G, xg)
h2.hmv_multi(G, np.random.default_rng(4).random((2, 1 << 13)))
# partitioned one-call mat-vec, P = 2 partitions driven sequentially through a
# communicator whose all-gather copies between the two handles' buffers
import ctypes as C  # noqa: E402

import torch  # noqa: E402

from paper_1902_01829_b200 import _lib  # noqa: E402
from paper_1902_01829_b200.dist import DistributedH2Matrix, ThreadComm  # noqa: E402
import threading  # noqa: E402

parts = [DistributedH2Matrix(2, n, grid_order=6, nparts=2, part=g, device=0) for g in range(2)]
tc = ThreadComm(2, device=0)
xt = torch.from_numpy(x).cuda()
outs = [None, None]


def run(g):
    torch.cuda.set_device(0)
    st = torch.cuda.Stream()
    with torch.cuda.stream(st):
        yv = torch.zeros_like(xt)
        parts[g].hmv(xt, yv, comm=tc.rank(g), stream=st.cuda_stream)
        Xv = torch.from_numpy(np.random.default_rng(5).random((3, n))).cuda()
        parts[g].hmv_multi(Xv, comm=tc.rank(g), stream=st.cuda_stream)
        st.synchronize()
        outs[g] = yv.cpu().numpy()


th = [threading.Thread(target=run, args=(g,)) for g in range(2)]
for t in th:
    t.start()
for t in th:
    t.join()
# asynchronous pinned-host calls on two contexts
xp = torch.from_numpy(x).pin_memory()
yps = [torch.zeros(n, dtype=torch.float64).pin_memory() for _ in range(2)]
ctxs = [h2.HmvContext(A), h2.HmvContext(A)]
sts = [torch.cuda.Stream(), torch.cuda.Stream()]
for i in range(4):
    h2.hmv(A, xp.numpy(), yps[i & 1].numpy(), stream=sts[i & 1].cuda_stream, ctx=ctxs[i & 1], asynchronous=True)
torch.cuda.synchronize()
print("ok", rep.new_ranks, float(np.linalg.norm(y2 - y) / np.linalg.norm(y)),
      float(np.linalg.norm(yps[1].numpy() - y2) / np.linalg.norm(y2)))
