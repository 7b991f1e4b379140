"""Where does the distributed e2e time go (N=1 through NCCL)?"""
import os, sys, time
sys.path.insert(0, ".")
os.environ.setdefault("MASTER_ADDR", "127.0.0.1"); os.environ.setdefault("MASTER_PORT", "29555")
os.environ.setdefault("RANK", "0"); os.environ.setdefault("WORLD_SIZE", "1")
import torch, torch.distributed as dist
torch.cuda.set_device(0)
dist.init_process_group("nccl", device_id=torch.device("cuda", 0))
from paper_1902_01829_b200.dist import DistributedH2Matrix
n = 1 << 22
D = DistributedH2Matrix(2, n, device=0)
s = torch.cuda.Stream(); torch.cuda.set_stream(s)
x = torch.rand(n, dtype=torch.float64, device="cuda"); y = torch.zeros_like(x)
xh = torch.empty(n, dtype=torch.float64, pin_memory=True); yh = torch.empty(n, dtype=torch.float64, pin_memory=True)
xh.copy_(x.cpu()); xd = torch.empty_like(x)
def timed(fn, k=10):
    for _ in range(2): fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    for _ in range(k): fn()
    e1.record(s); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / k
print("hmv", timed(lambda: D.hmv(x, y)))
print("h2d", timed(lambda: xd.copy_(xh, non_blocking=True)))
print("d2h", timed(lambda: yh.copy_(y, non_blocking=True)))
print("all", timed(lambda: (xd.copy_(xh, non_blocking=True), D.hmv(xd, y), yh.copy_(y, non_blocking=True))))
import paper_1902_01829_b200 as h2
print("scatter", timed(lambda: y.__setitem__(D.perm, D.y_cluster)))
dist.destroy_process_group()
