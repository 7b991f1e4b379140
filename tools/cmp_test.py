import sys, time, json
sys.path.insert(0, ".")
import torch
import paper_1902_01829_b200 as h2
import bench
def run(tag):
    r = bench.compression_run(h2, torch, 0, 2)
    print(tag, json.dumps({k: r[k] for k in ("ms", "wall_ms", "phase_ms")}), flush=True)
run("fresh")
A = h2.H2Matrix.construct(2, 1 << 22)
y = h2.hmv(A, torch.rand(1 << 22, dtype=torch.float64, device="cuda"))
A.close(); del A
torch.cuda.synchronize()
run("after-77GB")
run("again")
