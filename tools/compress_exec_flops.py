"""Executed FP64 flops of one compress() ("also report
unpadded executed flops"), from the SASS counters of every compress kernel:

    flops = 2 DFMA + DADD + DMUL (thread instructions, predicated on)
          + 512 x DMMA.8x8x4 warp instructions

    ncu --metrics <the four counters> --kernel-name regex:<compress kernels> \
        --csv --log-file gpurun_out/exec_flops.csv python tools/compress_exec_flops.py run DIM N ORDER EPS
    python tools/compress_exec_flops.py sum gpurun_out/exec_flops.csv   # -> JSON per kernel + total

Counts are what the kernels execute: the unpadded weight stacks, the upper
blocks only of symmetric levels, the skipped triangular fragments, the
Jacobi sweeps actually run -- and the dead-lane FMAs that SIMT still issues."""
import csv
import json
import sys
from collections import defaultdict

METRICS = ["sm__sass_thread_inst_executed_op_dfma_pred_on.sum", "sm__sass_thread_inst_executed_op_dadd_pred_on.sum",
           "sm__sass_thread_inst_executed_op_dmul_pred_on.sum", "sm__inst_executed_pipe_tensor_subpipe_dmma.sum"]
KERNELS = "regex:^k_(orth|project|sumsq|weights|trunc|jacobi|svd|compact)"


def run(dim, n, order, eps):
    sys.path.insert(0, ".")
    import torch
    import paper_1902_01829_b200 as h2
    A = h2.H2Matrix.construct(dim, n, grid_order=order)
    torch.cuda.synchronize()
    rep = h2.compress(A, eps)
    torch.cuda.synchronize()
    print(json.dumps({"model_flops": rep.total_flops(), "ms": rep.total_ms(), "new_ranks": rep.new_ranks}))


def summarise(path):
    lines = [l for l in open(path) if l.startswith('"')]
    per = defaultdict(lambda: defaultdict(float))
    for r in csv.DictReader(lines):
        k = r["Kernel Name"].split("(")[0].split("::")[-1].split("<")[0]
        per[k][r["Metric Name"]] += float(r["Metric Value"].replace(",", ""))
    out, tot = {}, 0.0
    for k, m in per.items():
        f = (2 * m[METRICS[0]] + m[METRICS[1]] + m[METRICS[2]] + 512 * m[METRICS[3]])
        out[k] = {"flops": f, "dmma_share": 512 * m[METRICS[3]] / f if f else 0.0}
        tot += f
    print(json.dumps({"executed_flops": tot, "per_kernel": out}, indent=1))


if __name__ == "__main__":
    if sys.argv[1] == "run":
        run(int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4]), float(sys.argv[5]))
    else:
        summarise(sys.argv[2])
