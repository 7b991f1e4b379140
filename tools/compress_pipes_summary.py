"""Time-weighted pipe utilisation per compression kernel from an ncu CSV
(tools/ncu_compress_pipes.sh):  python tools/compress_pipes_summary.py CSV"""
import collections
import csv
import json
import sys

KERNELS = ("k_weights", "k_project", "k_jacobi64", "k_orth_level", "k_trunc_level_pre", "k_trunc_leaf_pre",
           "k_orth_leaf", "k_svd_apply")
rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
h = rows[0]
ki, mi, vi, ui, ii = (h.index(x) for x in ("Kernel Name", "Metric Name", "Metric Value", "Metric Unit", "ID"))
per = collections.defaultdict(dict)
for r in rows[1:]:
    name = r[ki].split("(")[0].split("::")[-1].split("<")[0]
    per[(r[ii], name)][r[mi]] = (float(r[vi].replace(",", "")), r[ui])
acc = collections.defaultdict(lambda: [0.0, 0.0, 0.0])
for (_, name), m in per.items():
    if name not in KERNELS:
        continue
    t, u = m["gpu__time_duration.sum"]
    t *= {"ns": 1e-6, "nsecond": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0}[u]
    a = acc[name]
    a[0] += t
    a[1] += t * m.get("sm__inst_executed_pipe_tensor_subpipe_dmma.avg.pct_of_peak_sustained_active", (0.0, ""))[0]
    a[2] += t * m.get("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", (0.0, ""))[0]
out = {k: {"ms": round(a[0], 1), "dmma_pct": round(a[1] / a[0], 1), "fp64_pct": round(a[2] / a[0], 1)}
       for k, a in sorted(acc.items(), key=lambda kv: -kv[1][0])}
print(json.dumps(out, indent=1))
