"""Kernel timeline (CUPTI via torch.profiler) of compress() runs: per-run
kernel-busy time vs the phase times, and the largest idle gaps.
    python tools/compress_timeline.py DIM N ORDER EPS REPS [seq]"""
import json
import sys

sys.path.insert(0, ".")
import torch
from torch.profiler import ProfilerActivity, profile

import paper_1902_01829_b200 as h2

dim, n, order, eps, reps = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3]), float(sys.argv[4]), int(sys.argv[5])
for _ in range(reps):
    A = h2.H2Matrix.construct(dim, n, grid_order=order)
    torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        rep = h2.compress(A, eps)
        torch.cuda.synchronize()
    ev = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
    ev.sort(key=lambda e: e.time_range.start)
    busy = sum(e.time_range.elapsed_us() for e in ev) / 1e3
    span = (ev[-1].time_range.end - ev[0].time_range.start) / 1e3 if ev else 0
    gaps = []
    for a, b in zip(ev, ev[1:]):
        g = (b.time_range.start - a.time_range.end) / 1e3
        gaps.append((g, a.name[:40], b.name[:40]))
    big = [(round(g, 2), a, b) for g, a, b in gaps if g > 1.0]
    gaps.sort(reverse=True)
    # device idle time: the span minus the union of kernel intervals
    idle, cur_end, holes = 0.0, None, []
    for e in ev:
        st, en = e.time_range.start, e.time_range.end
        if cur_end is not None and st > cur_end:
            idle += (st - cur_end) / 1e3
            holes.append((round((st - cur_end) / 1e3, 3), e.name.replace("h2b::(anonymous namespace)::", "")[:28]))
        cur_end = en if cur_end is None else max(cur_end, en)
    holes.sort(reverse=True)
    print(json.dumps(dict(idle_ms=round(idle, 2), n_holes=len(holes), top_holes=holes[:12])), flush=True)
    slow = sorted(((e.time_range.elapsed_us() / 1e3, e.name[:50]) for e in ev), reverse=True)[:6]
    agg = {}
    for e in ev:
        k = e.name.replace("h2b::(anonymous namespace)::", "").replace("void ", "").split("(")[0][:30]
        agg[k] = agg.get(k, 0.0) + e.time_range.elapsed_us() / 1e3
    print(json.dumps(dict(ms=round(rep.total_ms(), 1), kernels_busy_ms=round(busy, 1), span_ms=round(span, 1),
                          gaps_over_1ms=big, gap_total_ms=round(sum(g for g, _, _ in gaps), 1),
                          top_kernels=[(round(t, 2), k) for t, k in slow],
                          per_kernel={k: round(v, 1) for k, v in sorted(agg.items(), key=lambda kv: -kv[1])})), flush=True)
    if len(sys.argv) > 6:  # every launch in order: name, ms
        t0 = ev[0].time_range.start
        for e in ev:  # start offset, duration, kernel
            k = e.name.replace("h2b::(anonymous namespace)::", "").replace("void ", "").split("(")[0][:28]
            print(f"  {(e.time_range.start - t0) / 1e3:9.3f} {e.time_range.elapsed_us() / 1e3:8.3f}  {k}", flush=True)
    A.close()
    del A
