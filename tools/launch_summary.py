"""Per-kernel totals of an ncu launch list (--metrics gpu__time_duration.sum --csv).
    python tools/launch_summary.py LAUNCHES.csv > SUMMARY.txt"""
import csv
import sys
from collections import defaultdict

rows = [r for r in csv.reader(l for l in open(sys.argv[1]) if l.startswith('"'))]
h = rows[0]
ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
tot, cnt = defaultdict(float), defaultdict(int)
for r in rows[1:]:
    name = r[ki].split("(")[0].replace("h2b::<unnamed>::", "").replace("void ", "").strip()
    v = float(r[vi].replace(",", ""))
    scale = {"ns": 1e-6, "us": 1e-3, "usecond": 1e-3, "nsecond": 1e-6, "ms": 1.0, "msecond": 1.0}.get(r[ui], 1e-6)
    tot[name] += v * scale
    cnt[name] += 1
all_ms = sum(tot.values())
print("# ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv python bench.py --steps 2 --warmup 1 "
      "--no-compress (B200, round 2)")
print("# cold-cache, serialised launches; the bench numbers printed under ncu are not bench values")
print(f"{'kernel':40s} {'launches':>9s} {'total ms':>10s} {'share':>7s}")
for k, v in sorted(tot.items(), key=lambda kv: -kv[1]):
    print(f"{k[:40]:40s} {cnt[k]:9d} {v:10.3f} {100 * v / all_ms:6.2f}%")
