"""Summarise an `ncu --metrics gpu__time_duration.sum --csv` launch list:
per-kernel launch count, total device time and share (cold-cache, serialised)."""
import csv
import io
import sys
from collections import defaultdict

SCALE = {"ns": 1e-6, "nsecond": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0,
         "s": 1e3, "second": 1e3}


def summarize(path):
    txt = open(path).read().splitlines()
    start = [i for i, l in enumerate(txt) if l.startswith('"ID"')][0]
    rows = list(csv.reader(io.StringIO("\n".join(txt[start:]))))
    hdr = rows[0]
    ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    tot, cnt = defaultdict(float), defaultdict(int)
    for r in rows[1:]:
        name = r[ki].split("(")[0].replace("h2b::<unnamed>::", "").replace("void ", "")
        tot[name] += float(r[vi].replace(",", "")) * SCALE[r[ui]]
        cnt[name] += 1
    s = sum(tot.values())
    out = [f"{'kernel':40s} {'launches':>8s} {'total ms':>10s} {'share':>7s}"]
    for k in sorted(tot, key=lambda k: -tot[k]):
        out.append(f"{k[:40]:40s} {cnt[k]:8d} {tot[k]:10.3f} {100 * tot[k] / s:6.2f}%")
    out.append(f"{'TOTAL':40s} {sum(cnt.values()):8d} {s:10.3f}")
    return "\n".join(out)


if __name__ == "__main__":
    print(summarize(sys.argv[1]))
