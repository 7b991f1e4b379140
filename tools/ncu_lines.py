"""Per-CUDA-source-line warp-stall samples from an ncu report
(--page source --print-source cuda,sass), top lines per kernel.
    python tools/ncu_lines.py REPORT.ncu-rep [TOP]"""
import csv
import io
import subprocess
import sys
from collections import defaultdict

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
per = defaultdict(lambda: defaultdict(float))
src_of = {}
fn = None
fpath = None
for row in csv.reader(io.StringIO(txt)):
    if not row:
        continue
    if row[0] == "File Path":
        fpath = row[1].split("/")[-1]
        continue
    if row[0] == "Function Name":
        fn = row[1].split("(")[0].replace("h2b::<unnamed>::", "")
        continue
    if row[0] == "Line No" or not row[0]:
        continue
    try:
        s = float(row[4])
    except (ValueError, IndexError):
        continue
    key = (fpath, int(row[0]))
    per[fn][key] += s
    src_of[key] = row[1].strip()
for f, d in per.items():
    tot = sum(d.values())
    print(f"== {f}: {tot:.0f} samples")
    for key, s in sorted(d.items(), key=lambda kv: -kv[1])[:top]:
        print(f"{100 * s / tot:5.1f}% {key[0]}:{key[1]:<5d} {src_of[key][:90]}")
