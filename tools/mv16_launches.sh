#!/bin/bash
# Launch list (ncu gpu__time_duration + DRAM bytes, serialised, cold-ish) of one
# 16-vector pass at C4 after warm-up: gpurun_out/mv16_launches${MVTAG}.csv.
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    --kernel-name-base function -k regex:'_mv' -s 60 -c 40 --csv --log-file gpurun_out/mv16_launches${MVTAG}.csv \
    python tools/mv16_time.py > /dev/null 2>&1
python - <<'PY'
import csv, collections
import os
lines = [l for l in open("gpurun_out/mv16_launches" + os.environ.get("MVTAG", "") + ".csv") if l.startswith('"')]
rows = list(csv.DictReader(lines))
agg = collections.OrderedDict()
for r in rows:
    k = r["Kernel Name"].split("(")[0].split("::")[-1]; m = r["Metric Name"]; v = float(r["Metric Value"].replace(",", "")) * (1e0 if r["Metric Unit"] in ("byte", "ns", "nsecond") else {"Kbyte":1e3,"Mbyte":1e6,"Gbyte":1e9,"usecond":1e3,"us":1e3,"msecond":1e6,"ms":1e6}.get(r["Metric Unit"], 1.0))
    d = agg.setdefault((r["ID"], k), {})
    d[m] = v
tot = collections.defaultdict(lambda: [0, 0.0, 0.0, 0.0])
for (i, k), d in agg.items():
    t = tot[k]; t[0] += 1; t[1] += d.get("gpu__time_duration.sum", 0)
    t[2] += d.get("dram__bytes_read.sum", 0); t[3] += d.get("dram__bytes_write.sum", 0)
for k, (c, ns, rd, wr) in tot.items():
    print(f"{k:20s} launches {c:3d}  ms/launch {ns/c/1e6:8.3f}  GB read/launch {rd/c/1e9:7.3f}  written {wr/c/1e9:7.3f}")
PY
