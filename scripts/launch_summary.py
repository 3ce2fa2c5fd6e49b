"""Summarize an ncu `--metrics gpu__time_duration.sum --csv` launch list."""
import csv
import sys
from collections import defaultdict

rows = list(csv.reader(open(sys.argv[1])))
hdr, data = None, []
for r in rows:
    if "Kernel Name" in r:
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        d = dict(zip(hdr, r))
        if d.get("Metric Name") == "gpu__time_duration.sum":
            scale = {"ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3}.get(d.get("Metric Unit", "ns"), 1e-3)
            data.append((d["Kernel Name"], float(d["Metric Value"].replace(",", "")) * scale))
agg = defaultdict(lambda: [0, 0.0])
for n, v in data:
    key = n.split("(")[0].replace("void ", "").replace("(anonymous namespace)::", "")[:60]
    agg[key][0] += 1
    agg[key][1] += v
tot = sum(v for _, v in data)
print(f"launches {len(data)}  total {tot:.1f} us")
for k, (c, v) in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"{v:9.1f} us {100 * v / tot:5.1f}%  n={c:4d}  avg {v / c:7.1f} us  {k}")
