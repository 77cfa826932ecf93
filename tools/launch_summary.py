"""Summarise an `ncu --metrics gpu__time_duration.sum --csv` launch list by kernel:
launches, total time, share.  usage: python tools/launch_summary.py launches.csv"""
import csv
import re
import sys
from collections import defaultdict

rows = []
with open(sys.argv[1]) as f:
    lines = [ln for ln in f if ln.startswith('"')]
for r in csv.DictReader(lines):
    if r.get("Metric Name") != "gpu__time_duration.sum":
        continue
    v = float(r["Metric Value"].replace(",", ""))
    unit = r.get("Metric Unit", "ns")
    ns = v * {"ns": 1, "usecond": 1e3, "us": 1e3, "msecond": 1e6, "ms": 1e6}.get(unit, 1)
    name = re.sub(r"\(.*", "", r["Kernel Name"]).replace("void ", "")
    name = re.sub(r"pp200::<unnamed>::|pp200::\(anonymous namespace\)::", "", name)
    rows.append((name, ns))
tot = sum(ns for _, ns in rows)
agg = defaultdict(lambda: [0, 0.0])
for n, ns in rows:
    agg[n][0] += 1
    agg[n][1] += ns
print(f"{len(rows)} launches, {tot / 1e6:.2f} ms serialized kernel time (ncu, cold caches)")
for n, (c, ns) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
    print(f"{ns / 1e6:8.3f} ms {100 * ns / tot:5.1f}%  x{c:5d}  {n}")
