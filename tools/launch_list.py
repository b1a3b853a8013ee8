"""Per-kernel summary of an ncu launch list (`--metrics gpu__time_duration.sum --csv`).
Usage: python tools/launch_list.py launches.csv "header line" > profiles/<name>.txt"""
import csv
import re
import sys
from collections import defaultdict

rows = list(csv.reader(l for l in open(sys.argv[1]) if not l.startswith("==")))
h = rows[0]
ki, mi, vi, ui = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("Metric Unit")
agg = defaultdict(lambda: [0, 0.0])
for r in rows[1:]:
    if len(r) <= vi or r[mi] != "gpu__time_duration.sum":
        continue
    name = re.sub(r"\(.*", "", r[ki]).replace("valve::", "")
    scale = {"ns": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3, "nsecond": 1e-3}.get(r[ui], 1.0)
    agg[name][0] += 1
    agg[name][1] += float(r[vi].replace(",", "")) * scale
tot = sum(v[1] for v in agg.values())
print("# ncu launch list (gpu__time_duration.sum, --clock-control none): " + (sys.argv[2] if len(sys.argv) > 2 else ""))
print("# cold-cache, serialised by ncu: compare SHARES, not absolutes.")
print(f"{'kernel':40s} {'launches':>9s} {'total_ms':>10s} {'avg_us':>10s} {'share':>6s}")
for k, (n, us) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
    print(f"{k:40s} {n:9d} {us / 1e3:10.2f} {us / n:10.1f} {us / tot * 100:5.1f}%")
