"""Summarise `ncu --page source --csv --print-source cuda,sass` output: stall samples per CUDA
source line (top N).  Usage: python tools/ncu_hot_lines.py REPORT.ncu-rep [N]"""
import csv
import subprocess
import sys

rep = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 25
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(txt.splitlines()))
hdr = None
cur = None
agg = {}
for r in rows:
    if len(r) > 4 and r[0] == "Line No":
        hdr = r
        si = r.index("Warp Stall Sampling (All Samples)")
        continue
    if hdr is None or len(r) <= si:
        continue
    if r[0]:
        cur = (int(r[0]), r[1].strip())
        continue
    try:
        s = int(r[si])
    except ValueError:
        continue
    if cur:
        agg[cur] = agg.get(cur, 0) + s
tot = sum(agg.values()) or 1
for (ln, src), s in sorted(agg.items(), key=lambda x: -x[1])[:n]:
    print(f"{s / tot * 100:5.1f}%  L{ln:4d}  {src[:110]}")
