"""Summarise ncu reports into profiles/: key metrics per kernel (duration, DRAM bytes, throughput
%s, occupancy, registers) and the top source lines by stall samples.
Usage: python tools/ncu_summary.py OUT.txt REPORT.ncu-rep [...]"""
import csv
import subprocess
import sys

KEYS = ["Duration", "Elapsed Cycles", "DRAM Throughput", "Memory Throughput", "Compute (SM) Throughput",
        "L2 Cache Throughput", "Achieved Occupancy", "Registers Per Thread", "Block Size", "Grid Size",
        "Dynamic Shared Memory Per Block", "Executed Ipc Active"]
RAW = ["dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__time_duration.sum",
       "lts__t_bytes.sum", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
       "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed"]


def summarize(rep):
    out = []
    det = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(det.splitlines()))
    if not rows:
        return [f"{rep}: empty"]
    h = rows[0]
    name = None
    seen = set()
    for r in rows[1:]:
        d = dict(zip(h, r))
        name = d.get("Kernel Name", name)
        m = d.get("Metric Name")
        if m in KEYS and m not in seen:
            seen.add(m)
            out.append(f"  {m:32s} {d.get('Metric Value')} {d.get('Metric Unit')}")
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rr = list(csv.reader(raw.splitlines()))
    if len(rr) > 2:
        hdr, units, vals = rr[0], rr[1], rr[2]
        for k in RAW:
            if k in hdr:
                i = hdr.index(k)
                out.append(f"  {k:32s} {vals[i]} {units[i]}")
    hot = subprocess.run([sys.executable, "tools/ncu_hot_lines.py", rep, "8"], capture_output=True, text=True).stdout
    return [f"== {name}  ({rep})"] + out + ["  top source lines by stall samples:"] + ["   " + l for l in hot.splitlines()]


def main():
    lines = []
    for rep in sys.argv[2:]:
        lines += summarize(rep) + [""]
    open(sys.argv[1], "w").write("\n".join(lines))
    print("\n".join(lines))


if __name__ == "__main__":
    main()
