"""Pairs the per-step device times of two replayed runs (same plan => same decode steps in the same
order): ratio distribution colo/solo of the decode graph time, by step index.
usage: python tools/rt_steps.py SOLO_steps.json COLO_steps.json"""
import json
import sys

a, b = (json.load(open(p)) for p in sys.argv[1:3])
for key in ("decode_gpu_us", "prefill_us"):
    x, y = a[key], b[key]
    n = min(len(x), len(y))
    r = sorted(y[i] / x[i] for i in range(n) if x[i] > 0)
    if not r:
        continue
    q = lambda p: r[min(len(r) - 1, int(p / 100 * (len(r) - 1)))]  # noqa: E731
    print(f"{key}: n={n} (lens {len(x)} / {len(y)}) ratio mean {sum(r) / len(r):.4f} p10 {q(10):.4f} "
          f"p50 {q(50):.4f} p90 {q(90):.4f} p99 {q(99):.4f}; sums {sum(x[:n]) / 1e3:.1f} / {sum(y[:n]) / 1e3:.1f} ms")
    # drift over the run: mean ratio per tenth
    tenth = max(1, n // 10)
    print("  by tenth:", " ".join(f"{sum(y[i] / x[i] for i in range(s, min(n, s + tenth))) / len(range(s, min(n, s + tenth))):.3f}"
                                   for s in range(0, n, tenth)))
