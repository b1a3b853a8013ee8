"""Does the online slowdown after a busy edge depend on how much memory the offline tenant
touched, or only on how many bytes it streamed?  (the colocated decode runs ~5-8 %
slower for a few hundred ms after each busy edge.)

A decode-shaped "online" step (bf16 weights of Llama-3-8B size, 16 GB, read once per step by
skinny GEMMs, batch 8) runs in bursts; between bursts an "offline" sweep streams the same number
of bytes either over a LARGE footprint (48 GB read once) or a SMALL one (1 GB read 48 times), or
nothing (idle for the same wall time).  Per-step device times after each gap, bucketed by the
time since the burst started, over the mean of the last steps of the previous burst.

usage: python tools/rt_footprint.py [reps]   -> one JSON line per gap kind
"""
import json
import statistics
import sys
import time

import torch

BUCKETS = ((0, 20, "<20ms"), (20, 100, "20-100ms"), (100, 500, "100-500ms"), (500, 1e9, ">500ms"))


def main(reps=8):
    dev = torch.device("cuda:0")
    torch.manual_seed(0)
    # 32 layers x (qkv 4096x6144, o 4096x4096, gate/up 4096x28672, down 14336x4096) bf16 ~ 14 GB
    shapes = [(6144, 4096), (4096, 4096), (28672, 4096), (4096, 14336)]
    W = [[torch.randn(s, device=dev, dtype=torch.bfloat16) * 0.01 for s in shapes] for _ in range(32)]
    x0 = torch.randn(8, 4096, device=dev, dtype=torch.bfloat16)

    def step():
        x = x0
        for lw in W:
            q = x @ lw[0].t()
            x = (q[:, :4096] @ lw[1].t())
            h = x @ lw[2].t()
            x = h[:, :14336] @ lw[3].t()
        return x

    big = torch.empty(48 << 30, dtype=torch.uint8, device=dev)
    small = torch.empty(1 << 30, dtype=torch.uint8, device=dev)
    big.fill_(1)
    small.fill_(1)
    sink = torch.zeros((), device=dev, dtype=torch.int64)

    def sweep(kind):
        if kind == "large":
            for c in big.view(torch.int64).split((1 << 30) // 8):  # 48 x 1 GB chunks, each once
                torch.sum(c, dim=0, dtype=torch.int64, out=sink)
        elif kind == "small":
            v = small.view(torch.int64)
            for _ in range(48):
                torch.sum(v, dim=0, dtype=torch.int64, out=sink)

    g = torch.cuda.CUDAGraph()
    step()
    torch.cuda.synchronize()
    with torch.cuda.graph(g):
        step()
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(400)]
    out = {}
    for kind in ("idle", "large", "small") * reps:
        # burst A (baseline tail), gap, burst B (measured)
        for _ in range(100):
            g.replay()
        torch.cuda.synchronize()
        a0 = [torch.cuda.Event(enable_timing=True) for _ in range(21)]
        for i in range(20):
            a0[i].record()
            g.replay()
        a0[20].record()
        t_gap = time.perf_counter()
        sweep(kind)
        torch.cuda.synchronize()
        if kind == "idle":
            time.sleep(0.010)
        gap_ms = (time.perf_counter() - t_gap) * 1e3
        for b, e in evs:
            b.record()
            g.replay()
            e.record()
        torch.cuda.synchronize()
        base = statistics.mean(a0[i].elapsed_time(a0[i + 1]) for i in range(20))
        t = 0.0
        rows = out.setdefault(kind, {n: [] for _, _, n in BUCKETS})
        out.setdefault(kind + "_gap_ms", []).append(gap_ms)
        for b, e in evs:
            ms = b.elapsed_time(e)
            for lo, hi, n in BUCKETS:
                if lo <= t < hi:
                    rows[n].append(ms / base)
            t += ms
    for kind in ("idle", "large", "small"):
        print(json.dumps({"gap": kind, "gap_ms": round(statistics.median(out[kind + "_gap_ms"]), 1),
                          "step_ratio_by_time_since_burst_start":
                              {n: [len(v), round(statistics.mean(v), 4) if v else None]
                               for n, v in out[kind].items()}}), flush=True)


if __name__ == "__main__":
    main(int(sys.argv[1]) if len(sys.argv) > 1 else 8)
