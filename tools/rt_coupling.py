"""Where does a colocated online step lose time?  One B200, the real-time harness's models:
for each offline-tenant configuration, run the tenant in a gap of `gap_ms`, raise the gate, wait
for the quiesce, then time the next online decode iterations (CUDA events on the online stream)
and sample the SM clock (NVML) right before each.  Compare with the same sequence after an idle
gap.  One JSON line per configuration: per-iteration ms (mean over repeats) and clocks.

usage: python tools/rt_coupling.py [gap_ms] [repeats]"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_2604_07874_b200 import api as A  # noqa: E402
from paper_2604_07874_b200 import realtime as RT  # noqa: E402


def main(gap_ms=200.0, repeats=12, iters=24, B=24, ctx=3000, spread="low"):
    import pynvml

    pynvml.nvmlInit()
    hnd = pynvml.nvmlDeviceGetHandleByIndex(0)
    dev = torch.device("cuda", 0)
    shape = RT.ModelShape()
    model = RT.OnlineModel(shape, dev)
    pool = A.DevicePool(1024, 64, 16, device=0, slot_bytes=shape.page_bytes, page_bytes=RT.QWEN_PAGE,
                        max_requests=4096, max_pages_per_request=512)
    model.bind(pool)
    chain = RT.qwen_chain(dev, 2048)
    # offline KV for the decode pass: fill the upper half of the pool
    pool.online_grow(128, 0)
    r = 0
    while r < 200 and pool.offline_reserve(r, 200, r):
        r += 1
    pool.fill_pages()
    S = pool.handle_size_pages()
    # contiguous online slots, or the same count spread over the whole 128 GiB page store (the
    # colocated runs' online pages sit in reclaimed handles all over the pool)
    n = 128 * S
    slots = {"low": list(range(0, n)), "high": list(range(1024 * S - n, 1024 * S)),
             "mid": list(range(448 * S, 448 * S + n)),
             "spread": [(i * 8 + i // 128) % (1024 * S) for i in range(n)]}[spread]
    npg = -(-ctx // 16)
    tables = [slots[b * npg:(b + 1) * npg] for b in range(B)]
    model.decode([1] * B, [t[-1] for t in tables], [ctx] * B, tables, slots[-1])
    online = torch.cuda.Stream(device=dev, priority=-1)
    off, gst = torch.cuda.Stream(device=dev), torch.cuda.Stream(device=dev)
    gate, ggate = A.Gate(0), A.Gate(0)
    gate.attach_peers([ggate])
    configs = [("idle", -1, -1)]
    gen = 0
    gi = 0
    for name, dctas, gctas in configs:
        per_it = [[] for _ in range(iters)]
        clk = [[] for _ in range(iters)]
        for rep in range(repeats + 1):
            gen += 1
            if dctas >= 0:
                gate.reset_work()
                gate.launch_offline(pool, None, None, 0, 0, None, ctas=dctas, stream=off.cuda_stream)
            if gctas >= 0:
                a, b_, c, m, n, k, tiles = chain[gi % len(chain)]
                gi += 1
                ggate.launch_gemm(a.data_ptr(), b_.data_ptr(), c.data_ptr(), m, n, k, ctas=gctas,
                                  stream=gst.cuda_stream, fresh=True)
            time.sleep(gap_ms / 1e3)
            gate.raise_(gen, online.cuda_stream)
            gate.wait_quiesced(gen, online.cuda_stream)
            evs = []
            for it in range(iters):
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                clock = pynvml.nvmlDeviceGetClockInfo(hnd, pynvml.NVML_CLOCK_SM)
                with torch.cuda.stream(online):
                    e0.record(online)
                    model.decode([1] * B, [t[-1] for t in tables], [ctx] * B, tables, slots[-1])
                    e1.record(online)
                online.synchronize()
                evs.append((e0, e1, clock))
            gate.cancel_work()
            ggate.cancel_work()
            gate.release(gen, online.cuda_stream)
            torch.cuda.synchronize()
            if rep:
                for it, (e0, e1, clock) in enumerate(evs):
                    per_it[it].append(e0.elapsed_time(e1))
                    clk[it].append(clock)
        ms = [sum(x) / len(x) for x in per_it]
        print(json.dumps({"tenant": name, "spread": spread, "gap_ms": gap_ms, "batch": B, "ctx": ctx,
                          "iter_ms": [round(x, 3) for x in ms], "mean_ms": round(sum(ms) / len(ms), 4),
                          "first4_ms": round(sum(ms[:4]) / 4, 4), "last8_ms": round(sum(ms[-8:]) / 8, 4),
                          "sm_mhz": [round(sum(c) / len(c)) for c in clk]}), flush=True)


if __name__ == "__main__":
    main(float(sys.argv[1]) if len(sys.argv) > 1 else 200.0, int(sys.argv[2]) if len(sys.argv) > 2 else 12,
         spread=sys.argv[3] if len(sys.argv) > 3 else "low")
