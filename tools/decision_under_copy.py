"""Fused-decision wall time with the previous op's gather copy still crossing the link (as in the
pipelined bench) vs with the link idle, for several copy configurations.  The decision's results
come back over the same PCIe direction the copy saturates (the completion word in pinned host
memory, the report counts); a rate-bounded copy leaves headroom.  One JSON line per config."""
import json
import os
import statistics
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2604_07874_b200 import api as A  # noqa: E402


def main(k=36, reps=12):
    H = 1024
    pool = A.DevicePool(H, bench.HSZ, 16, slot_bytes=bench.SLOT, page_bytes=bench.PAGE,
                        max_requests=4096, max_pages_per_request=1024)
    pool.online_grow(-(-H // 10), 0)
    live, t = bench.populate(pool, bench.offline_requests(3, 4 * H))
    pool.set_costs({r: c for r, (p, c) in live.items()})
    hosts = [A.HostBuffer(k * bench.HSZ * bench.PAGE) for _ in range(2)]

    def restore(evicted):
        nonlocal t
        pool.online_release(k)
        for r in evicted:
            pages, cost = live.pop(r)
            t += 1
            if pool.offline_reserve(r, pages, t):
                live[r] = (pages, cost)
        pool.set_costs({r: live[r][1] for r in evicted if r in live})

    configs = [("idle", None), ("tma8", dict(ctas=8)), ("ldg8", dict(ctas=8, use_tma=0)),
               ("tma4", dict(ctas=4)), ("tma8_rate40", dict(ctas=8, rate_bytes_per_s=40e9, burst_bytes=8 << 20)),
               ("tma8_rate30", dict(ctas=8, rate_bytes_per_s=30e9, burst_bytes=8 << 20))]
    for name, kw in configs:
        walls = []
        for i in range(reps + 2):
            t += 10
            if kw is not None:  # a copy of the previous report is in flight while we decide
                pool.reclaim(k, t, 0)
                res = pool.last_reclaim()
                pool.reclaim_copy_start(hosts[i % 2].ptr, hosts[0].nbytes, A.copy_params(**kw))
                restore(res.evicted_requests)
                time.sleep(0.004)  # the copy is well under way (an op's copy takes ~39 ms)
            t += 10
            w0 = time.perf_counter()
            pool.reclaim(k, t, 0)
            w1 = time.perf_counter()
            res = pool.last_reclaim()
            if kw is not None:
                pool.reclaim_copy_wait()
            restore(res.evicted_requests)
            if i >= 2:
                walls.append((w1 - w0) * 1e6)
        torch.cuda.synchronize()
        print(json.dumps({"copy": name, "k": k, "decision_wall_us_p50": round(statistics.median(walls), 1),
                          "min": round(min(walls), 1), "max": round(max(walls), 1)}), flush=True)


if __name__ == "__main__":
    main()
