"""Decision-path microbenchmark (device): per-phase device time of the fused reclaim
(instance build / Algorithm 1 / apply) and the per-call latency of the bookkeeping ops, at the
C2 geometry of bench.py.  Prints one JSON line."""
import json
import statistics
import sys
import time
import os

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import ctypes as C  # noqa: E402

import bench  # noqa: E402
from paper_2604_07874_b200 import api as A  # noqa: E402


def main(k=36, H=1024, reps=20):
    pool = A.DevicePool(H, bench.HSZ, 16, max_requests=4096, max_pages_per_request=1024)
    pool.online_grow(-(-H // 10), 0)
    reqs = bench.offline_requests(2604, 4 * H)
    live, t = bench.populate(pool, reqs)
    pool.set_costs({r: c for r, (p, c) in live.items()})
    f = pool._b.lib.valve_pool_reclaim_phases
    f.argtypes = [C.c_void_p, C.POINTER(C.c_int64)]
    phases, wall, reserve_us, release_us = [], [], [], []
    nxt = 0
    for i in range(reps):
        w0 = time.perf_counter()
        nh, ne, npg = pool.reclaim(k, t + 10 * i, 0)
        wall.append((time.perf_counter() - w0) * 1e6)
        out = (C.c_int64 * 5)()
        f(pool.handle, out)
        phases.append([out[j] / 1e3 for j in range(3)] + [out[3], out[4]])
        res = pool.last_reclaim()
        pool.online_release(k)
        for r in res.evicted_requests:
            pages, cost = live.pop(r)
            w0 = time.perf_counter()
            ok = pool.offline_reserve(r, pages, t)
            reserve_us.append((time.perf_counter() - w0) * 1e6)
            if ok:
                live[r] = (pages, cost)
        pool.set_costs({r: live[r][1] for r in res.evicted_requests if r in live})
    for r in list(live)[:50]:
        w0 = time.perf_counter()
        pool.offline_release(r)
        release_us.append((time.perf_counter() - w0) * 1e6)
    ph = list(zip(*phases))
    print(json.dumps({
        "k": k, "handles": H, "reps": reps,
        "instance_us": statistics.median(ph[0]), "select_us": statistics.median(ph[1]),
        "apply_us": statistics.median(ph[2]), "argmin_cycles": statistics.median(ph[3]), "update_cycles": statistics.median(ph[4]), "reclaim_call_wall_us": statistics.median(wall),
        "offline_reserve_call_us": statistics.median(reserve_us),
        "offline_release_call_us": statistics.median(release_us),
    }))


if __name__ == "__main__":
    main()


def sweep():
    for k in (1, 8, 36, 64):
        main(k=k, reps=10)
