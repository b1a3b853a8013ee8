"""Decision-path microbenchmark (device): per-phase device time of the fused reclaim
(instance build / Algorithm 1 / apply and its sub-phases) and the per-call latency of the
bookkeeping ops, at the C2 geometry of bench.py.  Prints one JSON line per k."""
import ctypes as C
import json
import os
import statistics
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2604_07874_b200 import api as A  # noqa: E402

NAMES = ["instance_us", "select_us", "apply_us", "argmin_cycles", "update_cycles",
         "apply_evrows_us", "apply_sort_us", "apply_release_us", "apply_erase_us",
         "apply_validate_us", "apply_collect_us", "apply_rank_us",
         "select_dense_us", "select_csr_us", "select_checks_us", "select_rounds_us"]


def main(k=36, H=1024, reps=20):
    pool = A.DevicePool(H, bench.HSZ, 16, max_requests=4096, max_pages_per_request=1024)
    pool.online_grow(-(-H // 10), 0)
    live, t = bench.populate(pool, bench.offline_requests(2604, 4 * H))
    pool.set_costs({r: c for r, (p, c) in live.items()})
    f = pool._b.lib.valve_pool_reclaim_phases
    f.argtypes = [C.c_void_p, C.POINTER(C.c_int64)]
    rows, wall, reserve_us, release_us = [], [], [], []
    for i in range(reps):
        w0 = time.perf_counter()
        pool.reclaim(k, t + 10 * i, 0)
        wall.append((time.perf_counter() - w0) * 1e6)
        out = (C.c_int64 * 16)()
        f(pool.handle, out)
        rows.append([out[j] / 1e3 if j not in (3, 4) else out[j] for j in range(16)])
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
    cols = list(zip(*rows))
    out = {"k": k, "handles": H, "reps": reps}
    out.update({n: round(statistics.median(c), 2) for n, c in zip(NAMES, cols)})
    out.update(reclaim_call_wall_us=round(statistics.median(wall), 1),
               offline_reserve_call_us=round(statistics.median(reserve_us), 1),
               offline_release_call_us=round(statistics.median(release_us), 1))
    print(json.dumps(out), flush=True)


def sweep():
    for k in (1, 8, 36, 64):
        main(k=k, reps=10)


if __name__ == "__main__":
    sweep() if "--sweep" in sys.argv else main()
