"""Pool and selection operations while a gated offline launch is parked behind a closed gate.

Run as a subprocess by tests/test_gpu_parked.py (so a deadlock times out instead of hanging the
suite).  The tenant's stream waits on the gate word (cuStreamWaitValue32 closed == 0) until the
host reopens it, so nothing the host calls in between may wait for the whole device: a
device-synchronizing cudaFree / cudaMalloc in a growth path would wait for that stream while the
host that would release it is inside the call.  Exercised here: selection-buffer growth (a larger
host instance than any before), request-table growth (more live requests than the table's rows)
and a fused reclaim, all with the tenant parked; then the gate reopens and the tenant runs.

Usage: python tests/parked_tenant_probe.py [path/to/libvalve.so]
"""
import os
import random
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2604_07874_b200 import api as A  # noqa: E402

if len(sys.argv) > 1:  # A/B against another build of the library
    A.LIBVALVE = sys.argv[1]


def main():
    import torch

    rng = random.Random(11)
    pool = A.DevicePool(64, 16, 16, slot_bytes=1 << 20, page_bytes=917504, max_requests=8,
                        max_pages_per_request=64)
    live = {}
    for r in range(6):
        if pool.offline_reserve(r, rng.randint(4, 12), r):
            live[r] = rng.randint(100, 900)
    pool.set_costs(live)
    pool.fill_pages()
    small = pool.snapshot()
    small.cost = {r: live[r] for h in small.handles for r in h.requests}
    A.selective_reclaim(small, 1)  # selection buffers at their first (small) size

    gate = A.Gate(0)
    gate.raise_(1)
    torch.cuda.synchronize()
    off = torch.cuda.Stream()
    gate.reset_work()
    gate.launch_offline(pool, None, None, 0, 0, None, stream=off.cuda_stream)  # parks: gate closed
    print("parked", flush=True)

    # request-table growth (8 rows -> more) with the tenant parked
    for r in range(6, 40):
        if pool.offline_reserve(r, rng.randint(1, 6), r):
            live[r] = rng.randint(100, 900)
    pool.set_costs(live)
    print("table grown", flush=True)
    # selection-buffer growth: a host instance larger than any before
    big = A.ReclaimInstance()
    for i in range(400):
        big.handles.append(A.ReclaimHandle(i, i, [1000 + (i * 7 + j) % 300 for j in range(6)]))
    big.cost = {1000 + q: 10 + q for q in range(300)}
    pick = A.selective_reclaim(big, 5)
    assert len(pick) == 5
    print("selection grown", flush=True)
    res = pool.reclaim(2, 100)
    print("fused reclaim", res is not None, flush=True)
    pool.check_invariants()

    gate.release(1)  # the parked launch now runs over its frozen work list and the current pages
    off.synchronize()
    torch.cuda.synchronize()
    print("released", flush=True)


if __name__ == "__main__":
    main()
