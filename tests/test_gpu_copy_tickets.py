"""Landed tickets and the cross-copy rate bound of the reclaim gather copy (sm_100a).

* Tickets (SURVEY §7 hard part 2: when may a reclaimed slot be rewritten?).  The SM copy runs
  wave-major -- wave w = bytes [w*chunk, (w+1)*chunk) of every reclaimed page -- and publishes
  each wave to a monotone pool counter once all its chunks have been read out of HBM.  The test
  plays the online tenant: on its own stream it waits for each wave's ticket and immediately
  overwrites exactly that byte range of every reclaimed slot.  If a wave were published before
  its bytes were read, the host image would contain the overwrite; it must equal the oracle's.
* Rate bound per window, across copies: two back-to-back copies with a chunk issue-time trace;
  every window [t_i, t_j] of the merged trace may carry at most rate*(t_j - t_i) + burst + one
  chunk of bytes (the bucket persists in the pool instead of restarting at each launch).
"""
import random

import numpy as np
import pytest

from paper_2604_07874_b200 import api as A
from test_gpu_copy_gate import _expected_images, _pool_with_pages

pytestmark = pytest.mark.gpu


def _slot_tensor(torch, pool):
    """The pool's page store as a uint8 [slots, slot_bytes] torch tensor (no copy)."""
    v = pool.view()
    n = pool.total_handles() * pool.handle_size_pages()

    class _Arr:
        __cuda_array_interface__ = {"shape": (n, v.slot_bytes), "typestr": "|u1",
                                    "data": (v.pages, False), "version": 3}

    return torch.as_tensor(_Arr(), device=f"cuda:{pool.device}")


@pytest.mark.parametrize("use_tma", [0, 1])
def test_tickets_guard_every_wave_against_online_overwrites(oracle_c, use_tma):
    """Both copy kernels (register-staged LDG/STG and shared-memory staged cp.async.bulk) publish
    waves only after the wave's bytes were read out of HBM."""
    torch = pytest.importorskip("torch")
    rng = random.Random(5)
    pool, live = _pool_with_pages(rng, H=48, S=8, slot=65536, page=49152, n_req=80)
    _, _, n_pages = pool.reclaim(6, 1000)
    res = pool.last_reclaim()
    want = _expected_images(oracle_c, res, pool.page_bytes)
    phys = torch.tensor([p for r in res.evicted_requests for p in res.physical_pages[r]],
                        device="cuda", dtype=torch.long)
    buf = A.HostBuffer(n_pages * pool.page_bytes)
    chunk = 8192
    slots = _slot_tensor(torch, pool)
    assert slots.data_ptr() == pool.view().pages  # a view of the page store, not a copy
    online = torch.cuda.Stream()
    with torch.cuda.stream(online):  # first-use costs outside the race below
        pool.wait_landed(0, online.cuda_stream)
        slots[phys[:1], 0:16] = slots[phys[:1], 0:16]
        torch.cuda.Event(enable_timing=True).record(online)
    online.synchronize()
    # slow enough (0.1 GB/s, ~24 ms) that an early overwrite would certainly beat the copy
    pool.reclaim_copy_start(buf.ptr, buf.nbytes, A.copy_params(ctas=3, chunk_bytes=chunk, use_tma=use_tma,
                                                                 rate_bytes_per_s=1e8, burst_bytes=chunk))
    base, waves, wave_bytes = pool.copy_ticket()
    assert waves == -(-pool.page_bytes // chunk) and wave_bytes == chunk
    events = []
    with torch.cuda.stream(online):
        e_start = torch.cuda.Event(enable_timing=True)
        e_start.record(online)
        for w in range(waves):
            pool.wait_landed(base + w + 1, online.cuda_stream)
            lo, hi = w * chunk, min((w + 1) * chunk, pool.page_bytes)
            slots[phys, lo:hi] = 0xA5  # the online tenant's writes into the reclaimed slots
            e = torch.cuda.Event(enable_timing=True)
            e.record(online)
            events.append(e)
    st = pool.reclaim_copy_wait()
    online.synchronize()
    assert np.array_equal(buf.view(), want), "a wave was published before its bytes were read"
    landed, issued = pool.landed()
    assert landed == issued == base + waves
    # the overwrites really landed in the page store, wave after wave over the copy's duration
    assert bool((slots[phys, :pool.page_bytes] == 0xA5).all())
    rel = [e_start.elapsed_time(e) for e in events]
    assert rel[0] < 0.5 * st.kernel_ms and rel[-1] > 0.7 * st.kernel_ms, (rel, st.kernel_ms)
    assert all(b > a for a, b in zip(rel, rel[1:])), rel


def test_tickets_accumulate_across_pipelined_copies(oracle_c):
    torch = pytest.importorskip("torch")
    rng = random.Random(6)
    pool, live = _pool_with_pages(rng, H=48, n_req=70)
    _, _, n1 = pool.reclaim(4, 1000)
    res1 = pool.last_reclaim()
    b1 = A.HostBuffer(n1 * pool.page_bytes)
    pool.reclaim_copy_start(b1.ptr, b1.nbytes, A.copy_params(ctas=2, chunk_bytes=4096, rate_bytes_per_s=3e8))
    base1, w1, _ = pool.copy_ticket()
    _, _, n2 = pool.reclaim(5, 1001)
    res2 = pool.last_reclaim()
    b2 = A.HostBuffer(n2 * pool.page_bytes)
    pool.reclaim_copy_start(b2.ptr, b2.nbytes, A.copy_params(ctas=4, chunk_bytes=4096, use_tma=1))
    base2, w2, wb2 = pool.copy_ticket()
    assert base2 == base1 + w1 and w2 == -(-pool.page_bytes // 4096) and wb2 == 4096  # TMA: wave-major too
    with pytest.raises(A.InvalidArgument):
        pool.wait_landed(base2 + w2 + 1)
    s = torch.cuda.Stream()
    pool.wait_landed(base2 + w2, s.cuda_stream)
    e = torch.cuda.Event()
    e.record(s)
    pool.reclaim_copy_wait()
    pool.reclaim_copy_wait()
    e.synchronize()
    assert pool.landed() == (base2 + w2, base2 + w2)
    assert np.array_equal(b1.view(), _expected_images(oracle_c, res1, pool.page_bytes))
    assert np.array_equal(b2.view(), _expected_images(oracle_c, res2, pool.page_bytes))


def test_rate_bound_holds_per_window_across_copies(oracle_c):
    torch = pytest.importorskip("torch")
    rng = random.Random(7)
    pool, live = _pool_with_pages(rng, H=64, S=8, slot=65536, page=65536, n_req=110)
    rate, burst, chunk = 2e9, 256 << 10, 16384
    k = 6
    cap = k * pool.handle_size_pages()  # pages per op at most
    # everything allocated up front (cudaHostAlloc blocks for ms): the second copy is queued
    # right behind the first, so the two share the bucket with no idle gap between them
    bufs = [A.HostBuffer(cap * pool.page_bytes) for _ in range(2)]
    traces = [torch.zeros(cap * (pool.page_bytes // chunk), dtype=torch.int64, device="cuda") for _ in range(2)]
    torch.cuda.synchronize()
    ns = []
    for op in range(2):
        _, _, n = pool.reclaim(k, 1000 + op)
        ns.append(n * (pool.page_bytes // chunk))
        pool.reclaim_copy_start(bufs[op].ptr, bufs[op].nbytes,
                                A.copy_params(ctas=4, chunk_bytes=chunk, rate_bytes_per_s=rate, burst_bytes=burst,
                                              trace=traces[op].data_ptr()))
    for _ in range(2):
        pool.reclaim_copy_wait()
    tr = [traces[i][: ns[i]].cpu().numpy().astype(np.int64) for i in range(2)]
    t = np.sort(np.concatenate(tr))
    assert t.size > 100 and (t > 0).all()
    ns_per_byte = 1e9 / rate
    # bytes started in [t_i, t_j] vs the budget, for every pair (two-pointer over the sorted trace)
    worst = -1e30
    for i in range(t.size):
        n = np.arange(1, t.size - i + 1)
        span = (t[i:] - t[i]).astype(np.float64)
        excess = n * chunk - (span / ns_per_byte + burst + chunk)
        worst = max(worst, float(excess.max()))
    # %globaltimer granularity and the sleep loop: allow one more chunk of slack
    assert worst <= chunk, worst
    # the second copy started right behind the first and got no fresh burst (a per-launch bucket
    # would start its first burst/chunk chunks at once)
    t1, t2 = np.sort(tr[0]), np.sort(tr[1])
    m = burst // chunk
    assert t2[0] - t1[-1] < 0.25 * burst * ns_per_byte, (t2[0] - t1[-1])
    assert t2[m - 1] - t2[0] >= 0.5 * (m - 1) * chunk * ns_per_byte, (t2[:m] - t2[0])
