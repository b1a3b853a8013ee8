"""Reclaimed byte images and the device preemption gate (sm_100a kernels).

Byte images: every page reported by apply_reclaim / the fused reclaim is gathered from its
physical slot into pinned host memory; the bytes must equal the C restatement's image of
(request, block) in report order -- bit-exact, through the SM copy kernel (LDG/STG and the
bulk-copy/TMA variant), the copy-engine baseline, and under a rate bound.

Gate: the gated offline kernel quiesces on a raised gate, never claims a tile afterwards,
and resumes from its HBM cursor so every tile runs exactly once across preemptions; a
reclaim issued without waiting for quiesce is caught by the quarantine canary.
"""
import ctypes as C
import random
import time

import numpy as np
import pytest

from paper_2604_07874_b200 import api as A

pytestmark = pytest.mark.gpu


def _expected_images(oracle_c, res, page_bytes):
    reqs, blks = [], []
    for r in res.evicted_requests:
        reqs += [r] * len(res.invalidated_pages[r])
        blks += res.block_index[r]
    n = len(reqs)
    out = np.zeros(n * page_bytes, dtype=np.uint8)
    rq = (C.c_int64 * max(n, 1))(*reqs)
    bk = (C.c_int32 * max(n, 1))(*blks)
    oracle_c.lib.vo_gather_images(rq, bk, n, page_bytes, out.ctypes.data)
    return out


def _pool_with_pages(rng, H=32, S=8, slot=16384, page=12288, n_req=40):
    pool = A.DevicePool(H, S, 16, slot_bytes=slot, page_bytes=page)
    live = []
    for r in range(n_req):
        if pool.offline_reserve(r * 7 + 3, rng.randint(1, 2 * S), r):
            live.append(r * 7 + 3)
    pool.fill_pages()
    pool.set_costs({r: rng.randint(1, 100) for r in live})
    return pool, live


@pytest.mark.parametrize("engine,kw", [
    ("sm", dict(ctas=4, chunk_bytes=4096)),
    ("sm", dict(ctas=1, threads=128, chunk_bytes=12288)),
    ("sm", dict(ctas=8, use_tma=1, chunk_bytes=8192)),
    ("sm", dict(ctas=3, chunk_bytes=4096, rate_bytes_per_s=2e9, burst_bytes=8192)),
    ("ce", {}),
])
def test_reclaim_byte_images(oracle_c, engine, kw):
    rng = random.Random(11)
    pool, live = _pool_with_pages(rng)
    _, _, n_pages = pool.reclaim(5, 1000)
    res = pool.last_reclaim()
    assert n_pages == sum(len(v) for v in res.invalidated_pages.values()) > 0
    buf = A.HostBuffer(n_pages * pool.page_bytes)
    st = pool.reclaim_copy(buf.ptr, buf.nbytes, A.copy_params(**kw) if kw else None, engine=engine)
    assert st.bytes == n_pages * pool.page_bytes
    want = _expected_images(oracle_c, res, pool.page_bytes)
    assert np.array_equal(buf.view(), want)
    if kw.get("rate_bytes_per_s"):
        # token bucket: the copy cannot finish before (bytes - burst) / rate
        floor_ns = (st.bytes - kw["burst_bytes"] - kw["chunk_bytes"]) / kw["rate_bytes_per_s"] * 1e9
        assert st.t_last_ns - st.t_first_ns >= floor_ns * 0.95


def test_apply_reclaim_copy_matches_explicit_ids(oracle_c):
    """apply_reclaim with caller-chosen handles -> the copy list follows its report."""
    rng = random.Random(3)
    pool, live = _pool_with_pages(rng)
    inst = pool.snapshot()
    ids = [h.id for h in inst.handles][::3][:4]
    res = pool.apply_reclaim(ids, 99)
    n = sum(len(v) for v in res.invalidated_pages.values())
    buf = A.HostBuffer(max(n, 1) * pool.page_bytes)
    pool.reclaim_copy(buf.ptr, buf.nbytes, A.copy_params(ctas=2, chunk_bytes=4096))
    assert np.array_equal(buf.view()[: n * pool.page_bytes], _expected_images(oracle_c, res, pool.page_bytes))


# ------------------------------------------------------------------------------ gate

def _offline_setup(torch, pool, reqs):
    rows = [pool.request_row(r) for r in reqs]
    npages = [pool.offline_pages_of(r) for r in reqs]
    cpp = -(-pool.page_bytes // 16384)  # default tile: 16 KiB
    total = sum(npages) * cpp
    t_rows = torch.tensor(rows, dtype=torch.int32, device="cuda")
    t_np = torch.tensor(npages, dtype=torch.int32, device="cuda")
    out = torch.full((total,), float("nan"), dtype=torch.float32, device="cuda")
    return t_rows, t_np, out, total


def test_gate_preempt_resume_conserves_work():
    torch = pytest.importorskip("torch")
    rng = random.Random(5)
    pool = A.DevicePool(64, 16, 16, slot_bytes=1 << 20, page_bytes=917504)
    reqs = []
    for r in range(40):
        if pool.offline_reserve(r, rng.randint(8, 40), 0):
            reqs.append(r)
    pool.fill_pages()
    t_rows, t_np, out_ref, total = _offline_setup(torch, pool, reqs)
    gate = A.Gate(0)
    # uninterrupted run (reference outputs)
    gate.reset_work()
    gate.launch_offline(pool, t_rows.data_ptr(), t_np.data_ptr(), len(reqs), total,
                        out_ref.data_ptr(), stream=gate.stream)
    torch.cuda.synchronize()
    assert gate.read().tiles_done == total
    # preempted runs: raise after a short delay, wait quiesce, resume from the cursor
    out = torch.full_like(out_ref, float("nan"))
    gate.reset_work()
    gen = 0
    preemptions = 0
    while True:
        gate.launch_offline(pool, t_rows.data_ptr(), t_np.data_ptr(), len(reqs), total, out.data_ptr(),
                            ctas=4)
        time.sleep(rng.uniform(0.0002, 0.0008))
        gen += 1
        gate.raise_(gen)
        gate.wait_quiesced(gen)
        torch.cuda.synchronize()
        s = gate.read()
        assert s.live_ctas == 0
        done = s.tiles_done
        # context save = cursor: every claimed tile finished before the CTA retired
        assert s.tiles_done == min(s.tiles_claimed, total)
        gate.release(gen)
        torch.cuda.synchronize()
        preemptions += 1
        if done >= total:
            break
        assert preemptions < 200
    assert gate.read().tiles_done == total
    a = out.view(torch.int32).cpu().numpy()
    b = out_ref.view(torch.int32).cpu().numpy()
    assert np.array_equal(a, b)  # every tile exactly once, bit-identical results
    assert preemptions >= 2


def test_gate_closed_before_launch_runs_nothing():
    torch = pytest.importorskip("torch")
    pool = A.DevicePool(8, 8, 16, slot_bytes=1 << 20, page_bytes=917504)
    assert pool.offline_reserve(1, 10, 0)
    pool.fill_pages()
    t_rows, t_np, out, total = _offline_setup(torch, pool, [1])
    gate = A.Gate(0)
    gate.reset_work()
    gate.raise_(1)
    gate.wait_quiesced(1)
    torch.cuda.synchronize()
    # the launch waits for an open gate: nothing runs while raised
    gate.launch_offline(pool, t_rows.data_ptr(), t_np.data_ptr(), 1, total, out.data_ptr(),
                        stream=None)
    time.sleep(0.05)
    assert gate.read().tiles_done == 0
    gate.release(2)
    torch.cuda.synchronize()
    pool_stream_sync = pool.view().stream  # the launch went to the pool's stream
    assert pool_stream_sync
    deadline = time.time() + 10
    while gate.read().tiles_done < total and time.time() < deadline:
        time.sleep(0.01)
    assert gate.read().tiles_done == total


def test_quarantine_canary_catches_ungated_reclaim():
    """Negative test (sim.cpp:1003-1008 fault detector): reclaiming while the
    offline kernel still runs makes it read remapped block-table entries -> canary hits."""
    torch = pytest.importorskip("torch")
    pool = A.DevicePool(16, 16, 16, slot_bytes=1 << 20, page_bytes=917504)
    reqs = [r for r in range(12) if pool.offline_reserve(r, 20, 0)]
    pool.fill_pages()
    pool.set_costs({r: 1 for r in reqs})
    t_rows, t_np, out, total = _offline_setup(torch, pool, reqs)
    gate = A.Gate(0)
    gate.reset_work()
    side = torch.cuda.Stream()
    # one CTA so the kernel is still walking the list when the reclaim lands
    gate.launch_offline(pool, t_rows.data_ptr(), t_np.data_ptr(), len(reqs), total, out.data_ptr(),
                        ctas=1, threads=64, stream=side.cuda_stream)
    time.sleep(0.002)
    pool.reclaim(8, 1)  # no gate raise, no quiesce wait (unsafe_skip_compute_gate analogue)
    side.synchronize()
    s = gate.read()
    assert s.canary_hits >= 1


def test_async_copy_overlaps_bookkeeping(oracle_c):
    """copy_start -> reserve/release calls on the pool stream -> wait: images unchanged; the
    next reclaim waits for the copy before rewriting the report."""
    rng = random.Random(21)
    pool, live = _pool_with_pages(rng)
    _, _, n_pages = pool.reclaim(4, 1000)
    res = pool.last_reclaim()
    buf = A.HostBuffer(n_pages * pool.page_bytes)
    pool.reclaim_copy_start(buf.ptr, buf.nbytes, A.copy_params(ctas=2, chunk_bytes=4096,
                                                                 rate_bytes_per_s=5e8))
    for r in res.evicted_requests:  # re-admit while the (rate-bounded) copy still runs
        pool.offline_reserve(r, 3, 1001)
    pool.reclaim(2, 1002)           # must not overwrite the report under the copy
    st = pool.reclaim_copy_wait()
    assert st.bytes == n_pages * pool.page_bytes
    assert np.array_equal(buf.view(), _expected_images(oracle_c, res, pool.page_bytes))
    pool.check_invariants()


def test_pipelined_copies_back_to_back_reclaims(oracle_c):
    """Two reclaim ops back to back with both copies in flight: the second decision rewrites
    the report while the first (rate-bounded) copy still streams; each copy works from its own
    snapshot, so both byte images match their own reports; waits complete FIFO."""
    rng = random.Random(33)
    pool, live = _pool_with_pages(rng, H=48, n_req=70)
    _, _, n1 = pool.reclaim(4, 1000)
    res1 = pool.last_reclaim()
    buf1 = A.HostBuffer(n1 * pool.page_bytes)
    pool.reclaim_copy_start(buf1.ptr, buf1.nbytes, A.copy_params(ctas=2, chunk_bytes=4096,
                                                                   rate_bytes_per_s=3e8))
    _, _, n2 = pool.reclaim(5, 1001)  # op 2 decides while op 1's bytes are in flight
    res2 = pool.last_reclaim()
    assert n2 > 0 and set(res2.handles).isdisjoint(res1.handles)
    buf2 = A.HostBuffer(n2 * pool.page_bytes)
    pool.reclaim_copy_start(buf2.ptr, buf2.nbytes, A.copy_params(ctas=4, chunk_bytes=8192))
    with pytest.raises(A.LogicError):  # the synchronous form needs an idle ring
        pool.reclaim_copy(buf2.ptr, buf2.nbytes)
    # the same report again until the ring (VALVE_COPY_RING slots) is full, then one more fails
    spare = A.HostBuffer(n2 * pool.page_bytes)
    for _ in range(A.COPY_RING - 2):
        pool.reclaim_copy_start(spare.ptr, spare.nbytes, A.copy_params(ctas=4, chunk_bytes=8192))
    with pytest.raises(A.LogicError):
        pool.reclaim_copy_start(spare.ptr, spare.nbytes)
    st1 = pool.reclaim_copy_wait()
    st2 = pool.reclaim_copy_wait()
    for _ in range(A.COPY_RING - 2):
        assert pool.reclaim_copy_wait().bytes == n2 * pool.page_bytes
    assert (st1.bytes, st2.bytes) == (n1 * pool.page_bytes, n2 * pool.page_bytes)
    assert np.array_equal(buf1.view(), _expected_images(oracle_c, res1, pool.page_bytes))
    assert np.array_equal(buf2.view(), _expected_images(oracle_c, res2, pool.page_bytes))
    with pytest.raises(A.LogicError):
        pool.reclaim_copy_wait()
    pool.check_invariants()


def test_pipelined_copies_per_request_page_sizes(oracle_c):
    """The ring also snapshots the variable-size layout (weight pages of a whole slot next to
    KV pages): op 2's report (other sizes, other offsets) cannot leak into op 1's copy."""
    rng = random.Random(8)
    slot, page = 65536, 49152
    pool = A.DevicePool(32, 8, 16, slot_bytes=slot, page_bytes=page)
    weights = {3_000_000 + i: 9 for i in range(4)}
    for w, n in weights.items():
        assert pool.offline_reserve(w, n, 0)
    kv = [r for r in range(60) if pool.offline_reserve(r, rng.randint(1, 6), 1)]
    sizes = {w: slot for w in weights}
    pool.set_page_bytes(sizes)
    pool.fill_pages()
    pool.set_costs({**{w: rng.randint(1, 10**6) for w in weights}, **{r: rng.randint(1, 100) for r in kv}})
    ids1 = sorted(set(pool.handles_of_request(3_000_000)) | set(pool.handles_of_request(kv[0])))
    res1 = pool.apply_reclaim(ids1, 10)
    tot1, _ = pool.last_copy_layout()
    buf1 = A.HostBuffer(tot1)
    pool.reclaim_copy_start(buf1.ptr, buf1.nbytes, A.copy_params(ctas=2, chunk_bytes=8192,
                                                                   rate_bytes_per_s=3e8))
    pool.reclaim(6, 11)
    res2 = pool.last_reclaim()
    tot2, _ = pool.last_copy_layout()
    buf2 = A.HostBuffer(max(tot2, 16))
    pool.reclaim_copy_start(buf2.ptr, buf2.nbytes, A.copy_params(ctas=3, chunk_bytes=16384))
    assert pool.reclaim_copy_wait().bytes == tot1
    assert pool.reclaim_copy_wait().bytes == tot2
    assert np.array_equal(buf1.view(), _expected_images_var(oracle_c, res1, sizes, page))
    assert np.array_equal(buf2.view()[:tot2], _expected_images_var(oracle_c, res2, sizes, page))


# ------------------------------------------------------------------- weight pages (C3)

@pytest.mark.parametrize("slot,page,n_w", [(16384, 12288, 21), (1 << 20, 917504, 48)])
def test_weight_pages_evict_restore_round_trip(oracle_c, slot, page, n_w):
    """Offline weight pages evicted with their handles go to host (gather) and come back
    (scatter) into freshly reserved slots; a second eviction must gather the same bytes."""
    rng = random.Random(slot + n_w)
    H, S = 24, 8
    W = 1_000_003
    pool = A.DevicePool(H, S, 16, slot_bytes=slot, page_bytes=page)
    assert pool.offline_reserve(W, n_w, 0)
    kv = [r for r in range(30) if pool.offline_reserve(r, rng.randint(1, 6), 1)]
    pool.fill_pages()
    blocks_w = list(range(n_w))
    # evict every handle holding a weight page
    res = pool.apply_reclaim(sorted(pool.handles_of_request(W)), 10)
    assert W in res.evicted_requests
    n = sum(len(v) for v in res.invalidated_pages.values())
    buf = A.HostBuffer(n * page)
    pool.reclaim_copy(buf.ptr, buf.nbytes, A.copy_params(ctas=4, chunk_bytes=4096))
    img = buf.view()
    assert np.array_equal(img, _expected_images(oracle_c, res, page))
    # weight pages out of the report, in block order, into their own staging buffer
    off, pos = 0, {}
    for r in res.evicted_requests:
        for b in res.block_index[r]:
            if r == W:
                pos[b] = off
            off += 1
    assert sorted(pos) == blocks_w
    wbuf = A.HostBuffer(n_w * page)
    order = rng.sample(blocks_w, n_w)  # restore takes any page -> block order
    for i, b in enumerate(order):
        wbuf.view()[i * page:(i + 1) * page] = img[pos[b] * page:(pos[b] + 1) * page]
    # give the handles back, let other requests churn the freed slots, re-admit the weights
    pool.online_release(len(res.handles))
    for r in range(100, 110):
        pool.offline_reserve(r, rng.randint(1, 4), 20)
    pool.fill_pages()
    assert pool.offline_reserve(W, n_w, 30)
    st = pool.restore(W, wbuf.ptr, order, A.copy_params(ctas=8, chunk_bytes=8192))
    assert st.bytes == n_w * page and st.kernel_ms > 0
    # second eviction: the weights' bytes must be the original images again
    res2 = pool.apply_reclaim(sorted(pool.handles_of_request(W)), 40)
    n2 = sum(len(v) for v in res2.invalidated_pages.values())
    buf2 = A.HostBuffer(n2 * page)
    pool.reclaim_copy(buf2.ptr, buf2.nbytes)
    got = buf2.view()
    want = _expected_images(oracle_c, res2, page)
    off = 0
    for r in res2.evicted_requests:
        k = len(res2.block_index[r])
        sl = slice(off * page, (off + k) * page)
        if r == W:
            assert np.array_equal(got[sl], want[sl])
        off += k
    assert W in res2.evicted_requests


def test_restore_rejects_bad_blocks():
    pool = A.DevicePool(8, 4, 16, slot_bytes=4096, page_bytes=4096)
    buf = A.HostBuffer(4 * 4096)
    with pytest.raises(A.LogicError):
        pool.restore(5, buf.ptr, [0])  # not reserved
    assert pool.offline_reserve(5, 3, 0)
    with pytest.raises(A.OutOfRange):
        pool.restore(5, buf.ptr, [0, 1 << 20])
    with pytest.raises(A.LogicError):
        pool.restore(5, buf.ptr, [3])  # block 3 is not mapped (3 pages)
    pool.restore(5, buf.ptr, [2, 0, 1])
    pool.check_invariants()


def _expected_images_var(oracle_c, res, sizes, default):
    """Byte images of a report with per-request page sizes: request e's pages (its own size)
    follow those of the earlier evicted requests."""
    parts = []
    for r in res.evicted_requests:
        blks = res.block_index[r]
        n = len(blks)
        pb = sizes.get(r, default)
        out = np.zeros(max(n, 1) * pb, dtype=np.uint8)
        rq = (C.c_int64 * max(n, 1))(*([r] * n))
        bk = (C.c_int32 * max(n, 1))(*blks)
        oracle_c.lib.vo_gather_images(rq, bk, n, pb, out.ctypes.data)
        parts.append(out[: n * pb])
    return np.concatenate(parts) if parts else np.zeros(0, np.uint8)


@pytest.mark.parametrize("engine,kw", [
    ("sm", dict(ctas=6, chunk_bytes=8192)),
    ("sm", dict(ctas=2, chunk_bytes=65536)),
    ("sm", dict(ctas=4, use_tma=1, chunk_bytes=8192)),  # variable sizes through the bulk-copy kernel
    ("ce", {}),
])
def test_weight_pages_fill_whole_slots(oracle_c, engine, kw):
    """C3 geometry in miniature: offline KV pages of page_bytes and weight pages that fill the
    whole slot, reclaimed together; the copy lays each request's pages out at its own size."""
    rng = random.Random(21)
    slot, page = 65536, 49152
    H, S = 24, 8
    pool = A.DevicePool(H, S, 16, slot_bytes=slot, page_bytes=page)
    weights = {2_000_000 + layer: 11 for layer in range(3)}  # three "layers" of 11 slots
    for w, n in weights.items():
        assert pool.offline_reserve(w, n, 0)
    kv = [r for r in range(40) if pool.offline_reserve(r, rng.randint(1, 6), 1)]
    sizes = {w: slot for w in weights}
    pool.set_page_bytes(sizes)
    pool.fill_pages()
    pool.set_costs({**{w: 10**9 for w in weights}, **{r: rng.randint(1, 100) for r in kv}})
    ids = sorted(set(pool.handles_of_request(2_000_001)) | set(pool.handles_of_request(0)))
    res = pool.apply_reclaim(ids, 10)
    assert 2_000_001 in res.evicted_requests
    total, pbs = pool.last_copy_layout()
    assert pbs == [sizes.get(r, page) for r in res.evicted_requests]
    want = _expected_images_var(oracle_c, res, sizes, page)
    assert total == len(want)
    buf = A.HostBuffer(total)
    st = pool.reclaim_copy(buf.ptr, buf.nbytes, A.copy_params(**kw) if kw else None, engine=engine)
    assert st.bytes == total
    assert np.array_equal(buf.view(), want)
    # the fused device reclaim reports the same layout
    pool.online_release(len(res.handles))
    t, n = 20, pool.reclaim(6, 20)
    res2 = pool.last_reclaim()
    total2, _ = pool.last_copy_layout()
    buf2 = A.HostBuffer(max(total2, 16))
    pool.reclaim_copy(buf2.ptr, buf2.nbytes, A.copy_params(ctas=3, chunk_bytes=16384))
    assert np.array_equal(buf2.view()[:total2], _expected_images_var(oracle_c, res2, sizes, page))


def test_weight_restore_uses_request_page_size(oracle_c):
    slot, page = 65536, 49152
    pool = A.DevicePool(16, 8, 16, slot_bytes=slot, page_bytes=page)
    W = 7_000_000
    assert pool.offline_reserve(W, 13, 0)
    pool.set_page_bytes({W: slot})
    pool.fill_pages()
    res = pool.apply_reclaim(sorted(pool.handles_of_request(W)), 5)
    total, _ = pool.last_copy_layout()
    assert total == 13 * slot
    buf = A.HostBuffer(total)
    pool.reclaim_copy(buf.ptr, buf.nbytes)
    pool.online_release(len(res.handles))
    assert pool.offline_reserve(W, 13, 6)
    pool.set_page_bytes({W: slot})
    order = res.block_index[W]
    st = pool.restore(W, buf.ptr, order)
    assert st.bytes == 13 * slot
    res2 = pool.apply_reclaim(sorted(pool.handles_of_request(W)), 7)
    buf2 = A.HostBuffer(13 * slot)
    pool.reclaim_copy(buf2.ptr, buf2.nbytes)
    assert np.array_equal(buf2.view(), _expected_images_var(oracle_c, res2, {W: slot}, page))


def test_set_page_bytes_validation():
    pool = A.DevicePool(8, 4, 16, slot_bytes=8192, page_bytes=4096)
    assert pool.offline_reserve(1, 2, 0)
    with pytest.raises(A.InvalidArgument):
        pool.set_page_bytes({1: 8192 + 16})
    with pytest.raises(A.InvalidArgument):
        pool.set_page_bytes({1: 100})
    with pytest.raises(A.InvalidArgument):
        pool.set_page_bytes({99: 4096})  # no live pages
    pool.set_page_bytes({1: 8192})
    pool.set_page_bytes({1: 0})
