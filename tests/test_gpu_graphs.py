"""Gated offline kernels captured in CUDA graphs (north star (b): the gate is polled by the offline
model's persistent *and graph-captured* kernels).  The launch sequence -- wait for an open gate
(stream memop), publish the CTA count, the gated kernel -- is captured once and replayed; a raise
between replays still quiesces it and the HBM cursors still give exactly-once tiles."""
import random
import time

import pytest

from paper_2604_07874_b200 import api as A

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


def _capture(stream, fn):
    g = torch.cuda.CUDAGraph()
    with torch.cuda.stream(stream):
        fn()  # warm-up outside capture (one-time allocations)
    torch.cuda.synchronize()
    with torch.cuda.graph(g, stream=stream):
        fn()
    torch.cuda.synchronize()
    return g


def test_graph_captured_gemm_preempt_resume():
    m, n, k = 2048, 4864, 3584
    gen_ = torch.Generator(device="cuda").manual_seed(3)
    a = torch.randn(m, k, device="cuda", generator=gen_).to(torch.bfloat16)
    b = (torch.randn(n, k, device="cuda", generator=gen_) * 0.02).to(torch.bfloat16)
    ref = torch.empty(m, n, device="cuda", dtype=torch.bfloat16)
    c = torch.full_like(ref, float("nan"))
    gate = A.Gate(0)
    gate.launch_gemm(a.data_ptr(), b.data_ptr(), ref.data_ptr(), m, n, k, fresh=True, mode=1)
    torch.cuda.synchronize()
    side = torch.cuda.Stream()
    # the graph resumes from the cursors (fresh=False); 4 CTAs so a replay takes a while
    graph = _capture(side, lambda: gate.launch_gemm(a.data_ptr(), b.data_ptr(), c.data_ptr(), m, n, k, ctas=4,
                                                     mode=1, stream=side.cuda_stream))
    gate.reset_work()
    c.fill_(float("nan"))
    total = (m // 128) * (n // 256)
    rng = random.Random(2)
    gen = preemptions = 0
    while True:
        with torch.cuda.stream(side):
            graph.replay()
        time.sleep(rng.uniform(0.0002, 0.0006))
        gen += 1
        gate.raise_(gen)
        gate.wait_quiesced(gen)
        torch.cuda.synchronize()
        s = gate.read()
        assert s.live_ctas == 0 and s.tiles_done == min(s.tiles_claimed, total)
        gate.release(gen)
        torch.cuda.synchronize()
        preemptions += 1
        if s.tiles_done >= total:
            break
        assert preemptions < 400
    assert preemptions >= 2
    assert torch.equal(c.view(torch.int16), ref.view(torch.int16))


def test_graph_captured_decode_quiesces():
    pool = A.DevicePool(64, 16, 16, slot_bytes=1 << 20, page_bytes=917504)
    rng = random.Random(9)
    for r in range(40):
        pool.offline_reserve(r, rng.randint(8, 40), 0)
    pool.fill_pages()
    gate = A.Gate(0)
    side = torch.cuda.Stream()
    graph = _capture(side, lambda: gate.launch_offline(pool, None, None, 0, 0, None, ctas=8,
                                                       stream=side.cuda_stream))
    gate.reset_work()
    gs = torch.cuda.ExternalStream(gate.stream)
    waits = []
    for gen in range(1, 11):
        with torch.cuda.stream(side):
            graph.replay()
        time.sleep(0.0003)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(gs)
        gate.raise_(gen)
        gate.wait_quiesced(gen)
        e1.record(gs)
        gate.release(gen)
        torch.cuda.synchronize()
        assert gate.read().live_ctas == 0
        waits.append(e0.elapsed_time(e1) * 1e3)
    waits.sort()
    assert waits[len(waits) // 2] < 500.0, waits
    # a replay into a closed gate runs nothing until release
    gate.raise_(100)
    gate.wait_quiesced(100)
    torch.cuda.synchronize()
    before = gate.read().tiles_done
    with torch.cuda.stream(side):
        graph.replay()
    time.sleep(0.02)
    assert gate.read().tiles_done == before
    gate.release(100)
    torch.cuda.synchronize()
