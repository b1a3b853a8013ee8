"""Gated offline GEMM (tcgen05 + TMA, sm_100a): numerics against a torch fp32 reference of the same
op, and the gate contract -- quiesce at tile granularity, resume from the HBM cursors, every
128x256 tile computed exactly once across preemptions (bit-identical to an uninterrupted run).
SURVEY §8f.2; work conservation as in SPEC.md:207 / test_sim.cpp:105-131."""
import random
import time

import pytest

from paper_2604_07874_b200 import api as A

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


def _operands(m, n, k, seed=0):
    g = torch.Generator(device="cuda").manual_seed(seed)
    a = torch.randn(m, k, device="cuda", generator=g).to(torch.bfloat16)
    b = (torch.randn(n, k, device="cuda", generator=g) * 0.02).to(torch.bfloat16)  # N(0, 0.02) weights
    return a, b


def _run(gate, a, b, c, **kw):
    gate.reset_work()
    gate.launch_gemm(a.data_ptr(), b.data_ptr(), c.data_ptr(), a.shape[0], b.shape[0], a.shape[1], **kw)
    torch.cuda.synchronize()


@pytest.mark.parametrize("mode", [1, 2])
@pytest.mark.parametrize("m,n,k", [(128, 256, 64), (256, 512, 3584), (384, 1024, 1024), (512, 4608, 3584),
                                   (1024, 2048, 192)])
def test_gemm_matches_fp32_reference(m, n, k, mode):
    a, b = _operands(m, n, k, seed=m + n + k)
    if mode == 2 and m % 256:  # CTA pairs tile M by 256: such a shape is refused up front
        c = torch.empty((m, n), dtype=torch.bfloat16, device="cuda")
        with pytest.raises(A.InvalidArgument):
            _run(A.Gate(0), a, b, c, mode=2)
        return
    c = torch.full((m, n), float("nan"), dtype=torch.bfloat16, device="cuda")
    gate = A.Gate(0)
    _run(gate, a, b, c, mode=mode)
    ref = a.float() @ b.float().t()
    # fp32 accumulation, one bf16 rounding of the output: |err| <= 2^-8 |ref| (+ accumulation-order slack)
    torch.testing.assert_close(c.float(), ref, rtol=8e-3, atol=2e-3 * ref.abs().max().item())
    s = gate.read()
    assert s.tiles_done == (m // (128 * mode)) * (n // 256) and s.live_ctas == 0


def test_gemm_pair_and_single_agree_bitwise():
    m, n, k = 512, 1024, 3584
    a, b = _operands(m, n, k, seed=5)
    gate = A.Gate(0)
    c1 = torch.empty((m, n), dtype=torch.bfloat16, device="cuda")
    c2 = torch.empty_like(c1)
    _run(gate, a, b, c1, mode=1)
    _run(gate, a, b, c2, mode=2, ctas=6)
    assert torch.equal(c1.view(torch.int16), c2.view(torch.int16))  # same K order per output tile


def test_gemm_ctas_fewer_than_tiles_and_no_poll():
    m, n, k = 512, 2048, 512
    a, b = _operands(m, n, k, seed=3)
    gate = A.Gate(0)
    c1 = torch.empty((m, n), dtype=torch.bfloat16, device="cuda")
    c2 = torch.empty_like(c1)
    _run(gate, a, b, c1, ctas=3)
    _run(gate, a, b, c2, poll=False)
    assert torch.equal(c1, c2)  # same tile -> same bits, whatever CTA ran it


@pytest.mark.parametrize("mode", [1, 2])
def test_gemm_preempt_resume_conserves_tiles(mode):
    m, n, k = 2048, 4864, 3584  # 304 tiles of ~0.23 GFLOP (152 pair tiles)
    a, b = _operands(m, n, k, seed=7)
    gate = A.Gate(0)
    c_ref = torch.empty((m, n), dtype=torch.bfloat16, device="cuda")
    _run(gate, a, b, c_ref, mode=1)
    total = (m // (128 * mode)) * (n // 256)
    c = torch.full_like(c_ref, float("nan"))
    gate.reset_work()
    rng = random.Random(1)
    gen = preemptions = 0
    while True:
        gate.launch_gemm(a.data_ptr(), b.data_ptr(), c.data_ptr(), m, n, k, ctas=4, mode=mode)
        time.sleep(rng.uniform(0.0001, 0.0005))
        gen += 1
        gate.raise_(gen)
        gate.wait_quiesced(gen)
        torch.cuda.synchronize()
        s = gate.read()
        assert s.live_ctas == 0
        assert s.tiles_done == min(s.tiles_claimed, total)  # claimed tiles all completed
        gate.release(gen)
        torch.cuda.synchronize()
        preemptions += 1
        if s.tiles_done >= total:
            break
        assert preemptions < 400
    assert preemptions >= 2
    assert torch.equal(c.view(torch.int16), c_ref.view(torch.int16))


def _drain(what, ev, gate, limit_s=10.0):
    """Wait for `ev` (an event or stream) with a deadline; a timeout fails with the gate state
    instead of hanging the session."""
    t0 = time.perf_counter()
    while not ev.query():
        if time.perf_counter() - t0 > limit_s:
            s = gate.read()
            pytest.fail(f"{what} did not complete: live_ctas={s.live_ctas} claimed={s.tiles_claimed} "
                        f"done={s.tiles_done} closed={s.closed} quiesced_gen={s.quiesced_gen}")


@pytest.mark.parametrize("mode", [1, 2])
def test_gemm_quiesce_is_one_tile(mode):
    m, n, k = 8192, 18944, 3584  # Qwen2-7B gate/up projection over 8192 tokens: 4,736 tiles
    a, b = _operands(m, n, k, seed=11)
    c = torch.empty((m, n), dtype=torch.bfloat16, device="cuda")
    gate = A.Gate(0)
    gs = torch.cuda.ExternalStream(gate.stream)
    total = (m // (128 * mode)) * (n // 256)
    side = torch.cuda.Stream()  # one stream for the whole test (pool streams are recycled)
    waits = []
    torch.cuda.synchronize()
    for gen in range(1, 21):
        gate.reset_work()
        gate.launch_gemm(a.data_ptr(), b.data_ptr(), c.data_ptr(), m, n, k, stream=side.cuda_stream, mode=mode)
        # raise once the kernel is running (a raise that lands before the launch's "gate open"
        # wait, or after the last tile, preempts nothing and is not a quiesce sample)
        deadline = time.perf_counter() + 0.5
        while gate.read().tiles_claimed < 300 and time.perf_counter() < deadline:
            pass
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(gs)
        gate.raise_(gen)
        gate.wait_quiesced(gen)
        e1.record(gs)
        _drain(f"quiesce wait (gen {gen})", e1, gate)
        gate.release(gen)
        _drain(f"gated GEMM launch (gen {gen})", side, gate)
        s = gate.read()
        assert s.live_ctas == 0
        assert s.tiles_done == min(s.tiles_claimed, total) <= total  # every claimed tile finished once
        if 0 < s.tiles_done < total:
            waits.append(e0.elapsed_time(e1) * 1e3)
    assert len(waits) >= 10, waits  # most raises really preempted the GEMM mid-run
    waits.sort()
    # one 256x256 (pair) / 128x256 tile x 3584 is ~0.23-0.47 GFLOP (~15-30 us on its SMs)
    assert waits[len(waits) // 2] < 100.0, waits


def test_gemm_rejects_bad_shapes():
    gate = A.Gate(0)
    a, b = _operands(128, 256, 64)
    c = torch.empty((128, 256), dtype=torch.bfloat16, device="cuda")
    with pytest.raises(A.InvalidArgument):
        gate.launch_gemm(a.data_ptr(), b.data_ptr(), c.data_ptr(), 100, 256, 64)
    with pytest.raises(A.InvalidArgument):
        gate.launch_gemm(a.data_ptr(), b.data_ptr(), c.data_ptr(), 128, 256, 48)
    with pytest.raises(A.InvalidArgument):
        gate.launch_gemm(0, b.data_ptr(), c.data_ptr(), 128, 256, 64)
    with pytest.raises(A.InvalidArgument):
        gate.launch_gemm(a.data_ptr(), b.data_ptr(), c.data_ptr(), 128, 256, 64, mode=2)
