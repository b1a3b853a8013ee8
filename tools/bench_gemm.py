"""Gated offline GEMM throughput (tcgen05/TMA, sm_100a) vs cuBLAS (torch.matmul) on the Qwen2-7B
offline projection shapes, gate polled vs not polled, plus preempt-to-quiesce with the GEMM as
the offline tenant.  CUDA events on the launching stream; prints one JSON line."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_2604_07874_b200 import api as A  # noqa: E402

SHAPES = {  # Qwen2-7B: hidden 3584, intermediate 18944, qkv 3584 + 2 x 512
    "qkv": (4608, 3584), "o": (3584, 3584), "gate_up": (37888, 3584), "down": (3584, 18944)}


def timed(fn, stream, reps=10):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(reps):
        fn()
    e1.record(stream)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def main():
    m = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
    gate = A.Gate(0)
    st = torch.cuda.Stream()
    out = {"tokens": m, "shapes": {}}
    for name, (n, k) in SHAPES.items():
        a = torch.randn(m, k, device="cuda").to(torch.bfloat16)
        b = (torch.randn(n, k, device="cuda") * 0.02).to(torch.bfloat16)
        c = torch.empty(m, n, device="cuda", dtype=torch.bfloat16)
        flop = 2.0 * m * n * k

        def valve(poll=True, mode=0):
            gate.launch_gemm(a.data_ptr(), b.data_ptr(), c.data_ptr(), m, n, k, poll=poll, stream=st.cuda_stream,
                             fresh=True, mode=mode)

        with torch.cuda.stream(st):
            ms_poll = timed(lambda: valve(True), st)
            ms_nopoll = timed(lambda: valve(False), st)
            ms_single = timed(lambda: valve(True, 1), st)
            ms_cublas = timed(lambda: torch.matmul(a, b.t(), out=c), st)
        out["shapes"][name] = {"n": n, "k": k, "tflops_polled": round(flop / ms_poll / 1e9, 1),
                               "tflops_unpolled": round(flop / ms_nopoll / 1e9, 1),
                               "tflops_cublas": round(flop / ms_cublas / 1e9, 1),
                               "tflops_single_cta": round(flop / ms_single / 1e9, 1),
                               "ms_polled": round(ms_poll, 4)}
    # quiesce with the GEMM as the tenant
    n, k = SHAPES["gate_up"]
    a = torch.randn(8192, k, device="cuda").to(torch.bfloat16)
    b = (torch.randn(n, k, device="cuda") * 0.02).to(torch.bfloat16)
    c = torch.empty(8192, n, device="cuda", dtype=torch.bfloat16)
    gs = torch.cuda.ExternalStream(gate.stream)
    q = []
    for gen in range(1, 201):
        gate.reset_work()
        gate.launch_gemm(a.data_ptr(), b.data_ptr(), c.data_ptr(), 8192, n, k, stream=st.cuda_stream)
        time.sleep(0.0002 + 0.0003 * (gen % 5) / 5)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(gs)
        gate.raise_(gen)
        gate.wait_quiesced(gen)
        e1.record(gs)
        gate.release(gen)
        torch.cuda.synchronize()
        if gate.read().tiles_done < (8192 // 256) * (n // 256):  # pair tiles
            q.append(e0.elapsed_time(e1) * 1e3)
    q.sort()
    out["gemm_quiesce_us"] = {"n": len(q), "p50": round(q[len(q) // 2], 2),
                              "p99": round(q[min(len(q) - 1, int(0.99 * (len(q) - 1)))], 2), "max": round(q[-1], 2)}
    print(json.dumps(out))


if __name__ == "__main__":
    main()
