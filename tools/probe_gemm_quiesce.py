"""Diagnostic: per-preemption tile accounting of the gated GEMM (tiles done / claimed / total)."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2604_07874_b200 import api as A  # noqa: E402


def main(mode, iters=40, m=8192, n=18944, k=3584, sleep=0.0003):
    g = torch.Generator(device="cuda").manual_seed(11)
    a = torch.randn(m, k, device="cuda", generator=g).to(torch.bfloat16)
    b = (torch.randn(n, k, device="cuda", generator=g) * 0.02).to(torch.bfloat16)
    c = torch.empty((m, n), dtype=torch.bfloat16, device="cuda")
    gate = A.Gate(0)
    gs = torch.cuda.ExternalStream(gate.stream)
    total = (m // (128 * mode)) * (n // 256)
    for gen in range(1, iters + 1):
        gate.reset_work()
        s0 = gate.read()
        side = torch.cuda.Stream()
        gate.launch_gemm(a.data_ptr(), b.data_ptr(), c.data_ptr(), m, n, k, stream=side.cuda_stream, mode=mode)
        time.sleep(sleep)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(gs)
        gate.raise_(gen)
        gate.wait_quiesced(gen)
        e1.record(gs)
        gate.release(gen)
        torch.cuda.synchronize()
        s = gate.read()
        print(json.dumps({"mode": mode, "gen": gen, "total": total, "done0": s0.tiles_done, "done": s.tiles_done,
                          "claimed": s.tiles_claimed, "live": s.live_ctas,
                          "wait_us": round(e0.elapsed_time(e1) * 1e3, 1)}))


if __name__ == "__main__":
    for mode in (1, 2):
        main(mode)
