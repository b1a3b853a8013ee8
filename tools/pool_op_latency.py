"""Latency of a one-CTA pool op (offline_release + offline_reserve) while the colocation's other
device work runs: the gated offline tenant (Qwen2-7B GEMM chain on 64 SMs + KV decode pass on 16
CTAs) and/or rate-bounded reclaim copies in flight.  Prints one JSON line per condition with the
median / max call wall (us)."""
import json
import os
import statistics
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2604_07874_b200 import api as A  # noqa: E402
from paper_2604_07874_b200 import realtime as RT  # noqa: E402
import torch  # noqa: E402


def main():
    dev = torch.device("cuda", 0)
    chain = RT.qwen_chain(dev, 2048)
    pool = A.DevicePool(1024, 64, 16, device=0, slot_bytes=2 << 20, page_bytes=RT.QWEN_PAGE,
                        max_requests=4096, max_pages_per_request=512)
    pool.online_grow(103, 0)
    rid = 0
    while pool.offline_reserve(rid, 200, rid):
        rid += 1
    pool.fill_pages()
    live = list(range(rid))
    gate, ggate = A.Gate(0), A.Gate(0)
    gate.attach_peers([ggate])
    off, gst = torch.cuda.Stream(), torch.cuda.Stream()
    arena = A.HostBuffer(12 << 30)
    gi = [0]

    def tenant(decode=True, gemm=True):
        if decode:
            gate.reset_work()
            gate.launch_offline(pool, None, None, 0, 0, None, ctas=16, stream=off.cuda_stream)
        if gemm:
            a, b, c, m, n, k, tiles = chain[gi[0] % len(chain)]
            gi[0] += 1
            ggate.launch_gemm(a.data_ptr(), b.data_ptr(), c.data_ptr(), m, n, k, ctas=64,
                              stream=gst.cuda_stream, fresh=True)

    def copies(n_ops):
        offs = 0
        for i in range(n_ops):
            pool.reclaim(2, 10_000 + i, 0)
            total, _ = pool.last_copy_layout()
            pool.reclaim_copy_start(arena.ptr + offs, total, A.copy_params(ctas=8, rate_bytes_per_s=32e9,
                                                                            burst_bytes=64 << 20))
            offs += total
            pool.online_release(2)

    gen = [0]
    for name, with_tenant, n_copy in (("idle", False, 0), ("decode_pass", "d", 0), ("gemm", "g", 0),
                                      ("tenant", True, 0), ("copies", False, 6), ("tenant+copies", True, 6)):
        walls = []
        if with_tenant:
            tenant(decode=with_tenant in (True, "d"), gemm=with_tenant in (True, "g"))
        if n_copy:
            copies(n_copy)
        time.sleep(0.002)
        for i in range(40):
            r = live[(7 * i + len(name)) % len(live)]
            w0 = time.perf_counter()
            pool.offline_release(r)
            w1 = time.perf_counter()
            pool.offline_reserve(r, 200, 20_000 + i)
            w2 = time.perf_counter()
            walls += [(w1 - w0) * 1e6, (w2 - w1) * 1e6]
            if with_tenant in (True, "g") and ggate.read().live_ctas == 0:  # keep the GEMM chain busy
                a, b, c, m, n, k, tiles = chain[gi[0] % len(chain)]
                gi[0] += 1
                ggate.launch_gemm(a.data_ptr(), b.data_ptr(), c.data_ptr(), m, n, k, ctas=64,
                                  stream=gst.cuda_stream, fresh=True)
            time.sleep(0.001)
        gen[0] += 1
        gate.raise_(gen[0])
        gate.wait_quiesced(gen[0])
        gate.cancel_work()
        ggate.cancel_work()
        gate.release(gen[0])
        while True:
            try:
                pool.reclaim_copy_wait()
            except A.LogicError:
                break
        torch.cuda.synchronize()
        print(json.dumps({"condition": name, "median_us": round(statistics.median(walls), 1),
                          "p90_us": round(sorted(walls)[int(0.9 * len(walls))], 1), "max_us": round(max(walls), 1),
                          "argmax": walls.index(max(walls))}),
              flush=True)


if __name__ == "__main__":
    main()
