"""Reclaim-copy throughput with the gated offline decode pass running beside it (HBM saturated by
the tenant, as between two pipelined reclaim ops) vs alone, for several copy CTA counts."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2604_07874_b200 import api as A  # noqa: E402


def main():
    H = 512
    pool = A.DevicePool(H, bench.HSZ, 16, slot_bytes=bench.SLOT, page_bytes=bench.PAGE,
                        max_requests=4096, max_pages_per_request=1024)
    live, t = bench.populate(pool, bench.offline_requests(1, 4 * H))
    pool.set_costs({r: c for r, (p, c) in live.items()})
    pool.fill_pages()
    _, _, npg = pool.reclaim(36, t + 1)
    host = A.HostBuffer(npg * bench.PAGE)
    gate = A.Gate(0)
    off = torch.cuda.Stream()
    peak = bench.link_peak_d2h(torch, torch.device("cuda", 0))
    print(json.dumps({"pages": npg, "link_peak_d2h_gbs": round(peak, 2)}), flush=True)
    gen = 0
    for ctas in (8, 16, 32, 64):
        for loaded in (False, True):
            best = 0.0
            for _ in range(3):
                if loaded:
                    gate.reset_work()
                    gate.launch_offline(pool, None, None, 0, 0, None, stream=off.cuda_stream)
                st = pool.reclaim_copy(host.ptr, host.nbytes, A.copy_params(ctas=ctas))
                if loaded:
                    gen += 1
                    gate.raise_(gen)
                    gate.wait_quiesced(gen)
                    gate.release(gen)
                torch.cuda.synchronize()
                best = max(best, st.bytes / (st.kernel_ms * 1e-3) / 1e9)
            print(json.dumps({"ctas": ctas, "offline_running": loaded, "gbs": round(best, 2),
                              "frac": round(best / peak, 4)}), flush=True)


if __name__ == "__main__":
    main()
