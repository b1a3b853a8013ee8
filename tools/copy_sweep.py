"""Reclaim-copy parameter sweep on the C2 page geometry: SM copy (LDG/STG), bulk-copy (TMA)
variant and the copy-engine baseline, vs the pinned cudaMemcpy D2H peak.  One JSON line per
config (GB/s = bytes / CUDA-event kernel time)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2604_07874_b200 import api as A  # noqa: E402


def main():
    H = 256
    pool = A.DevicePool(H, bench.HSZ, 16, slot_bytes=bench.SLOT, page_bytes=bench.PAGE,
                        max_requests=4096, max_pages_per_request=1024)
    live, t = bench.populate(pool, bench.offline_requests(1, 4 * H))
    pool.set_costs({r: c for r, (p, c) in live.items()})
    _, _, npg = pool.reclaim(36, t + 1)
    host = A.HostBuffer(npg * bench.PAGE)
    peak = bench.link_peak_d2h(torch, torch.device("cuda", 0))
    print(json.dumps({"pages": npg, "bytes": npg * bench.PAGE, "link_peak_d2h_gbs": round(peak, 2)}))
    configs = [("ce", {})]
    for ctas in (8, 16, 32, 64, 148):
        for chunk in (65536, 131072):
            configs.append(("sm", dict(ctas=ctas, threads=512, chunk_bytes=chunk)))
    for ctas in (8, 16, 32, 64):
        configs.append(("sm", dict(ctas=ctas, use_tma=1, chunk_bytes=65536)))
    for engine, kw in configs:
        best = 0.0
        for _ in range(3):
            st = pool.reclaim_copy(host.ptr, host.nbytes, A.copy_params(**kw) if kw else None, engine=engine)
            best = max(best, st.bytes / (st.kernel_ms * 1e-3) / 1e9)
        print(json.dumps({"engine": engine, **kw, "gbs": round(best, 2), "frac": round(best / peak, 4)}))


if __name__ == "__main__":
    main()
