"""Preempt-to-quiesce microbenchmark: stream-memop raise vs stamped-kernel raise, per tile size.
Host view = CUDA events on the gate stream around raise -> wait(live_ctas == 0); device view =
%globaltimer from the stamped raise to the first warp that saw the gate and to the last CTA's
retirement.  One JSON line per config."""
import json
import os
import random
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2604_07874_b200 import api as A  # noqa: E402


def pct(xs, p):
    xs = sorted(xs)
    return xs[min(len(xs) - 1, int(round(p / 100 * (len(xs) - 1))))]


def main(n=300):
    H = 256
    pool = A.DevicePool(H, bench.HSZ, 16, slot_bytes=bench.SLOT, page_bytes=bench.PAGE,
                        max_requests=4096, max_pages_per_request=1024)
    live, t = bench.populate(pool, bench.offline_requests(3, 4 * H))
    pool.fill_pages()
    gate = A.Gate(0)
    gstream = torch.cuda.ExternalStream(gate.stream)
    off = torch.cuda.Stream()
    rng = random.Random(1)
    gen = 0
    for tile in (8192, 16384, 32768, 65536):
        for stamped in (False, True):
            host, first, quies = [], [], []
            gate.reset_work()
            for i in range(n):
                gate.launch_offline(pool, None, None, 0, 0, None, stream=off.cuda_stream, tile_bytes=tile)
                d = time.perf_counter() + rng.uniform(100e-6, 400e-6)
                while time.perf_counter() < d:
                    pass
                gen += 1
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(gstream)
                (gate.raise_stamped if stamped else gate.raise_)(gen)
                gate.wait_quiesced(gen)
                e1.record(gstream)
                gate.release(gen)
                e1.synchronize()
                host.append(e0.elapsed_time(e1) * 1e3)
                s = gate.read()
                if stamped and s.t_first_seen_ns and s.t_quiesced_ns > s.t_raise_ns:
                    first.append((s.t_first_seen_ns - s.t_raise_ns) / 1e3)
                    quies.append((s.t_quiesced_ns - s.t_raise_ns) / 1e3)
                torch.cuda.synchronize()
                if s.tiles_claimed > 0.5 * sum(p for p, _ in live.values()) * (-(-bench.PAGE // tile)):
                    gate.reset_work()
            row = {"tile": tile, "raise": "kernel-stamped" if stamped else "stream-memop",
                   "host_p50_us": round(pct(host, 50), 2), "host_p99_us": round(pct(host, 99), 2),
                   "host_max_us": round(max(host), 2)}
            if quies:
                row.update(dev_first_seen_p50_us=round(pct(first, 50), 2),
                           dev_quiesce_p50_us=round(pct(quies, 50), 2),
                           dev_quiesce_p99_us=round(pct(quies, 99), 2))
            print(json.dumps(row), flush=True)


if __name__ == "__main__":
    main()
