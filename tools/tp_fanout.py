"""TP-group gate fan-out latency vs group size, one process per member, all on one GPU (the only
multi-process topology this run has).  Every member runs its gated offline kernel; the leader
raises the group gate (stream memops on every member's words through CUDA IPC) and waits for
every member's CTAs to retire.  Prints one JSON line per group size."""
import json
import os
import socket
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch.multiprocessing as mp  # noqa: E402


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def worker(rank, world, port, iters, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch
    import torch.distributed as dist

    from paper_2604_07874_b200 import api as A
    from paper_2604_07874_b200 import tp as TP

    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    gate = A.Gate(0)
    grp = TP.TPGate(gate, rank, world, world, dist, opener=lambda h: A.Gate.open_remote(h, 0))
    pool = A.DevicePool(32, 16, 16, slot_bytes=1 << 20, page_bytes=917504)
    for r in range(32):
        pool.offline_reserve(r, 16, 0)
    pool.fill_pages()
    s = torch.cuda.Stream()
    lat = []
    for it in range(iters):
        gate.reset_work()
        gate.launch_offline(pool, None, None, 0, 0, None, ctas=max(1, 64 // world), stream=s.cuda_stream)
        dist.barrier()
        if grp.is_leader:
            time.sleep(0.0003)
            gs = torch.cuda.ExternalStream(gate.stream)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(gs)
            grp.raise_(it + 1)
            grp.wait_quiesced(it + 1)
            e1.record(gs)
            e1.synchronize()
            lat.append(e0.elapsed_time(e1) * 1e3)
        dist.barrier()
        if grp.is_leader:
            grp.release(it + 1)
            torch.cuda.synchronize()
        dist.barrier()
        s.synchronize()
    if grp.is_leader:
        lat.sort()
        q.put({"group": world, "p50_us": lat[len(lat) // 2], "p99_us": lat[int(0.99 * (len(lat) - 1))],
               "max_us": lat[-1], "iters": iters})
    dist.barrier()
    dist.destroy_process_group()


def main():
    ctx = mp.get_context("spawn")
    for world in [int(x) for x in (sys.argv[1] if len(sys.argv) > 1 else "1,2,4,8").split(",")]:
        q = ctx.Queue()
        port = _port()
        ps = [ctx.Process(target=worker, args=(r, world, port, 200, q)) for r in range(world)]
        for p in ps:
            p.start()
        print(json.dumps(q.get(timeout=600)), flush=True)
        for p in ps:
            p.join(120)


if __name__ == "__main__":
    main()
