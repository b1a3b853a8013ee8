"""TP-group gate fan-out latency vs group size, one process per member (rank r on cuda:r when the
box has a GPU per rank; on a 1-GPU box the members share the device -- functional only).  Every
member runs its gated offline kernel; the leader raises the group gate (stream memops on every
member's words through CUDA IPC / NVLink peer memory) and waits for every member's CTAs to retire
(paper_2604_07874_b200.tp.measure_group_fanout).  Prints one JSON line per group size."""
import json
import os
import socket
import sys

os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")  # before any CUDA context

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

    gpu, shared = TP.rank_device(rank, world, torch.cuda.device_count())
    torch.cuda.set_device(gpu)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    gate = A.Gate(gpu)
    grp = TP.TPGate(gate, rank, world, world, dist, opener=TP.open_member(gpu))
    pool = A.DevicePool(512, 16, 16, device=gpu, slot_bytes=1 << 20, page_bytes=917504)  # a pass of ~7 GB
    for r in range(512):
        pool.offline_reserve(r, 16, 0)
    pool.fill_pages()
    lat, errs, viol = TP.measure_group_fanout(torch, gate, grp, pool, dist, gpu, iters=iters,
                                              ctas=max(1, 64 // world), seed=rank)
    if grp.is_leader:
        lat.sort()
        q.put({"group": world, "shared_device": shared, "p50_us": lat[len(lat) // 2] if lat else None,
               "p99_us": lat[int(0.99 * (len(lat) - 1))] if lat else None, "max_us": lat[-1] if lat else None,
               "iters": iters, "errors": errs[:2], "not_quiesced": viol})
    dist.barrier()
    dist.destroy_process_group()


def main():
    ctx = mp.get_context("spawn")
    for world in [int(x) for x in (sys.argv[1] if len(sys.argv) > 1 else "1,2,4,8").split(",")]:
        q = ctx.Queue()
        port = _port()
        ps = [ctx.Process(target=worker, args=(r, world, port, 100, q)) for r in range(world)]
        for p in ps:
            p.start()
        print(json.dumps(q.get(timeout=900)), flush=True)
        for p in ps:
            p.join(120)


if __name__ == "__main__":
    main()
