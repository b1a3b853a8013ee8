"""C4 harness (BASELINE configs[3]): a TP online group over per-rank offline pools under one group
gate.  Launch one process per GPU:

  python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 \\
      tools/c4_tp.py --tp 4 [--layers 80] [--horizon 30]

On a box with fewer GPUs than ranks the ranks share devices (gloo plumbing; functional only --
the JSON line says shared_device: true).  Group leaders print one JSON line each."""
import argparse
import json
import os
import sys

os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")  # before any CUDA context (see the package docstring)

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

if __name__ == "__main__":
    import torch
    import torch.distributed as dist

    from paper_2604_07874_b200 import tp as TP
    from paper_2604_07874_b200 import tp_colo as C4

    ap = argparse.ArgumentParser()
    ap.add_argument("--tp", type=int, default=4)
    ap.add_argument("--layers", type=int, default=80)
    ap.add_argument("--horizon", type=float, default=30.0)
    ap.add_argument("--repeats", type=int, default=1)
    ap.add_argument("--handles", type=int, default=64)
    ap.add_argument("--ctx", type=int, default=2048)
    ap.add_argument("--out", default="")
    a = ap.parse_args()
    rank, world = int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1"))
    gpu, shared = TP.rank_device(int(os.environ.get("LOCAL_RANK", "0")),
                                 int(os.environ.get("LOCAL_WORLD_SIZE", str(world))), torch.cuda.device_count())
    torch.cuda.set_device(gpu)
    dist.init_process_group("gloo" if shared else "nccl")
    c = C4.C4Config(tp=a.tp, layers=a.layers, horizon_s=a.horizon, handles=a.handles, ctx=a.ctx)
    r = C4.measure(dist, rank, world, gpu, shared, c, repeats=a.repeats)
    if r is not None:
        line = json.dumps(r)
        print(line, flush=True)
        if a.out:
            with open(a.out.replace(".json", f"_g{rank}.json"), "w") as f:
                f.write(line + "\n")
    dist.barrier()
    dist.destroy_process_group()
