"""Host-link bandwidth vs the NUMA node of the pinned buffer (diagnostic for the reclaim copy).

For each NUMA node: pin the thread to that node's CPUs, allocate a pinned host buffer (the
allocation lands on the calling thread's node), time D2H / H2D cudaMemcpy best-of-5."""
import glob
import json
import os
import sys

import torch


def cpulist(s):
    out = set()
    for part in s.strip().split(","):
        if not part:
            continue
        if "-" in part:
            a, b = part.split("-")
            out.update(range(int(a), int(b) + 1))
        else:
            out.add(int(part))
    return out


def main():
    nodes = {}
    for d in sorted(glob.glob("/sys/devices/system/node/node*")):
        nodes[int(d.rsplit("node", 1)[1])] = cpulist(open(os.path.join(d, "cpulist")).read())
    dev = torch.device("cuda", 0)
    bus = torch.cuda.get_device_properties(0).pci_bus_id if hasattr(torch.cuda.get_device_properties(0), "pci_bus_id") else None
    info = {"nodes": {k: sorted(v) for k, v in nodes.items()}, "all_cpus": sorted(os.sched_getaffinity(0))}
    try:
        import pynvml
        pynvml.nvmlInit()
        h = pynvml.nvmlDeviceGetHandleByIndex(0)
        info["pci"] = pynvml.nvmlDeviceGetPciInfo(h).busId.decode() if isinstance(pynvml.nvmlDeviceGetPciInfo(h).busId, bytes) else pynvml.nvmlDeviceGetPciInfo(h).busId
        mask = pynvml.nvmlDeviceGetCpuAffinity(h, 4)
        cpus = [i * 64 + b for i, w in enumerate(mask) for b in range(64) if (w >> b) & 1]
        info["nvml_cpu_affinity"] = cpus
    except Exception as e:  # noqa: BLE001
        info["nvml_error"] = repr(e)
    print(json.dumps(info))
    n = 1 << 30
    src = torch.empty(n, dtype=torch.uint8, device=dev)
    allc = os.sched_getaffinity(0)
    for node, cpus in list(nodes.items()) + [("unbound", allc)]:
        cpus = cpus & allc
        if not cpus:
            continue
        os.sched_setaffinity(0, cpus)
        dst = torch.empty(n, dtype=torch.uint8, pin_memory=True)
        dst.fill_(1)
        res = {}
        for name, fn in (("d2h", lambda: dst.copy_(src, non_blocking=True)),
                         ("h2d", lambda: src.copy_(dst, non_blocking=True))):
            best = 0.0
            for _ in range(5):
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                fn()
                e1.record()
                torch.cuda.synchronize()
                best = max(best, n / (e0.elapsed_time(e1) * 1e-3) / 1e9)
            res[name] = round(best, 2)
        print(json.dumps({"node": node, "cpus": len(cpus), **res}))
        del dst
    os.sched_setaffinity(0, allc)


if __name__ == "__main__":
    sys.exit(main())
