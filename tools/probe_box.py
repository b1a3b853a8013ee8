"""One-off hardware probe: pinned D2H/H2D link peak, device info (writes gpurun_out/probe.txt)."""
import os, subprocess, torch, time
os.makedirs("gpurun_out", exist_ok=True)
out = []
p = lambda *a: out.append(" ".join(str(x) for x in a))
p(subprocess.run(["nvidia-smi"], capture_output=True, text=True).stdout)
p(subprocess.run(["nvidia-smi", "topo", "-m"], capture_output=True, text=True).stdout)
p(subprocess.run(["bash", "-c", "lscpu | head -20; nproc; free -g"], capture_output=True, text=True).stdout)
dev = torch.device("cuda:0")
for mb in (64, 256, 1024):
    n = mb << 20
    d = torch.empty(n, dtype=torch.uint8, device=dev)
    h = torch.empty(n, dtype=torch.uint8, pin_memory=True)
    for name, (dst, src) in {"d2h": (h, d), "h2d": (d, h)}.items():
        best = 1e9
        for _ in range(10):
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s.record(); dst.copy_(src, non_blocking=True); e.record(); torch.cuda.synchronize()
            best = min(best, s.elapsed_time(e))
        p(f"{name} {mb} MiB best {n/best/1e6:.2f} GB/s")
free, total = torch.cuda.mem_get_info()
p("mem free/total GB", free/1e9, total/1e9)
open("gpurun_out/probe.txt", "w").write("\n".join(out))
print("\n".join(out[-8:]))
