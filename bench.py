#!/usr/bin/env python3
"""Benchmark of the colocation hot path (BASELINE.json metric:
"p99 preempt-to-quiesce us; reclaim GB/s vs link peak; online TTFT/TPOT delta %").

Workload = BASELINE.json configs[1] (C2): Llama-3-8B online + Qwen2-7B offline on one B200,
KV reclaim only.  Geometry: 2 MiB physical slots (one 16-token Llama-3-8B KV
page), 64-page handles (128 MiB), total_handles sized from free HBM after 31.3 GB of the two
models' weights (capped at 1024), a Qwen2-7B offline page = 917,504 B; offline requests of
2000-4000 prompt + 100-200 output tokens (synthetic, deterministic seed), online reserve 10%.

One step = one reclaim op of k handles (k = 36, the C2 probe shape), as Sim::finish_op runs it
(sim.cpp:912-992), on the device:
    gate raise -> quiesce of the running gated offline kernel -> fused snapshot + Algorithm 1 +
    apply_reclaim (multi-CTA instance pass + one CTA) -> start the gather-copy of the invalidated
    pages to pinned host memory -> online_release + offline re-admission of the evicted
    requests.  The K steps are one burst (the online lane stays busy while it needs memory): the
    first op preempts the running offline tenant, the gate is released after the last copy.
Steps are pipelined through the copy ring: op i+1's quiesce and decision run while op i's bytes
cross the link (one copy queued behind the running one); the ring is drained inside the timed
region.
value = reclaimed bytes / device time of the K timed steps (inputs resident in HBM; every step
reads 2.1 GB of distinct pages out of a 128 GiB pool, far above the 126 MB L2).
e2e   = the same ops through the reference-facing API with host buffers: snapshot() to host,
        selective_reclaim(instance) (upload), apply_reclaim(ids), reclaim_copy_start(), as Sim
        calls them, pipelined the same way.
p99 preempt-to-quiesce: >= 1000 preemptions of the gated offline kernel, CUDA events on the gate
stream around (gate store -> wait for every offline CTA to retire).

`--impl reference` times the reference's own CPU implementation of the path (oracle/_ref:
/root/reference/proj/src/{memory,reclaim}.cpp compiled unmodified) plus a host memcpy gather of
the same pages, on this box's host cores.
"""
import argparse
import ctypes as C
import json
import math
import os
import random
import statistics
import subprocess
import sys
import threading
import time

os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")  # before any CUDA context (see the package docstring)

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "p99 preempt-to-quiesce µs; reclaim GB/s vs link peak; online TTFT/TPOT delta %"
SLOT = 2 << 20            # 2 MiB: one 16-token Llama-3-8B KV page (SURVEY §8 geometry)
PAGE = 917_504            # Qwen2-7B 16-token KV page (28 x 2 x 4 x 128 x 2 B x 16)
HSZ = 64                  # pages per handle
TILE = 16384              # offline tile (quiesce granularity), the library default
WEIGHTS = 31.3e9          # Llama-3-8B + Qwen2-7B bf16 weights (not allocated here)


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="valve", choices=["valve", "reference"])
    ap.add_argument("--k", type=int, default=36)
    ap.add_argument("--handles", type=int, default=0)
    ap.add_argument("--preemptions", type=int, default=1000)
    ap.add_argument("--copy-ctas", type=int, default=8,
                    help="copy CTAs: 8 already saturate the link (tools/copy_sweep.py); fewer CTAs keep fewer "
                         "bytes queued on PCIe ahead of the next decision's small host-mapped writes")
    ap.add_argument("--copy-threads", type=int, default=512)
    ap.add_argument("--tma", type=int, default=1, help="1: cp.async.bulk copy through shared memory, 0: LDG/STG")
    ap.add_argument("--seed", type=int, default=2604)
    ap.add_argument("--skip-realtime", action="store_true", help="skip the measured TTFT/TPOT run")
    ap.add_argument("--skip-fanout", action="store_true", help="skip the same-device TP fan-out sweep")
    ap.add_argument("--rt-horizon", type=float, default=60.0, help="C2 online trace length (s)")
    ap.add_argument("--rt-tail", type=float, default=20.0, help="drain time after the horizon (s)")
    ap.add_argument("--rt-repeats", type=int, default=2, help="valve runs (interleaved with standalone)")
    ap.add_argument("--rt-policies", default="valve-fifo,channel+prism",
                    help="extra policies run once each on the same kernels (policies.cpp:5-14)")
    ap.add_argument("--rt-horizon-multi", type=float, default=30.0, help="C5 per-GPU trace length at N > 1 (s)")
    ap.add_argument("--c4-layers", type=int, default=80, help="C4 online model layers (Llama-3-70B: 80)")
    ap.add_argument("--c4-horizon", type=float, default=20.0, help="C4 online trace length (s)")
    ap.add_argument("--rt-decode-ctas", type=int, default=16, help="offline KV decode-pass CTAs (-1 = none)")
    ap.add_argument("--rt-gemm-ctas", type=int, default=64,
                    help="offline Qwen2-7B projection-chain CTAs (0 = all SMs, -1 = no GEMM tenant)")
    ap.add_argument("--profile-mode", action="store_true",
                    help="ncu launch-list runs: no offline kernel (ncu serialises it to completion)")
    return ap.parse_args()


# --------------------------------------------------------------------------- workload

def _hbm_peak():
    """Measured HBM copy bandwidth of this pool's B200s (driver-written MEASURED_PEAKS.json),
    else the profiling recipe's fallback."""
    try:
        v = float(json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"])
        return v, "MEASURED_PEAKS.json hbm_gbs"
    except (OSError, KeyError, ValueError):
        return 6541.5, "B200_PROFILING.md fallback (MEASURED_PEAKS.json absent)"


HBM_PEAK, HBM_PEAK_SOURCE = _hbm_peak()


def workload_config(handles, k, world):
    """The workload both arms run (identical dicts: the driver compares them)."""
    return {"workload": "C2: Llama-3-8B online + Qwen2-7B offline, 1 B200, KV reclaim only "
                        "(BASELINE.json configs[1])",
            "total_handles": handles, "handle_size_pages": HSZ, "slot_bytes": SLOT, "page_bytes": PAGE,
            "k_handles_per_op": k,
            "l2": "inputs larger than L2 (distinct 2.1 GB of a 128 GiB pool per step)",
            "parallelism": f"replicas{world}"}


def offline_requests(seed, n):
    """Qwen2-7B offline stream: prompt 2000-4000, output 100-200 tokens."""
    rng = random.Random(seed)
    out = []
    for r in range(n):
        inp, outp = rng.randint(2000, 4000), rng.randint(100, 200)
        out.append((r, inp, outp, rng.randint(0, outp)))  # id, input, output, generated
    return out


def populate(pool, reqs, page_tokens=16):
    """Admit offline requests until the pool is full (sim.cpp:730-753 admit_offline)."""
    live = {}
    t = 0
    for r, inp, outp, gen in reqs:
        pages = -(-(inp + outp) // page_tokens)
        t += 1
        if not pool.offline_reserve(r, pages, t):
            break
        live[r] = (pages, inp + gen)  # pages, recompute cost = input + generated
    return live, t


# --------------------------------------------------------------------------- clocks

class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu):
        self.gpu, self.rows, self.proc = gpu, [], None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            threading.Thread(target=self._read, daemon=True).start()
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([x.strip() for x in line.split(",")])

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(2)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4)
                          if len(r) > 3 + i and r[3 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(self.rows)}


# --------------------------------------------------------------------------- device arm

def aggregate_ranks(dist, elapsed_ms, total_bytes, device):
    """Whole-job numbers: the slowest rank's device time and the bytes of all ranks (replicas,
    weak scaling).  Works on any backend (nccl on GPUs, gloo in the CPU tests)."""
    import torch

    tt = torch.tensor([elapsed_ms, float(total_bytes)], device=device, dtype=torch.float64)
    mx = tt.clone()
    dist.all_reduce(mx, op=dist.ReduceOp.MAX)
    sm = tt.clone()
    dist.all_reduce(sm, op=dist.ReduceOp.SUM)
    return mx[0].item(), sm[1].item()


def link_peak_d2h(torch, dev):
    n = 256 << 20
    d = torch.empty(n, dtype=torch.uint8, device=dev)
    h = torch.empty(n, dtype=torch.uint8, pin_memory=True)
    best = 1e9
    for _ in range(8):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        h.copy_(d, non_blocking=True)
        e.record()
        torch.cuda.synchronize()
        best = min(best, s.elapsed_time(e))
    return n / (best * 1e-3) / 1e9


def link_peak_h2d(torch, dev):
    n = 256 << 20
    d = torch.empty(n, dtype=torch.uint8, device=dev)
    h = torch.empty(n, dtype=torch.uint8, pin_memory=True)
    best = 1e9
    for _ in range(8):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        d.copy_(h, non_blocking=True)
        e.record()
        torch.cuda.synchronize()
        best = min(best, s.elapsed_time(e))
    return n / (best * 1e-3) / 1e9


def c3_weights(torch, A, gpu, cp, seed, d2h_peak):
    """BASELINE configs[2] (C3) mechanism at real geometry: Qwen2-7B weights as reclaimable
    residents -- 28 layers x 260 whole-slot (2 MiB) pages = 7,280 slots (15.3 GB, ~114 handles) --
    next to offline KV on a 256-handle (32 GiB) pool.  One op evicts 4 layers' handles (their
    co-resident KV goes too): gather to host at each request's own page size, then the layers are
    re-reserved and scattered back (k_restore_scatter).  GB/s against the measured link peaks."""
    H = 256
    pool = A.DevicePool(H, HSZ, 16, device=gpu, slot_bytes=SLOT, page_bytes=PAGE, max_requests=4096,
                        max_pages_per_request=1024)
    pool.online_grow(-(-H // 10), 0)
    layers = {3_000_000 + i: 260 for i in range(28)}
    for w, n in layers.items():
        assert pool.offline_reserve(w, n, 0)
    pool.set_page_bytes({w: SLOT for w in layers})
    live, t = populate(pool, offline_requests(seed, 4 * H))
    pool.set_costs({**{w: 10**12 for w in layers}, **{r: c for r, (p, c) in live.items()}})
    pool.fill_pages()
    out = {"pool_handles": H, "weight_layers": len(layers), "weight_pages": sum(layers.values()),
           "weight_gb": round(sum(layers.values()) * SLOT / 1e9, 2), "ops": []}
    h2d_peak = link_peak_h2d(torch, torch.device("cuda", gpu))
    for op, first in enumerate((0, 8, 16)):
        evict = list(layers)[first:first + 4]
        ids = sorted(set().union(*[set(pool.handles_of_request(w)) for w in evict]))
        t += 10
        res = pool.apply_reclaim(ids, t)
        total, pbs = pool.last_copy_layout()
        host = A.HostBuffer(total)
        st = pool.reclaim_copy(host.ptr, host.nbytes, cp)
        pool.online_release(len(res.handles))
        base, rest_bytes, rest_ms = 0, 0, 0.0
        for r, pb in zip(res.evicted_requests, pbs):
            n = len(res.invalidated_pages[r])
            if r in layers:
                t += 1
                assert pool.offline_reserve(r, layers[r], t)
                pool.set_page_bytes({r: SLOT})
                rs = pool.restore(r, host.ptr + base, res.block_index[r], A.copy_params(ctas=32))
                rest_bytes += rs.bytes
                rest_ms += rs.kernel_ms
            base += n * pb
        weights = sum(len(res.invalidated_pages[w]) for w in evict) * SLOT
        out["ops"].append({"handles": len(res.handles), "evicted_requests": len(res.evicted_requests),
                           "bytes": total, "weight_bytes": weights, "copy_gbs": round(st.bytes / st.kernel_ms / 1e6, 2),
                           "restore_gbs": round(rest_bytes / rest_ms / 1e6, 2) if rest_ms else None})
        del host
    gb = [o["copy_gbs"] for o in out["ops"]]
    rb = [o["restore_gbs"] for o in out["ops"] if o["restore_gbs"]]
    out.update({"copy_gbs": round(statistics.mean(gb), 2), "copy_frac_d2h": round(statistics.mean(gb) / d2h_peak, 4),
                "restore_gbs": round(statistics.mean(rb), 2) if rb else None, "h2d_peak_gbs": round(h2d_peak, 2),
                "restore_frac_h2d": round(statistics.mean(rb) / h2d_peak, 4) if rb else None})
    del pool
    return out


def gemm_tenant(torch, A, gate, dev, stream, gate_stream, preemptions, next_gen):
    """The compute-bound offline tenant: Qwen2-7B gate/up projection (4096 tokens x 37888 x 3584)
    on the gated tcgen05 GEMM -- TFLOP/s polled / unpolled / cuBLAS, and preempt-to-quiesce."""
    m, n, k = 4096, 37888, 3584
    a = torch.randn(m, k, device=dev).to(torch.bfloat16)
    b = (torch.randn(n, k, device=dev) * 0.02).to(torch.bfloat16)
    c = torch.empty(m, n, device=dev, dtype=torch.bfloat16)
    flop = 2.0 * m * n * k

    def timed(fn, reps=10):
        fn()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(reps):
            fn()
        e1.record(stream)
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) / reps

    def run(poll):
        gate.launch_gemm(a.data_ptr(), b.data_ptr(), c.data_ptr(), m, n, k, poll=poll,
                         stream=stream.cuda_stream, fresh=True)

    with torch.cuda.stream(stream):
        t_poll, t_nopoll = timed(lambda: run(True)), timed(lambda: run(False))
        t_cublas = timed(lambda: torch.matmul(a, b.t(), out=c))
    q = []
    total = (m // 256) * (n // 256)  # CTA-pair tiles (the default when m % 256 == 0)
    for i in range(preemptions):
        gate.launch_gemm(a.data_ptr(), b.data_ptr(), c.data_ptr(), m, n, k, stream=stream.cuda_stream, fresh=True)
        time.sleep(0.0001 + 0.0004 * (i % 7) / 7)
        gen = next_gen()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(gate_stream)
        gate.raise_(gen)
        gate.wait_quiesced(gen)
        e1.record(gate_stream)
        gate.release(gen)
        torch.cuda.synchronize()
        if gate.read().tiles_done < total:  # count only launches the raise really preempted
            q.append(e0.elapsed_time(e1) * 1e3)
    q.sort()
    pick = (lambda p: round(q[min(len(q) - 1, int(round(p / 100 * (len(q) - 1))))], 2)) if q else (lambda p: None)
    gate.reset_work()
    return {"shape": [m, n, k], "tflops_polled": round(flop / t_poll / 1e9, 1),
            "tflops_unpolled": round(flop / t_nopoll / 1e9, 1), "tflops_cublas": round(flop / t_cublas / 1e9, 1),
            "polling_overhead_pct": round((t_poll / t_nopoll - 1) * 100, 2),
            "preemptions": len(q), "p50_quiesce_us": pick(50), "p99_quiesce_us": pick(99),
            "max_quiesce_us": q[-1] if q else None}


def tp_fanout_same_device(torch, A, pool, dev, groups=(1, 2, 4, 8), iters=300, seed=0, mode=0, ctas=0):
    """TP-group gate fan-out with every member gate on this one GPU: the leader's
    raise writes all N gate words (stream memory operations), its wait joins N concurrent
    live_ctas waits on helper streams; each member runs its own gated offline kernel on 148/N
    CTAs.  Measures how preempt-to-quiesce scales with the group size for the fan-out mechanism
    itself (the reference's unpatched toggle is linear in GPUs, scenario.hpp:56-58).  Caveat: the
    members share one device, so the NVLink hop of a real TP group is not in these numbers."""
    rng = random.Random(seed)
    out = {}
    for n in groups:
        gates = [A.Gate(dev.index) for _ in range(n)]
        gates[0].set_fanout(mode)
        if n > 1:
            gates[0].attach_peers(gates[1:])
        streams = [torch.cuda.Stream(device=dev) for _ in range(n)]
        gs = torch.cuda.ExternalStream(gates[0].stream, device=dev)
        ctas_m = ctas or max(1, 148 // n)
        lat = []
        for it in range(iters + 20):
            for g, st in zip(gates, streams):
                g.reset_work()  # a fresh pass each time (one pass is far longer than a sample)
                g.launch_offline(pool, None, None, 0, 0, None, ctas=ctas_m, stream=st.cuda_stream)
            deadline = time.perf_counter() + rng.uniform(100e-6, 400e-6)
            while time.perf_counter() < deadline:
                pass
            gen = it + 1
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(gs)
            gates[0].raise_(gen)
            gates[0].wait_quiesced(gen)
            e1.record(gs)
            gates[0].release(gen)
            e1.synchronize()
            if it >= 20:
                lat.append(e0.elapsed_time(e1) * 1e3)
        torch.cuda.synchronize()
        lat.sort()
        out[str(n)] = {"p50_us": round(lat[len(lat) // 2], 2), "p99_us": round(lat[int(0.99 * (len(lat) - 1))], 2),
                       "max_us": round(lat[-1], 2), "preemptions": len(lat), "ctas_per_member": ctas_m}
        del gates
    return {"note": "one leader + N-1 member gates on one B200 (no NVLink hop); offline decode pass "
                    "per member on 148/N CTAs; leader raise -> all members quiesced",
            "ack_wait": ["batched memops on the waiting stream", "helper stream per member"][mode], "groups": out}


def tp_fanout_across_ranks(torch, A, pool, dist, rank, world, gpu, groups=(2, 4, 8), iters=200, seed=0):
    """TP-group gate fan-out with one process per GPU (SURVEY §8e, configs[3]): for each group
    size tp dividing the world, consecutive ranks form groups, every member's gate words live in
    its own HBM, the leader opens them over CUDA IPC and raises / waits over NVLink peer memory
    (paper_2604_07874_b200.tp).  Every member runs its gated decode pass on all its SMs.
    Returns group size -> the leaders' p50 / p99 preempt-to-quiesce (max over the groups)."""
    from paper_2604_07874_b200 import tp as TP

    out = {}
    for tp in groups:
        if tp > world or world % tp:
            continue
        gate = A.Gate(gpu)
        grp = TP.TPGate(gate, rank, world, tp, dist, opener=TP.open_member(gpu))
        lat, errs, viol = TP.measure_group_fanout(torch, gate, grp, pool, dist, gpu, iters=iters, seed=seed + rank)
        if grp.error:
            errs = [grp.error] + errs
        lat.sort()
        mine = {"lat": [lat[len(lat) // 2], lat[int(0.99 * (len(lat) - 1))], lat[-1]] if lat else None,
                "errors": errs[:2], "not_quiesced": viol}
        allr = [None] * world
        dist.all_gather_object(allr, mine)
        lats = [x["lat"] for x in allr if x["lat"]]
        out[str(tp)] = {"p50_us": round(max(x[0] for x in lats), 2) if lats else None,
                        "p99_us": round(max(x[1] for x in lats), 2) if lats else None,
                        "max_us": round(max(x[2] for x in lats), 2) if lats else None,
                        "preemptions_per_group": iters, "groups": world // tp,
                        "members_not_quiesced": sum(x["not_quiesced"] for x in allr),
                        "errors": [e for x in allr for e in x["errors"]][:4]}
        del grp, gate
        dist.barrier()
    return {"note": "one process per GPU; leader raise -> every member's CTAs retired, over NVLink peer "
                    "memory (max over the TP groups of the job)", "groups": out}


def c5_instances(torch, dist, gpu, rank, world, args):
    """C5 (configs[4]): every GPU runs its own colocation instance on its own online trace (the
    C2 spike shape, seed per rank) -- the north star's independent per-GPU instances, no collective.
    One A B A pair per rank (shorter than the N=1 leg); all ranks' deltas are reported."""
    from paper_2604_07874_b200 import realtime as RT

    rcfg = RT.RtConfig(decode_ctas=args.rt_decode_ctas, gemm_ctas=args.rt_gemm_ctas)
    try:
        r = RT.measure(horizon=args.rt_horizon_multi, tail_s=10.0, device=gpu, seed=args.seed + 101 * rank,
                       repeats=1, cfg=rcfg, policies=(), handles=args.handles or 0)
        v = r["valve"]
        mine = {"rank": rank, "gpu": gpu, "online_requests": r["trace"]["online_requests"],
                "ttft_delta_pct": v["ttft_delta_pct"], "tpot_delta_pct": v["tpot_delta_pct"],
                "aa_noise_ttft_pct": r["aa_noise_ttft_pct"], "reclaims": v["reclaims"],
                "offline_tokens_per_s": v["offline_tokens_per_s"], "quiesce_wait_us": v["quiesce_wait_us"]}
    except Exception as e:  # noqa: BLE001 -- every rank must still reach the gather
        mine = {"rank": rank, "gpu": gpu, "error": repr(e)[:300], "ttft_delta_pct": None, "tpot_delta_pct": None,
                "offline_tokens_per_s": 0.0}
    allr = [None] * world
    dist.all_gather_object(allr, mine)
    return {"config": "C5: %d independent colocation instances (one per GPU), C2 spike trace per instance "
                      "(seed per rank), %.0f s horizon" % (world, args.rt_horizon_multi),
            "ranks": allr,
            "ttft_delta_pct_max": max((x["ttft_delta_pct"] for x in allr if x["ttft_delta_pct"] is not None), default=None),
            "tpot_delta_pct_max": max((x["tpot_delta_pct"] for x in allr if x["tpot_delta_pct"] is not None), default=None),
            "offline_tokens_per_s_total": sum(x["offline_tokens_per_s"] for x in allr)}


def c4_job(world, args):
    """C4 (configs[3]): Llama-3-70B TP = 4 (2 for N = 2, 6) online groups over per-rank offline
    pools, one group gate per TP group broadcast over NVLink peer memory
    (paper_2604_07874_b200.tp_colo via tools/c4_tp.py).  Launched by rank 0 as its own torchrun
    job on the same GPUs once the bench's ranks have released their memory, under a timeout, so a
    stuck collective there cannot take the bench's JSON line with it."""
    import glob
    import socket
    import subprocess

    tp = 4 if world % 4 == 0 else 2
    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        port = so.getsockname()[1]
    out = os.path.join(ROOT, "gpurun_out", "c4", "c4.json")
    os.makedirs(os.path.dirname(out), exist_ok=True)
    for f in glob.glob(os.path.join(os.path.dirname(out), "c4_g*.json")):
        os.remove(f)
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={world}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.join(ROOT, "tools", "c4_tp.py"),
           "--tp", str(tp), "--layers", str(args.c4_layers), "--horizon", str(args.c4_horizon), "--out", out]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=1200, cwd=ROOT)
    groups = [json.load(open(f)) for f in sorted(glob.glob(os.path.join(os.path.dirname(out), "c4_g*.json")))]
    if r.returncode != 0 and not groups:
        raise RuntimeError(f"c4 job rc={r.returncode}: {r.stderr[-300:]}")
    return {"tp": tp, "groups": groups}


VALVE_OPS = os.path.join(ROOT, "tools", "_bin", "valve_ops")


def e2e_cpp(torch, dist, gpu, H, args, world):
    """`e2e` through the reference's C++ runtime API: tools/_bin/valve_ops (tools/cpp/
    colosim_ops.cpp compiled against include/colosim, linked to libvalve.so) runs the same burst
    of reclaim ops as the device leg -- gate raise + quiesce, MemoryPool::snapshot(),
    selective_reclaim(), MemoryPool::apply_reclaim(), the gather copy into pinned host memory,
    re-admission -- one copy queued behind the running one.  Whole job: bytes of all ranks over
    the slowest rank's seconds."""
    import subprocess

    env = dict(os.environ, VALVE_DEVICE=str(gpu))
    d, err = None, None
    try:
        r = subprocess.run([VALVE_OPS, "e2e", str(H), str(args.k), str(max(1, args.steps)), str(max(1, args.warmup)),
                            "0" if args.profile_mode else "1"], capture_output=True, text=True, timeout=600, env=env)
        if r.returncode != 0:
            raise RuntimeError(f"valve_ops e2e rc={r.returncode}: {r.stderr[-300:]}")
        d = json.loads(r.stdout.strip().splitlines()[-1])
    except Exception as e:  # noqa: BLE001 -- every rank must still reach the gather below
        err = repr(e)[:300]
    if world > 1:  # always gathered, so a failing rank cannot leave the others in a collective
        allr = [None] * world
        dist.all_gather_object(allr, (d["seconds"], d["bytes"]) if d else None)
        if any(x is None for x in allr):
            raise RuntimeError(err or "valve_ops e2e failed on another rank")
        secs, nbytes = max(x[0] for x in allr), sum(x[1] for x in allr)
    else:
        if d is None:
            raise RuntimeError(err)
        secs, nbytes = d["seconds"], d["bytes"]
    return {"value": round(nbytes / secs / 1e9, 3), "unit": "GB/s",
            "h2d_bytes_per_step": d["h2d_bytes_per_step"], "d2h_bytes_per_step": d["d2h_bytes_per_step"],
            "path": "C++: colosim::MemoryPool::snapshot() -> colosim::selective_reclaim() -> "
                    "MemoryPool::apply_reclaim() -> valve_pool_reclaim_copy_start(), pinned host buffers "
                    "(tools/_bin/valve_ops, include/colosim drop-in over libvalve.so)",
            "breakdown_ms_per_step": d["breakdown_ms_per_step"],
            "pipelining": "one reclaim copy queued behind the running one (op i+1 decides while op i copies); "
                          "the burst's first op preempts the offline tenant, which stays gated for the burst"}


def _progress(rank, what):
    """Phase marks on stderr (multi-rank runs: where a rank is when something stalls)."""
    print(f"bench[{rank}] {time.strftime('%H:%M:%S')} {what}", file=sys.stderr, flush=True)


def _guarded(name, fn):
    """Secondary measurements after the timed region: a failure is recorded in the JSON line
    instead of losing the line (the headline numbers are already measured)."""
    try:
        return fn()
    except Exception as e:  # noqa: BLE001
        print(f"bench: {name} failed: {e!r}", file=sys.stderr, flush=True)
        return {"error": repr(e)[:300]}


def _finite(o):
    """NaN / inf (e.g. an empty sample's percentile) -> null: the line stays strict JSON."""
    if isinstance(o, float):
        return o if math.isfinite(o) else None
    if isinstance(o, dict):
        return {k: _finite(v) for k, v in o.items()}
    if isinstance(o, (list, tuple)):
        return [_finite(v) for v in o]
    return o


def run_valve(args, rank, world, dist):
    import torch

    from paper_2604_07874_b200 import api as A

    dev = torch.device("cuda", torch.cuda.current_device())
    gpu = dev.index
    _progress(rank, f"start on cuda:{gpu}")
    free, _ = torch.cuda.mem_get_info(dev)
    free = free / getattr(args, "ranks_per_device", 1)
    H = args.handles or min(1024, int((free - WEIGHTS - 6e9) // (SLOT * HSZ)))
    pool = A.DevicePool(H, HSZ, 16, device=gpu, slot_bytes=SLOT, page_bytes=PAGE,
                        max_requests=4096, max_pages_per_request=1024)
    pool.online_grow(-(-H // 10), 0)  # initial reserve ceil(0.1 * total) (sim.cpp:207-210)
    reqs = offline_requests(args.seed + rank, 4 * H)
    live, t = populate(pool, reqs)
    next_req = len(live)
    pool.set_costs({r: c for r, (p, c) in live.items()})
    pool.fill_pages()
    gate = A.Gate(gpu)
    off_stream = torch.cuda.Stream(device=dev)
    gate_stream = torch.cuda.ExternalStream(gate.stream, device=dev)
    pool_stream = torch.cuda.ExternalStream(pool.view().stream, device=dev)
    cap_pages = args.k * HSZ
    hosts = [A.HostBuffer(cap_pages * PAGE), A.HostBuffer(cap_pages * PAGE)]  # two copies in flight
    host = hosts[0]
    cp = A.copy_params(ctas=args.copy_ctas, threads=args.copy_threads, use_tma=args.tma)
    peak = link_peak_d2h(torch, dev)
    gen = [0]
    rng = random.Random(args.seed)
    stats = {"quiesce_us": [], "copy_ms": [], "bytes": [], "reclaim_ms": [], "pages": []}

    def ev():
        return torch.cuda.Event(enable_timing=True)

    def restore(evicted, n_release=None):
        nonlocal next_req, t
        pool.online_release(n_release or args.k)
        costs = {}
        for r in evicted:  # re-admission of the evicted requests (resume recompute)
            pages, cost = live.pop(r)
            t += 1
            if pool.offline_reserve(r, pages, t):
                live[r] = (pages, cost)
                costs[r] = cost
        while True:  # top the pool back up with fresh requests
            _, inp, outp, g = reqs[next_req % len(reqs)]
            rid = 1_000_000 + next_req
            pages = -(-(inp + outp) // 16)
            t += 1
            if not pool.offline_reserve(rid, pages, t):
                break
            next_req += 1
            live[rid] = (pages, inp + g)
            costs[rid] = inp + g
        if costs:
            pool.set_costs(costs)

    def tiles_left_low():
        total = sum(p for p, _ in live.values()) * (-(-PAGE // TILE))
        return gate.read().tiles_claimed >= 0.8 * total

    pending = []  # copies in flight (FIFO): (record, pages)
    step_events = []

    def drain(keep):
        """Complete copies until at most `keep` are in flight; returns their bytes."""
        done = 0
        while len(pending) > keep:
            rec, npg_ = pending.pop(0)
            cs = pool.reclaim_copy_wait()
            done += cs.bytes
            if rec:
                stats["copy_ms"].append(cs.kernel_ms)
                stats["bytes"].append(cs.bytes)
                stats["pages"].append(npg_)
        return done

    def step(record, preempt):
        """One reclaim op: raise -> quiesce -> fused select/apply -> start the gather copy ->
        re-admit.  Ops come in bursts (the online lane is busy while it needs memory,
        sim.cpp:362-369): the burst's first op preempts the running offline tenant, and the gate
        stays closed until the burst's last copy has landed -- a decode pass running beside a
        copy costs it ~9 % of the link (shared L2/HBM path; tools/copy_under_load.py).  The copy
        works from its own snapshot of the report, so op i+1's decision overlaps op i's bytes on
        the link: one copy stays queued behind the running one and the link never idles."""
        nonlocal t
        if preempt:
            if tiles_left_low():  # offline work list exhausted: start a new pass
                gate.reset_work()
            if not args.profile_mode:
                gate.launch_offline(pool, None, None, 0, 0, None, stream=off_stream.cuda_stream)
        gen[0] += 1
        e0, e1, e2, e3 = ev(), ev(), ev(), ev()
        e0.record(gate_stream)
        gate.raise_(gen[0])
        gate.wait_quiesced(gen[0])
        e1.record(gate_stream)
        pool_stream.wait_event(e1)
        e2.record(pool_stream)
        t += 10
        nh, ne, npg = pool.reclaim(args.k, t, 0)
        e3.record(pool_stream)
        res = pool.last_reclaim()
        pool.reclaim_copy_start(hosts[step.n % 2].ptr, hosts[0].nbytes, cp)
        step.n += 1
        pending.append((record, npg))
        restore(res.evicted_requests)
        done = drain(1)
        if record:  # read after the timed region: a sync here would drain the copy pipeline
            step_events.append((e0, e1, e2, e3))
        return done
    step.n = 0

    for i in range(args.warmup):
        step(False, i == 0)
    drain(0)
    gate.release(gen[0])
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    launches0 = A.kernel_launches()
    with ClockSampler(gpu) as clocks:
        torch.cuda.synchronize()
        t0, t1 = ev(), ev()
        t0.record(pool_stream)
        total_bytes = 0
        for i in range(args.steps):
            total_bytes += step(True, i == 0)
        total_bytes += drain(0)
        t1.record(pool_stream)
        torch.cuda.synchronize()
    gate.release(gen[0])  # end of the burst
    for e0, e1, e2, e3 in step_events:
        stats["quiesce_us"].append(e0.elapsed_time(e1) * 1e3)
        stats["reclaim_ms"].append(e2.elapsed_time(e3))
    launches = A.kernel_launches() - launches0
    elapsed_ms = t0.elapsed_time(t1)
    if dist:
        elapsed_ms, total_bytes = aggregate_ranks(dist, elapsed_ms, total_bytes, dev)

    _progress(rank, "timed burst done; preemption latency")
    # ------------------------------------------------ p50/p99 preempt-to-quiesce
    q = []
    gate.reset_work()
    for i in range(0 if args.profile_mode else args.preemptions):
        gate.launch_offline(pool, None, None, 0, 0, None, stream=off_stream.cuda_stream)
        deadline = time.perf_counter() + rng.uniform(50e-6, 400e-6)
        while time.perf_counter() < deadline:
            pass
        gen[0] += 1
        e0, e1 = ev(), ev()
        e0.record(gate_stream)
        gate.raise_(gen[0])
        gate.wait_quiesced(gen[0])
        e1.record(gate_stream)
        gate.release(gen[0])
        e1.synchronize()
        q.append(e0.elapsed_time(e1) * 1e3)
        if tiles_left_low():
            gate.reset_work()
    torch.cuda.synchronize()
    q.sort()
    q = q or [float("nan")]
    pct = lambda p: q[min(len(q) - 1, int(round(p / 100 * (len(q) - 1))))]

    _progress(rank, "polling overhead")
    # ------------------------------------------------ polling overhead (offline throughput)
    def offline_rate(poll):
        gate.reset_work()
        s, e = ev(), ev()
        s.record(off_stream)
        gate.launch_offline(pool, None, None, 0, 0, None, poll=poll, stream=off_stream.cuda_stream)
        e.record(off_stream)
        torch.cuda.synchronize()
        tiles = gate.read().tiles_done
        return tiles * TILE / (s.elapsed_time(e) * 1e-3) / 1e9, tiles, s.elapsed_time(e)
    polled = unpolled = (float("nan"),)
    if not args.profile_mode:
        rates = {True: [], False: []}
        for poll in (True, False, True, False, True, False):
            rates[poll].append(offline_rate(poll))
        polled = max(rates[True])
        unpolled = max(rates[False])

    _progress(rank, "TP fan-out")
    # ------------------------------------------------ TP-group gate fan-out, one device
    fanout = None
    if not args.profile_mode and not args.skip_fanout and world == 1:
        fanout = tp_fanout_same_device(torch, A, pool, dev, seed=args.seed)
        fanout["alt_helper_streams"] = tp_fanout_same_device(torch, A, pool, dev, groups=(2, 4, 8), iters=200,
                                                             seed=args.seed, mode=1)["groups"]
    elif not args.profile_mode and not args.skip_fanout and world > 1:
        fanout = _guarded("tp_fanout", lambda: tp_fanout_across_ranks(torch, A, pool, dist, rank, world, gpu,
                                                                      seed=args.seed))

    _progress(rank, "GEMM tenant")
    # ------------------------------------------------ GEMM tenant (tcgen05)
    def next_gen():
        gen[0] += 1
        return gen[0]
    gemm = gemm_tenant(torch, A, gate, dev, off_stream, gate_stream, 0 if args.profile_mode else 200, next_gen)

    # ------------------------------------------------ copy-engine alternative (same report)
    pool.reclaim(args.k, t + 5, 0)
    ce_res = pool.last_reclaim()
    flat = [p for r in ce_res.evicted_requests for p in ce_res.physical_pages[r]]
    ce_runs = sum(1 for i, p in enumerate(flat) if i == 0 or p != flat[i - 1] + 1)  # 2D transfers
    ce = pool.reclaim_copy(host.ptr, host.nbytes, engine="ce")
    ce_gbs = ce.bytes / (ce.kernel_ms * 1e-3) / 1e9
    # the same report again through the SM kernel under a rate bound (token bucket, 1 MiB burst):
    # bytes / (first chunk issued -> last store retired) must sit at the configured rate
    rate = 25e9
    rb = pool.reclaim_copy(host.ptr, host.nbytes, A.copy_params(ctas=args.copy_ctas, threads=args.copy_threads,
                                                                rate_bytes_per_s=rate, burst_bytes=1 << 20))
    rate_gbs = rb.bytes / ((rb.t_last_ns - rb.t_first_ns) * 1e-9) / 1e9 if rb.t_last_ns > rb.t_first_ns else None
    restore(pool.last_reclaim().evicted_requests)

    # ------------------------------------------------ eviction-policy contrast on the device
    # (SURVEY §8f.4): Algorithm 1 vs FIFO (the uvm/static baseline, reclaim.cpp:69-83) on the
    # same C2 snapshots, both selected by the device kernels; cost = recompute tokens evicted
    # (reclaim.cpp:19-31 evicted_cost, also on the device)
    contrast = {}
    for kk in sorted({8, args.k}):
        sel_c = fifo_c = 0
        for _ in range(4):
            inst = pool.snapshot()
            inst.cost = {r: live[r][1] for h in inst.handles for r in h.requests}
            sel_c += A.evicted_cost(inst, A.selective_reclaim(inst, kk, device=gpu), device=gpu)
            fifo_c += A.evicted_cost(inst, A.fifo_reclaim(inst, kk, device=gpu), device=gpu)
            t += 10
            nh, _, _ = pool.reclaim(kk, t, 0)  # churn the pool between samples
            restore(pool.last_reclaim().evicted_requests, nh)
        contrast[f"k{kk}"] = {"selective_tokens": sel_c, "fifo_tokens": fifo_c,
                              "reduction_pct": round((1 - sel_c / fifo_c) * 100, 2) if fifo_c else None}

    _progress(rank, "e2e")
    # ------------------------------------------------ e2e through the reference-facing API
    # one copy stays in flight behind the running one (as in step()): op i+1's quiesce, snapshot,
    # selection and apply run on the host/pool stream while op i's bytes cross the link
    e2e_bytes = e2e_h2d = e2e_d2h = 0
    brk = {"quiesce": 0.0, "snapshot": 0.0, "select": 0.0, "apply": 0.0, "restore": 0.0, "copy_wait": 0.0}
    n_e2e = max(1, args.steps)
    torch.cuda.synchronize()
    w0 = time.perf_counter()
    for it in range(n_e2e + 1):  # iteration 0 is an untimed warm-up
        if it == 1:  # end of the warm-up burst; the timed burst starts with a preemption
            e2e_bytes += drain(0)
            gate.release(gen[0])
            torch.cuda.synchronize()
            w0 = time.perf_counter()
            e2e_bytes = e2e_h2d = e2e_d2h = 0
            brk = {key: 0.0 for key in brk}
        gen[0] += 1
        p0 = time.perf_counter()
        if it <= 1 and not args.profile_mode:  # each burst's first op preempts the running tenant
            gate.launch_offline(pool, None, None, 0, 0, None, stream=off_stream.cuda_stream)
        gate.raise_(gen[0])
        gate.wait_quiesced(gen[0])
        torch.cuda.current_stream().wait_stream(gate_stream)
        torch.cuda.current_stream().synchronize()
        p1 = time.perf_counter()
        inst = pool.snapshot()                                   # D2H instance
        inst.cost = {r: live[r][1] for h in inst.handles for r in h.requests}
        nnz = sum(len(h.requests) for h in inst.handles)
        p2 = time.perf_counter()
        ids = A.selective_reclaim(inst, args.k, device=gpu)      # H2D instance, D2H ids
        t += 10
        p3 = time.perf_counter()
        res = pool.apply_reclaim(ids, t)                         # H2D ids, D2H result
        npg = sum(len(v) for v in res.invalidated_pages.values())
        pool.reclaim_copy_start(hosts[it % 2].ptr, hosts[0].nbytes, cp)  # D2H page bytes
        pending.append((False, npg))
        p4 = time.perf_counter()
        restore(res.evicted_requests)
        p5 = time.perf_counter()
        e2e_bytes += drain(1)
        p6 = time.perf_counter()
        for key, a, b in (("quiesce", p0, p1), ("snapshot", p1, p2), ("select", p2, p3),
                          ("apply", p3, p4), ("restore", p4, p5), ("copy_wait", p5, p6)):
            brk[key] += (b - a) * 1e3
        n = len(inst.handles)
        m = len(inst.cost)
        e2e_d2h += n * 16 + 4 + nnz * 8 + 4 * len(ids) + len(res.evicted_requests) * 12 + npg * 16
        e2e_d2h += npg * PAGE  # the page bytes this op copies
        e2e_h2d += n * 16 + 4 + nnz * 8 + m * 16 + 4 * len(ids)
    e2e_bytes += drain(0)
    torch.cuda.synchronize()
    e2e_s = time.perf_counter() - w0
    gate.release(gen[0])  # end of the burst

    copy_gbs = statistics.mean(b / (ms * 1e-3) / 1e9 for b, ms in zip(stats["bytes"], stats["copy_ms"]))

    _progress(rank, "C3 + C++ e2e")
    # ------------------------------------------------ C3: weight pages (configs[2] mechanism)
    import gc

    del pool, host, hosts
    gc.collect()
    torch.cuda.synchronize()
    torch.cuda.empty_cache()
    c3 = _guarded("c3_weight_pages", lambda: c3_weights(torch, A, gpu, cp, args.seed + rank, peak))
    cpp_e2e = _guarded("e2e_cpp", lambda: e2e_cpp(torch, dist, gpu, H, args, world))

    _progress(rank, "real-time / C5 / C4")
    # ------------------------------------------------ measured online TTFT/TPOT deltas
    # (real-time loop: random-init Llama-3-8B online in PyTorch + the gated offline tenant on a
    # 32 GiB pool; the 128 GiB reclaim pool is released first)
    rt = {"note": "skipped (--skip-realtime)"}

    if world > 1 and not args.skip_realtime and not args.profile_mode:
        del gate
        gc.collect()
        torch.cuda.synchronize()
        torch.cuda.empty_cache()
        rt = _guarded("online_realtime_c5", lambda: c5_instances(torch, dist, gpu, rank, world, args))
        gc.collect()
        torch.cuda.synchronize()
        torch.cuda.empty_cache()
        # C4 runs after this function, as its own torchrun job (main(): a hang there is contained)
    elif not args.skip_realtime and not args.profile_mode:
        del gate
        gc.collect()
        torch.cuda.synchronize()
        torch.cuda.empty_cache()
        from paper_2604_07874_b200 import realtime as RT

        # BASELINE C2 trace + C3's MIAD resizing and rate-bounded copies (realtime.measure)
        rcfg = RT.RtConfig(decode_ctas=args.rt_decode_ctas, gemm_ctas=args.rt_gemm_ctas)
        rt = _guarded("online_realtime", lambda: RT.measure(
            horizon=args.rt_horizon, tail_s=args.rt_tail, device=gpu, seed=args.seed + rank,
            repeats=args.rt_repeats, cfg=rcfg,
            policies=tuple(p for p in args.rt_policies.split(",") if p),
            log_dir=os.path.join(ROOT, "gpurun_out", "realtime_logs")))
    try:
        traffic = json.load(open(os.path.join(ROOT, "profiles", "r2_copy_traffic.json")))
    except OSError:
        traffic = {}
    value = total_bytes / (elapsed_ms * 1e-3) / 1e9
    out = {
        "metric": METRIC,
        "value": round(value, 3),
        "unit": "GB/s",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": round(elapsed_ms / args.steps, 3),
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "u8",
        "data": "synthetic",
        "config": workload_config(H, args.k, world),
        "run": {"live_offline_requests": len(live), "pages_per_op_mean": statistics.mean(stats["pages"]),
                "copy_ctas": args.copy_ctas, "copy_threads": args.copy_threads, "copy_tma": args.tma},
        "p50_preempt_to_quiesce_us": round(pct(50), 2),
        "p99_preempt_to_quiesce_us": round(pct(99), 2),
        "max_preempt_to_quiesce_us": round(q[-1], 2),
        "preemptions": len(q),
        "reference_modeled_quiesce_us": 1000,
        "link_peak_d2h_gbs": round(peak, 2),
        "reclaim_copy_gbs": round(copy_gbs, 2),
        "reclaim_frac_of_link_peak": round(copy_gbs / peak, 4),
        "decision_us_mean": round(statistics.mean(stats["reclaim_ms"]) * 1e3, 1),
        "copy_engine_alt_gbs": round(ce_gbs, 2),
        "copy_engine_alt_frac": round(ce_gbs / peak, 4),
        "copy_engine_alt_transfers": ce_runs,
        "rate_bound": {"set_gbs": rate / 1e9, "achieved_gbs": round(rate_gbs, 2) if rate_gbs else None,
                       "bytes": rb.bytes, "burst_bytes": 1 << 20},
        "copy_note": "SM-issued sysmem stores leave as 128 B PCIe TLPs vs 256 B for the copy engines: "
                     "the SM kernel's ceiling is (128/152)/(256/280) = 92.1% of the CE-measured peak",
        "burst_first_quiesce_us": round(stats["quiesce_us"][0], 1),
        "offline_polling_overhead_pct": round((1 - polled[0] / unpolled[0]) * 100, 2),
        "offline_gbs": {"polled": round(polled[0], 1), "unpolled": round(unpolled[0], 1)},
        "offline_gemm": gemm,
        "tp_fanout_same_device": fanout,
        "policy_contrast_recompute": contrast,
        "c3_weight_pages": c3,
        "ttft_delta_pct": (rt.get("valve") or {}).get("ttft_delta_pct", rt.get("ttft_delta_pct_max")),
        "tpot_delta_pct": (rt.get("valve") or {}).get("tpot_delta_pct", rt.get("tpot_delta_pct_max")),
        "aa_noise_ttft_pct": rt.get("aa_noise_ttft_pct"),
        "aa_noise_tpot_pct": rt.get("aa_noise_tpot_pct"),
        "shortfall_to_first_online_write_us": (rt.get("valve") or {}).get("shortfall_to_first_write_us"),
        "online_realtime": rt,
        "c4_tp_group": {"note": "runs at N >= 2 (one process per GPU)"},
        "roofline": {
            "bound": "pcie_d2h",
            "achieved": round(copy_gbs, 2),
            "peak": round(peak, 2),
            "unit": "GB/s",
            "frac": round(copy_gbs / peak, 4),
            "traffic": traffic.get("traffic_bytes_per_launch"),
            "traffic_source": traffic.get("source"),
            "peak_source": "pinned cudaMemcpy D2H measured in this run (the copy's true roofline; "
                           "HBM is ~110x faster)",
            "kernel": "k_reclaim_copy_tma" if args.tma else "k_reclaim_copy",
            "algorithmic_bytes_per_launch": round(statistics.mean(stats["bytes"])),
            "hbm": {"achieved": round(copy_gbs, 2), "peak": HBM_PEAK, "unit": "GB/s",
                    "frac": round(copy_gbs / HBM_PEAK, 5), "peak_source": HBM_PEAK_SOURCE},
        },
        "e2e": cpp_e2e if cpp_e2e and "value" in cpp_e2e else {
            "value": round(e2e_bytes / e2e_s / 1e9, 3),
            "unit": "GB/s",
            "h2d_bytes_per_step": int(e2e_h2d / n_e2e),
            "d2h_bytes_per_step": int(e2e_d2h / n_e2e),
            "path": "python ctypes mirror (C++ driver unavailable: %s)" % (cpp_e2e or {}).get("error", "?"),
        },
        "e2e_python_api": {
            "value": round(e2e_bytes / e2e_s / 1e9, 3),
            "unit": "GB/s",
            "path": "paper_2604_07874_b200.api (ctypes): snapshot() -> selective_reclaim(instance) -> "
                    "apply_reclaim(ids) -> reclaim_copy_start(), host buffers",
            "breakdown_ms_per_step": {k: round(v / n_e2e, 3) for k, v in brk.items()},
        },
        "gpu_launches": int(launches),
        "clocks": clocks.summary(),
    }
    return out


# --------------------------------------------------------------------------- CPU arms

def cpu_reference(args, n_ops, threads, kind_note=""):
    """The reference decision path (oracle/_ref, C++-timed) + host memcpy gather."""
    import numpy as np

    import oracle
    from paper_2604_07874_b200 import api as A

    b = oracle.ref_backend() if oracle.ref_available() else oracle.c_backend()
    kind = "reference" if oracle.ref_available() else "port"
    H = args.handles or 1024
    pool = A.MemoryPool(H, HSZ, 16, backend=b)
    pool.online_grow(-(-H // 10), 0)
    reqs = offline_requests(args.seed, 4 * H)
    live, t = populate(pool, reqs)
    mirror_slots = 4096  # 3.5 GiB host mirror; page ids map onto it modulo its size
    mirror = np.empty(mirror_slots * PAGE, dtype=np.uint8)
    mirror[::4096] = 1
    dst = np.empty(args.k * HSZ * PAGE, dtype=np.uint8)
    dst[::4096] = 1
    f = getattr(b.lib, "vr_time_reclaim", None)
    us_tot = gather_s = 0.0
    nbytes = 0
    next_req = len(live)
    for _ in range(n_ops):
        inst = pool.snapshot()
        keys = sorted({r for h in inst.handles for r in h.requests})
        ck = (C.c_int64 * len(keys))(*keys)
        cv = (C.c_int64 * len(keys))(*[live[r][1] for r in keys])
        cap = args.k * HSZ
        pages = (C.c_int64 * cap)()
        npg = C.c_int(0)
        us = (C.c_double * 3)()
        t += 10
        if f is not None:
            f.restype = C.c_int
            f.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int, C.c_int, C.c_int64,
                          C.c_void_p, C.c_void_p, C.c_int, C.c_void_p]
            b.check(f(pool.handle, ck, cv, len(keys), args.k, t, us, pages, cap, C.byref(npg)))
            ev = None
            us_tot += us[0] + us[1] + us[2]
        else:  # port: time through the API (includes ctypes marshalling)
            w0 = time.perf_counter()
            inst.cost = {r: live[r][1] for r in keys}
            ids = A.selective_reclaim(inst, args.k, backend=b)
            res = pool.apply_reclaim(ids, t)
            us_tot += (time.perf_counter() - w0) * 1e6
            pl = [p for r in res.evicted_requests for p in res.invalidated_pages[r]]
            npg.value = len(pl)
            for i, p in enumerate(pl[:cap]):
                pages[i] = p
        n = min(npg.value, cap)
        phys = (C.c_int * max(n, 1))(*[pages[i] % mirror_slots for i in range(n)])
        w0 = time.perf_counter()
        oracle.c_backend().lib.vo_gather_memcpy(mirror.ctypes.data, PAGE, PAGE, phys, n,
                                                dst.ctypes.data, threads)
        gather_s += time.perf_counter() - w0
        nbytes += n * PAGE
        # restore the pool shape (untimed)
        ev = res_evicted(pool, inst, pages, n)
        pool.online_release(args.k)
        for r in ev:
            pg, cost = live.pop(r)
            t += 1
            if pool.offline_reserve(r, pg, t):
                live[r] = (pg, cost)
        while True:
            _, inp, outp, g = reqs[next_req % len(reqs)]
            rid = 1_000_000 + next_req
            pg = -(-(inp + outp) // 16)
            t += 1
            if not pool.offline_reserve(rid, pg, t):
                break
            next_req += 1
            live[rid] = (pg, inp + g)
    secs = us_tot * 1e-6 + gather_s
    return {"value": nbytes / secs / 1e9, "decision_us_per_op": us_tot / n_ops,
            "gather_gbs": nbytes / gather_s / 1e9, "kind": kind, "bytes": nbytes, "secs": secs}


def res_evicted(pool, inst_before, pages, n):
    """Requests that left the pool in the last op (residents of the reclaimed handles)."""
    S = HSZ
    handles = {int(pages[i]) // S for i in range(n)}
    out = set()
    for h in inst_before.handles:
        if h.id in handles:
            out.update(h.requests)
    return sorted(out)


def cpu_baseline_block(args):
    threads = os.cpu_count() or 1
    r = cpu_reference(args, 3, threads)
    return {"value": round(r["value"], 3), "unit": "GB/s", "cores": threads, "kind": r["kind"],
            "sample": f"3 reclaim ops (k={args.k}, {args.handles or 1024} handles, C2 shape): reference "
                      f"snapshot+selective_reclaim+apply_reclaim (1 core, C++-timed; "
                      f"{r['decision_us_per_op']:.0f} us/op) + host memcpy gather of the same pages "
                      f"({threads} threads, {r['gather_gbs']:.1f} GB/s) from a 3.5 GiB host mirror",
            "decision_us_per_op": round(r["decision_us_per_op"], 1),
            "bookkeeping_vs_device": _guarded("bookkeeping", bookkeeping_table)}


def bookkeeping_table(handles=(128, 1024), ks="1,4,15,36,64"):
    """Per-op latency through the reference's C++ API on both sides of the link-swap
    (tools/cpp/colosim_ops.cpp): oracle/_ref/ref_ops = the reference's MemoryPool /
    selective_reclaim on one host core, tools/_bin/valve_ops = the same calls through the
    include/colosim drop-in on the B200 (plus the fused single-call reclaim).  Medians in us."""
    import subprocess

    ref = os.path.join(ROOT, "oracle", "_ref", "ref_ops")
    out = {}
    for h in handles:
        row = {}
        for name, exe in (("reference_cpu", ref), ("b200", VALVE_OPS)):
            if not os.path.exists(exe):
                row[name] = {"error": f"{exe} not built"}
                continue
            r = subprocess.run([exe, "table", str(h), ks], capture_output=True, text=True, timeout=600)
            row[name] = json.loads(r.stdout.strip().splitlines()[-1]) if r.returncode == 0 else {"error": r.stderr[-200:]}
        out[str(h)] = row
    return out


def run_reference(args, rank, world):
    threads = os.cpu_count() or 1
    for _ in range(args.warmup):
        cpu_reference(args, 1, threads)
    r = cpu_reference(args, args.steps, threads)
    return {
        "impl": "reference", "metric": METRIC, "value": round(r["value"], 3), "unit": "GB/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(r["secs"] / args.steps * 1e3, 3), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "u8", "data": "synthetic",
        "config": workload_config(args.handles or 1024, args.k, world),
        "p99_preempt_to_quiesce_us": 1000, "p99_note": "reference quiesce is the modeled toggle "
                                                       "constant (scenario.hpp:37), not a timing",
        "cpu_baseline": {"value": round(r["value"], 3), "unit": "GB/s", "cores": threads,
                         "kind": r["kind"],
                         "sample": f"{args.steps} reclaim ops: reference decision path (1 core) + "
                                   f"memcpy gather ({threads} threads)"},
        "e2e": {"value": round(r["value"], 3), "unit": "GB/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }


def main():
    args = parse()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    dist = None
    if args.impl == "reference":
        if rank == 0:
            print(json.dumps(_finite(run_reference(args, rank, world))), flush=True)
        return
    import torch

    if world > 1:
        import torch.distributed as dist

        from paper_2604_07874_b200 import tp as TP

        gpu, shared = TP.rank_device(int(os.environ.get("LOCAL_RANK", "0")),
                                     int(os.environ.get("LOCAL_WORLD_SIZE", str(world))), torch.cuda.device_count())
        torch.cuda.set_device(gpu)
        # rank r on cuda:r; a box with fewer GPUs than ranks (functional runs only) cannot run
        # NCCL with two ranks on one device, so it falls back to gloo for the plumbing
        import datetime

        # a hung collective aborts the job after 30 minutes instead of holding the box (the C4
        # job of up to 20 minutes runs while the other ranks wait in a barrier)
        dist.init_process_group("gloo" if shared else "nccl", timeout=datetime.timedelta(seconds=1800))
        if shared:
            # two contexts time-slicing one GPU with persistent gated kernels make no meaningful
            # (and a very slow) run: keep the replica burst + aggregation only, like --profile-mode
            args.profile_mode = True
            args.skip_realtime = args.skip_fanout = True
            # the ranks on one device split its memory (each would otherwise size a full pool)
            args.ranks_per_device = -(-int(os.environ.get("LOCAL_WORLD_SIZE", str(world))) //
                                      max(1, torch.cuda.device_count()))
            if rank == 0:
                print("bench: fewer GPUs than ranks -- ranks share devices (functional run: no offline tenant, "
                      "no TP / C4 / C5 legs); no number here is a multi-GPU number", file=sys.stderr, flush=True)
    else:
        torch.cuda.set_device(0)
    out = run_valve(args, rank, world, dist)
    if dist is not None and not args.skip_realtime and not args.profile_mode:
        # C4 as its own job on the same GPUs: every rank frees its memory and waits at a barrier
        torch.cuda.empty_cache()
        dist.barrier()
        if rank == 0:
            _progress(rank, "C4 job")
            out["c4_tp_group"] = _guarded("c4_tp_group", lambda: c4_job(world, args))
        dist.barrier()
    if rank == 0:
        try:
            out["cpu_baseline"] = cpu_baseline_block(args)
        except Exception as e:  # the checker must never block the device number
            out["cpu_baseline"] = {"value": None, "error": str(e)[:200]}
        print(json.dumps(_finite(out)), flush=True)
    if dist:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
