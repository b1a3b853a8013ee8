"""C4 (BASELINE.json configs[3]): a tensor-parallel online group over per-rank offline instances,
one process per GPU -- the one place the gate crosses GPUs.

The reference has one node-wide channel: a busy edge on an online lane disables offline compute
on every GPU, and the unpatched toggle costs `toggle x GPUs` (sim.cpp:362-380, 860-873,
scenario.hpp:56-58).  Here:

* every rank owns an independent colocation instance: its own device pool of offline (8B-shaped)
  KV pages and its own gated offline decode pass (k_offline_decode) -- replicas, no NCCL on the
  offline side;
* the TP group's online model is a random-init Llama-3-70B sharded tp ways (attention heads,
  KV heads and MLP columns split per rank, two all-reduces per layer over the TP group --
  the online tenant's own collective, as any TP serving engine has it);
* the group leader runs the serving loop and the host ChannelController bound to the GROUP gate:
  its raise writes every member's gate word over NVLink peer memory and its online stream waits
  until every member's CTAs retired (valve_gate_attach_peers / wait_quiesced); each member's own
  online stream waits for the raise to land on its words and its CTAs to retire
  (valve_gate_wait_closed_quiesced) -- no host round trip on the preemption path;
* steps are decided by the leader and broadcast to the members on a CPU (gloo) group, the way TP
  engines ship step metadata; idle heartbeats let members relaunch their offline pass.

Runs interleave standalone (no offline tenant) and colocated arms over the same recorded plan
(realtime.py's replay: prefills at the recorded decode counts), and report the leader's paired
TTFT / TPOT deltas (metrics.cpp:49-65), the group's preempt-to-quiesce samples and each rank's
harvested offline bytes.  Online KV is not in the pool here (C4 exercises the gate; C2/C3 cover
reclamation on one GPU, realtime.py).
"""
from __future__ import annotations

import heapq
import random
import time
from dataclasses import dataclass, field
from typing import Dict, List, Optional

import torch
import torch.nn.functional as F

from . import api as A
from . import tp as TP
from .realtime import OnlineReq, paired_increase, spike_trace, _med_runs, _pct

TILE = 16384


@dataclass
class C4Config:
    tp: int = 4
    layers: int = 80            # Llama-3-70B: 80 layers, d 8192, 64/8 heads x 128, MLP 28672
    d: int = 8192
    heads: int = 64
    kv_heads: int = 8
    head_dim: int = 128
    ffn: int = 28672
    ctx: int = 2048             # decode attends a dense context of this many tokens per request
    max_batch: int = 16
    horizon_s: float = 30.0
    base: float = 1.0
    spike: float = 8.0
    period: float = 6.0
    width: float = 1.0
    prompt: tuple = (1000, 2000)
    output: tuple = (16, 64)
    handles: int = 64           # offline pool per rank (handles of 64 x 2 MiB Llama-3-8B pages)
    offline_ctas: int = 0       # 0: one CTA set per SM
    max_gap_us: int = 300
    heartbeat_us: int = 2000
    seed: int = 2604


class TPShard:
    """One rank's shard of a random-init Llama-3-70B (bf16): per layer qkv / o / gate-up / down
    column- and row-split over tp ranks; o and down outputs all-reduced over the TP group."""

    def __init__(self, c: C4Config, tp: int, device, group, seed: int):
        assert c.heads % tp == 0 and c.kv_heads % tp == 0 and c.ffn % tp == 0
        self.c, self.dev, self.group = c, device, group
        self.h, self.kvh, self.f = c.heads // tp, c.kv_heads // tp, c.ffn // tp
        g = torch.Generator(device=device).manual_seed(seed)

        def w(*s):
            return (torch.randn(*s, generator=g, device=device) * 0.02).to(torch.bfloat16)

        hd = c.head_dim
        self.layers = [dict(qkv=w(c.d, (self.h + 2 * self.kvh) * hd), o=w(self.h * hd, c.d),
                            w13=w(c.d, 2 * self.f), w2=w(self.f, c.d)) for _ in range(c.layers)]
        # decode context: per layer K and V for max_batch requests x ctx tokens (read every step)
        self.kv = [torch.randn(2, c.max_batch, self.kvh, c.ctx, hd, generator=g, device=device).to(torch.bfloat16)
                   for _ in range(c.layers)]

    @staticmethod
    def _rms(x):
        return x * torch.rsqrt(x.float().pow(2).mean(-1, keepdim=True) + 1e-5).to(x.dtype)

    def _ar(self, x):
        torch.distributed.all_reduce(x, group=self.group)
        return x

    def _layer(self, L, x, attn):
        c, hd = self.c, self.c.head_dim
        q, k, v = (self._rms(x) @ L["qkv"]).split([self.h * hd, self.kvh * hd, self.kvh * hd], -1)
        x = x + self._ar(attn(q, k, v) @ L["o"])
        g1, g3 = (self._rms(x) @ L["w13"]).chunk(2, -1)
        return x + self._ar((F.silu(g1) * g3) @ L["w2"])

    @torch.no_grad()
    def prefill(self, T: int):
        hd = self.c.head_dim
        x = torch.randn(T, self.c.d, device=self.dev, dtype=torch.bfloat16) * 0.02

        def attn(q, k, v):
            q = q.view(T, self.h, hd).transpose(0, 1)
            k = k.view(T, self.kvh, hd).transpose(0, 1)
            v = v.view(T, self.kvh, hd).transpose(0, 1)
            o = F.scaled_dot_product_attention(q, k, v, is_causal=True, enable_gqa=True)
            return o.transpose(0, 1).reshape(T, -1)

        for L in self.layers:
            x = self._layer(L, x, attn)
        return x

    @torch.no_grad()
    def decode(self, B: int):
        hd = self.c.head_dim
        x = torch.randn(B, self.c.d, device=self.dev, dtype=torch.bfloat16) * 0.02
        for li, L in enumerate(self.layers):
            kv = self.kv[li]

            def attn(q, k, v, kv=kv):
                o = F.scaled_dot_product_attention(q.view(B, self.h, 1, hd), kv[0, :B], kv[1, :B], enable_gqa=True)
                return o.reshape(B, -1)

            x = self._layer(L, x, attn)
        return x


@dataclass
class C4Run:
    policy: str
    ttft_us: Dict[int, float] = field(default_factory=dict)
    tpot_us: Dict[int, float] = field(default_factory=dict)
    plan: list = field(default_factory=list)
    quiesce_us: List[float] = field(default_factory=list)
    disables: int = 0
    offline_tiles: int = 0
    wall_s: float = 0.0
    step_ms: List[float] = field(default_factory=list)


class C4Instance:
    """One rank of the TP group.  Collective calls line up across ranks: every rank runs the same
    sequence of broadcasts and all-reduces."""

    def __init__(self, c: C4Config, rank: int, world: int, dist, device: int, shared: bool):
        self.c, self.rank, self.world, self.dist, self.gpu = c, rank, world, dist, device
        self.dev = torch.device("cuda", device)
        groups = TP.tp_groups(world, c.tp)
        self.members = TP.group_of(rank, groups)
        self.leader = self.members[0]
        self.is_leader = rank == self.leader
        # every rank creates every group's sub-communicators, in the same order
        self.cpu_group = self.tp_group = None
        for g in groups:
            cg = dist.new_group(g, backend="gloo")
            tg = dist.new_group(g, backend="gloo" if shared else "nccl")
            if rank in g:
                self.cpu_group, self.tp_group = cg, tg
        self.model = TPShard(c, c.tp, self.dev, self.tp_group, seed=c.seed + rank)
        self.pool = A.DevicePool(c.handles, 64, 16, device=device, slot_bytes=2 << 20, page_bytes=2 << 20,
                                 max_requests=4096, max_pages_per_request=1024)
        rng = random.Random(c.seed + 17 * rank)
        rid = 0
        while self.pool.offline_reserve(rid, rng.randint(125, 250), rid):  # 2k-4k token 8B requests
            rid += 1
        self.pool.fill_pages()
        self.gate = A.Gate(device)
        self.group = TP.TPGate(self.gate, rank, world, c.tp, dist, opener=TP.open_member(device))
        self.online = torch.cuda.Stream(device=self.dev, priority=-1)
        self.off = torch.cuda.Stream(device=self.dev)
        self.off_done: Optional[torch.cuda.Event] = None
        self.tiles_prev = 0

    # ------------------------------------------------------------------ offline tenant
    def _offline_tick(self):
        """Keep one gated launch queued: relaunch when the previous one retired (a finished pass
        starts over with a fresh work list)."""
        if self.off_done is not None and not self.off_done.query():
            return
        st = self.gate.read()
        if st.live_ctas:
            return
        if st.total_tiles and st.tiles_claimed >= st.total_tiles:
            self.tiles_prev += st.tiles_done
            self.gate.reset_work()
        self.gate.launch_offline(self.pool, None, None, 0, 0, None, ctas=self.c.offline_ctas,
                                 stream=self.off.cuda_stream)
        self.off_done = torch.cuda.Event()
        self.off_done.record(self.off)

    def _offline_stop(self):
        """Raise (leader), every rank drops its work list, release: queued launches retire."""
        if self.is_leader:
            gen = 1 << 30
            self.group.raise_(gen, self.online.cuda_stream)
            self.group.wait_quiesced(gen, self.online.cuda_stream)
            self.online.synchronize()
        self.dist.barrier(group=self.cpu_group)
        st = self.gate.read()
        tiles = self.tiles_prev + st.tiles_done
        self.gate.cancel_work()
        self.dist.barrier(group=self.cpu_group)
        if self.is_leader:
            self.group.release(1 << 30, self.online.cuda_stream)
            self.online.synchronize()
        self.off.synchronize()
        self.dist.barrier(group=self.cpu_group)
        return tiles

    # ------------------------------------------------------------------ one run
    def run(self, trace: List[OnlineReq], policy: str, plan: Optional[list] = None) -> C4Run:
        c = self.c
        res = C4Run(policy)
        colo = policy != "standalone"
        timers: list = []
        seq = [0]
        channel = None
        self.gate.reset_work()
        self.tiles_prev, self.off_done = 0, None
        if colo:
            self._offline_tick()
            if self.is_leader:
                def sched(when, gen, cd):
                    heapq.heappush(timers, (int(when), seq[0], cd, gen))
                    seq[0] += 1

                hooks = A.Hooks(schedule=sched, on_disabled=lambda t: None, on_enabled=lambda t: None)
                channel = A.ChannelController(0, A.CooldownPolicy(c.max_gap_us).cooldown_us(), hooks,
                                              gate=self.gate, gate_stream=self.online.cuda_stream)
        torch.cuda.synchronize(self.dev)
        self.dist.barrier(group=self.cpu_group)
        reqs = [OnlineReq(r.rid, r.arrival_us, r.prompt, r.output) for r in trace]
        by = {r.rid: r for r in reqs}
        queue: List[OnlineReq] = []
        decoding: List[OnlineReq] = []
        nxt = pi = n_dec = 0
        busy = False
        last_beat = 0
        waits = []
        t0 = time.perf_counter()
        now_us = lambda: int((time.perf_counter() - t0) * 1e6)  # noqa: E731
        stop_us = int((c.horizon_s + 60) * 1e6)
        while True:
            msg = None
            if self.is_leader:
                while msg is None:
                    now = now_us()
                    while channel is not None and timers and timers[0][0] <= now:
                        when, _, cd, gen = heapq.heappop(timers)
                        (channel.handle_cooldown if cd else channel.handle_toggle)(when, gen)
                    while nxt < len(reqs) and reqs[nxt].arrival_us <= now:
                        queue.append(reqs[nxt])
                        nxt += 1
                    act = None
                    if plan is None:
                        if queue and (not decoding or len(decoding) < c.max_batch):
                            act = ("prefill", queue[0].rid)
                        elif decoding:
                            act = ("decode", len(decoding))
                        done = act is None and nxt >= len(reqs)
                    else:
                        done = pi >= len(plan) and not decoding
                        if pi < len(plan) and (n_dec >= plan[pi][1] or not decoding):
                            if by[plan[pi][0]].arrival_us <= now:
                                act = ("prefill", plan[pi][0])
                            elif decoding:
                                continue  # spin: the lane stays busy until the planned arrival
                        elif decoding:
                            act = ("decode", len(decoding))
                    if done or now > stop_us:
                        msg = ("stop", 0, False)
                    elif act is not None:
                        edge = not busy
                        if edge and channel is not None:
                            channel.note_busy(now)
                        msg = (act[0], act[1], edge)
                        busy = True
                    else:
                        if busy:
                            busy = False
                            if channel is not None:
                                channel.note_all_idle(now)
                        if now - last_beat >= c.heartbeat_us:
                            last_beat = now
                            msg = ("idle", 0, False)
                        else:
                            time.sleep(50e-6)
            box = [msg]
            self.dist.broadcast_object_list(box, src=self.leader, group=self.cpu_group)
            kind, arg, edge = box[0]
            if kind == "stop":
                break
            if kind == "idle":
                if colo:
                    self._offline_tick()
                continue
            if edge and colo:  # busy edge: the group gate is raised (leader's channel hook)
                if self.is_leader:
                    gen = channel.disables_issued()
                    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    e0.record(self.online)
                    self.group.wait_quiesced(gen, self.online.cuda_stream)
                    e1.record(self.online)
                    waits.append((e0, e1))
                else:
                    self.gate.wait_closed_quiesced(self.online.cuda_stream)
            t_s = time.perf_counter()
            with torch.cuda.stream(self.online):
                if kind == "prefill":
                    self.model.prefill(by[arg].prompt)
                else:
                    self.model.decode(min(arg, c.max_batch))
            self.online.synchronize()
            if colo:
                self._offline_tick()  # queue the next launch: it waits on the device for the release
            if not self.is_leader:
                continue
            t_e = now_us()
            res.step_ms.append((time.perf_counter() - t_s) * 1e3)
            if kind == "prefill":
                r = by[arg]
                queue.remove(r)
                res.plan.append((r.rid, n_dec))
                pi += 1
                decoding.append(r)
                continue
            n_dec += 1
            fin = []
            for r in decoding[: c.max_batch]:
                r.emits.append(t_e)
                if len(r.emits) == r.output:
                    fin.append(r)
            for r in fin:
                decoding.remove(r)
                res.ttft_us[r.rid] = r.emits[0] - r.arrival_us
                if r.output > 1:
                    res.tpot_us[r.rid] = (r.emits[-1] - r.emits[0]) / (r.output - 1)
        res.wall_s = time.perf_counter() - t0
        if colo:
            res.offline_tiles = self._offline_stop()
            if self.is_leader:
                res.disables = channel.disables_issued()
                res.quiesce_us = [a.elapsed_time(b) * 1e3 for a, b in waits]
        return res


def measure(dist, rank: int, world: int, device: int, shared: bool, c: Optional[C4Config] = None,
            repeats: int = 1) -> Optional[dict]:
    """Interleaved standalone / colocated runs of one TP group per `c.tp` ranks (every group runs
    its own instance).  Returns the report on each group leader (None on members)."""
    c = c or C4Config()
    inst = C4Instance(c, rank, world, dist, device, shared)
    trace = spike_trace(c.seed, c.horizon_s, c.base, c.spike, c.period, c.width, prompt=c.prompt, output=c.output)
    inst.model.prefill(c.prompt[1])  # first-use costs (cuBLAS heuristics, NCCL channels)
    inst.model.decode(c.max_batch)
    torch.cuda.synchronize(inst.dev)
    plan = inst.run(trace, "standalone").plan  # untimed: records the action sequence
    box = [plan]
    dist.broadcast_object_list(box, src=inst.leader, group=inst.cpu_group)
    plan = box[0]
    solos, colos = [], []
    for _ in range(repeats):
        solos.append(inst.run(trace, "standalone", plan))
        colos.append(inst.run(trace, "valve", plan))
    solos.append(inst.run(trace, "standalone", plan))
    gathered = [None] * world
    dist.all_gather_object(gathered, (rank, [r.offline_tiles for r in colos], [r.wall_s for r in colos]))
    if not inst.is_leader:
        return None
    base_t, base_p = _med_runs([s.ttft_us for s in solos]), _med_runs([s.tpot_us for s in solos])
    tt = paired_increase(base_t, _med_runs([r.ttft_us for r in colos]))
    tp_ = paired_increase(base_p, _med_runs([r.tpot_us for r in colos]))
    aa_t = paired_increase(_med_runs([s.ttft_us for s in solos[0::2]]), _med_runs([s.ttft_us for s in solos[1::2]]))
    aa_p = paired_increase(_med_runs([s.tpot_us for s in solos[0::2]]), _med_runs([s.tpot_us for s in solos[1::2]]))
    q = sorted(x for r in colos for x in r.quiesce_us)
    per_rank = {str(rk): {"offline_gb": [t * TILE / 1e9 for t in tl],
                          "offline_gbs": [t * TILE / w / 1e9 for t, w in zip(tl, ws)]}
                for rk, tl, ws in gathered if rk in inst.members}
    return {
        "config": "C4: Llama-3-70B-shaped TP=%d online (%d layers, random init bf16) + per-rank Llama-3-8B-shaped "
                  "offline KV pools (%d x 128 MiB handles) under one group gate" % (c.tp, c.layers, c.handles),
        "group": inst.members, "shared_device": shared,
        "trace": {"horizon_s": c.horizon_s, "online_requests": len(trace), "base_rate": c.base,
                  "spike_rate": c.spike, "period_s": c.period, "width_s": c.width},
        "ttft_delta_pct": tt["mean_pct"], "tpot_delta_pct": tp_["mean_pct"], "pairs": tt["pairs"],
        "aa_noise_ttft_pct": aa_t["mean_pct"], "aa_noise_tpot_pct": aa_p["mean_pct"],
        "group_quiesce_us": {"p50": _pct(q, 50), "p99": _pct(q, 99), "max": q[-1] if q else None, "n": len(q)},
        "disables": [r.disables for r in colos], "online_requests": len(trace),
        "decode_step_ms_p50": _pct([x for s in solos for x in s.step_ms], 50),
        "per_rank_offline": per_rank,
        "plan_prefills": len(plan),
    }
