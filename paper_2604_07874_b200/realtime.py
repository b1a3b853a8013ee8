"""Real-time colocation loop on one B200: measured online TTFT/TPOT deltas.

A thin runtime around the product kernels, following the reference simulator's online/offline
engines (sim.cpp:391-858) but in wall-clock time on the device:

* online: a random-init Llama-3-8B-shaped decoder in PyTorch (bf16, cuBLAS GEMMs, SDPA
  attention; never gated -- it is the latency-critical tenant).  Prefill emits no token; a
  decode iteration emits one token for every decoding request (sim.cpp:625-719).
* offline: the gated tile-looped kernel over the pool's offline KV pages
  (valve_offline_launch), running whenever the ChannelController is Enabled.
* lane edges drive the host ChannelController (channel.cpp), bound to the HBM gate: the busy
  edge raises the gate and the online stream waits (cuStreamWaitValue) for every offline CTA to
  retire before its first kernel; idle edge -> cooldown T_cool = 2G -> enable -> gate released ->
  offline relaunched from its HBM cursor.
* online KV pages are charged against the reservation on the device pool (MemoryPool API):
  free handles first, otherwise a fused device reclaim of k offline handles (Algorithm 1 +
  apply_reclaim) whose evicted requests are re-admitted later -- sim.cpp:469-556.

The same online trace is run standalone (no offline tenant, no gate) and colocated; the deltas
are the reference's paired per-request increases (metrics.cpp:49-65, 231-241).
"""
from __future__ import annotations

import heapq
import math
import random
import time
from dataclasses import dataclass, field
from typing import Dict, List, Optional

import torch
import torch.nn.functional as F

from . import api as A


# ------------------------------------------------------------------------- online model

@dataclass
class ModelShape:
    """Llama-3-8B: 32 layers, d 4096, GQA 32/8 heads x 128, MLP 14336, vocab 128256."""
    layers: int = 32
    d: int = 4096
    heads: int = 32
    kv_heads: int = 8
    head_dim: int = 128
    ffn: int = 14336
    vocab: int = 128256


class OnlineModel:
    """Random-init (N(0, 0.02), bf16) decoder.  KV lives in per-layer slot tensors
    [slots, kv_heads, max_tokens, head_dim]; prefill uses SDPA (causal, flash-eligible),
    decode attends the whole batch at once with a length mask."""

    def __init__(self, shape: ModelShape, device, seed: int = 0, slots: int = 16, max_tokens: int = 4352):
        g = torch.Generator(device=device).manual_seed(seed)
        s = shape
        self.s = s
        dt = torch.bfloat16

        def w(*shape_):
            return (torch.randn(*shape_, generator=g, device=device, dtype=torch.float32) * 0.02).to(dt)

        qkv = (s.heads + 2 * s.kv_heads) * s.head_dim
        self.layers = [dict(wqkv=w(s.d, qkv), wo=w(s.heads * s.head_dim, s.d), w13=w(s.d, 2 * s.ffn),
                            w2=w(s.ffn, s.d)) for _ in range(s.layers)]
        self.emb = w(s.vocab, s.d)
        self.lm = w(s.d, s.vocab)
        self.device = device
        self.max_tokens = max_tokens
        self.K = [torch.zeros(slots, s.kv_heads, max_tokens, s.head_dim, device=device, dtype=dt)
                  for _ in range(s.layers)]
        self.V = [torch.zeros_like(k) for k in self.K]
        self.free_slots = list(range(slots))

    @staticmethod
    def _rms(x):
        return x * torch.rsqrt(x.float().pow(2).mean(-1, keepdim=True) + 1e-5).to(x.dtype)

    def _qkv(self, L, x):
        s = self.s
        h = self._rms(x) @ L["wqkv"]
        return h.split([s.heads * s.head_dim, s.kv_heads * s.head_dim, s.kv_heads * s.head_dim], -1)

    def _mlp(self, L, x, a):
        x = x + a @ L["wo"]
        g1, g3 = (self._rms(x) @ L["w13"]).chunk(2, -1)
        return x + (F.silu(g1) * g3) @ L["w2"]

    def alloc(self):
        return self.free_slots.pop()

    def free(self, slot):
        self.free_slots.append(slot)

    @torch.no_grad()
    def prefill(self, tokens, slot):
        s = self.s
        T = tokens.shape[0]
        rep = s.heads // s.kv_heads
        x = self.emb[tokens]
        for li, L in enumerate(self.layers):
            q, k, v = self._qkv(L, x)
            kh = k.view(T, s.kv_heads, s.head_dim).transpose(0, 1)
            vh = v.view(T, s.kv_heads, s.head_dim).transpose(0, 1)
            self.K[li][slot, :, :T] = kh
            self.V[li][slot, :, :T] = vh
            qh = q.view(T, s.heads, s.head_dim).transpose(0, 1).unsqueeze(0)
            o = F.scaled_dot_product_attention(qh, kh.repeat_interleave(rep, 0).unsqueeze(0),
                                               vh.repeat_interleave(rep, 0).unsqueeze(0), is_causal=True)
            x = self._mlp(L, x, o[0].transpose(0, 1).reshape(T, -1))
        return (self._rms(x[-1:]) @ self.lm).argmax(-1)

    @torch.no_grad()
    def decode(self, tokens, slots, lens):
        s = self.s
        B = tokens.shape[0]
        rep = s.heads // s.kv_heads
        idx = torch.tensor(slots, device=self.device)
        pos = torch.tensor(lens, device=self.device)
        n = max(lens) + 1
        mask = torch.arange(n, device=self.device)[None, :] <= pos[:, None]  # (B, n)
        bias = torch.zeros(B, 1, 1, n, device=self.device, dtype=torch.float32)
        bias.masked_fill_(~mask[:, None, None, :], float("-inf"))
        scale = 1.0 / math.sqrt(s.head_dim)
        x = self.emb[tokens]
        for li, L in enumerate(self.layers):
            q, k, v = self._qkv(L, x)
            self.K[li][idx, :, pos] = k.view(B, s.kv_heads, s.head_dim)
            self.V[li][idx, :, pos] = v.view(B, s.kv_heads, s.head_dim)
            Kb = self.K[li][idx, :, :n]  # (B, G, n, D)
            Vb = self.V[li][idx, :, :n]
            qg = q.view(B, s.kv_heads, rep, s.head_dim)
            sc = torch.matmul(qg, Kb.transpose(-1, -2)).float() * scale + bias
            a = torch.matmul(sc.softmax(-1).to(Vb.dtype), Vb)  # (B, G, rep, D)
            x = self._mlp(L, x, a.reshape(B, -1))
        return (self._rms(x) @ self.lm).argmax(-1)


# ------------------------------------------------------------------------------ trace

@dataclass
class OnlineReq:
    rid: int
    arrival_us: int
    prompt: int
    output: int
    first_us: int = -1
    emits: List[int] = field(default_factory=list)
    pages: int = 0


def spike_trace(seed: int, horizon_s: float, base_rate: float, spike_rate: float, period_s: float,
                width_s: float, prompt=(2000, 4000), output=(32, 128)) -> List[OnlineReq]:
    """Poisson arrivals at base_rate, spike_rate inside [k*period, k*period + width)
    (the reference's 'spike' generator shape, trace.cpp:131-183)."""
    rng = random.Random(seed)
    out, t, rid = [], 0.0, 0
    while True:
        in_spike = (t % period_s) < width_s
        rate = spike_rate if in_spike else base_rate
        t += rng.expovariate(rate)
        if t >= horizon_s:
            break
        out.append(OnlineReq(rid, int(t * 1e6), rng.randint(*prompt), rng.randint(*output)))
        rid += 1
    return out


# ------------------------------------------------------------------------- event log

class EventLog:
    """The reference's events.jsonl schema (log.hpp:13-59, writer log.cpp:69-217): the same
    kinds, field names and key order, so the reference's own build_report / ttft_increase /
    tpot_increase (metrics.cpp:85-241) recompute the deltas from these logs (tests pin that)."""

    def __init__(self):
        self.recs = []

    def add(self, t: int, kind: str, **fields):
        self.recs.append((int(t), len(self.recs), kind, fields))

    def records(self):
        """Records in time order (ties keep emission order), sequence numbers reassigned."""
        out = []
        for seq, (t, _, kind, fields) in enumerate(sorted(self.recs, key=lambda r: (r[0], r[1]))):
            out.append(dict(time_us=t, seq=seq, kind=kind, **fields))
        return out

    def write_jsonl(self, path: str):
        import json

        with open(path, "w") as f:
            for r in self.records():
                f.write(json.dumps(r, separators=(",", ":")) + "\n")


def trace_fingerprint(trace: List["OnlineReq"]) -> str:
    """A u64 of the online trace (arrival, prompt, output per request) -- pairs runs the way
    the reference's online_fingerprint does (metrics.cpp:231-241 refuses unpaired logs)."""
    import hashlib

    h = hashlib.sha256(repr([(r.rid, r.arrival_us, r.prompt, r.output) for r in trace]).encode())
    return "0x" + h.hexdigest()[:16]


# ------------------------------------------------------------------------- the runtime

@dataclass
class RunResult:
    ttft_us: Dict[int, float]
    tpot_us: Dict[int, float]
    wall_s: float
    disables: int = 0
    reclaims: int = 0
    reclaimed_handles: int = 0
    offline_tiles: int = 0
    offline_bytes: float = 0.0
    offline_gemm_tiles: int = 0
    offline_gemm_flop: float = 0.0
    offline_gemms_done: float = 0.0
    quiesce_wait_us: List[float] = field(default_factory=list)
    decode_iter_us: List[float] = field(default_factory=list)
    prefill_us: List[float] = field(default_factory=list)
    # time the colocation mechanism itself put on each request's critical path: the busy-edge
    # quiesce wait (CUDA events on the online stream) + page acquisition incl. reclaim (host)
    mech_ttft_us: Dict[int, float] = field(default_factory=dict)
    mech_tpot_us: Dict[int, float] = field(default_factory=dict)
    log: EventLog = field(default_factory=EventLog)
    plan: list = field(default_factory=list)  # the action sequence this run executed


class Colocation:
    def __init__(self, model: OnlineModel, pool: Optional[A.DevicePool], gate: Optional[A.Gate],
                 page_tokens: int = 16, max_gap_us: int = 300, resparams: Optional[A.ReservationParams] = None,
                 tile_bytes: int = 16384, offline_ctas: int = 0, offline_gemm=None, offline_gemm_ctas: int = 0):
        """offline_gemm=(m, n, k): the offline tenant also runs the gated tcgen05 GEMM (its
        projection work, e.g. Qwen2-7B gate/up over m tokens) next to the decode pass, on its own
        gate attached to the channel's gate, so one raise quiesces both.
        offline_gemm=("qwen2-7b", m): the tenant runs a random-init Qwen2-7B's projection chain
        instead -- 28 layers x (qkv, o, gate/up, down) gated GEMMs over m tokens, each preempted
        and resumed at tile granularity, the chain advancing when a GEMM's work list completes."""
        self.model, self.pool, self.gate = model, pool, gate
        self.page_tokens = page_tokens
        self.tile_bytes = tile_bytes
        self.offline_ctas = offline_ctas  # 0 = library default (2 CTAs of 8 warps per SM); < 0 = no decode pass
        self.colocated = pool is not None
        self.online_stream = torch.cuda.current_stream()
        self.off_stream = torch.cuda.Stream()
        self.resctl = A.ReservationController(resparams) if self.colocated else None
        self.timers: list = []
        self.seq = 0
        self.offline_running = False
        self.gemm_gate = None
        self.gemm_ctas = offline_gemm_ctas  # 0 = one CTA per SM (power knob: fewer SMs, less draw)
        if self.colocated and offline_gemm:
            dev = model.device
            g = torch.Generator(device=dev).manual_seed(7)

            def rnd(*shape, scale=1.0):
                return (torch.randn(*shape, device=dev, generator=g) * scale).to(torch.bfloat16)

            self.gemm_seq = []  # (a, b, c, m, n, k, tiles) in execution order
            if offline_gemm[0] == "qwen2-7b":
                m = int(offline_gemm[1])
                d, qkv, ffn, layers = 3584, 4608, 18944, 28  # Qwen2-7B: 28 x (28 q + 2 x 4 kv heads x 128)
                x, act = rnd(m, d), rnd(m, ffn)
                outs = {n: torch.empty(m, n, device=dev, dtype=torch.bfloat16) for n in (qkv, d, 2 * ffn)}
                for _ in range(layers):
                    for (a, n, k) in ((x, qkv, d), (x, d, d), (x, 2 * ffn, d), (act, d, ffn)):
                        self.gemm_seq.append((a, rnd(n, k, scale=0.02), outs[n], m, n, k))
            else:
                m, n, k = offline_gemm
                self.gemm_seq.append((rnd(m, k), rnd(n, k, scale=0.02), torch.empty(m, n, device=dev, dtype=torch.bfloat16),
                                      m, n, k))
            self.gemm_seq = [(a, b, c, m, n, k, (m // (256 if m % 256 == 0 else 128)) * (n // 256))
                             for (a, b, c, m, n, k) in self.gemm_seq]
            self.gemm_gate = A.Gate(dev.index if dev.index is not None else 0)
            gate.attach_peers([self.gemm_gate])
            self.gemm_stream = torch.cuda.Stream()
        if self.colocated:
            hooks = A.Hooks(schedule=self._schedule, on_disabled=lambda t: None,
                            on_enabled=self._on_enabled, log=None)
            # real time: the device gate takes effect at issue; its quiesce is waited on the
            # online stream, so the modelled toggle latency is 0 (channel.cpp:13-20)
            self.channel = A.ChannelController(0, A.CooldownPolicy(max_gap_us).cooldown_us(), hooks, gate=gate)

    # timers (the channel's schedule hook, in run microseconds)
    def _schedule(self, when, gen, cooldown):
        heapq.heappush(self.timers, (when, self.seq, cooldown, gen))
        self.seq += 1

    def _fire_timers(self, now):
        while self.timers and self.timers[0][0] <= now:
            when, _, cd, gen = heapq.heappop(self.timers)
            (self.channel.handle_cooldown if cd else self.channel.handle_toggle)(when, gen)

    def _on_enabled(self, t):
        self.res.log.add(t, "enable_issued", effective_us=int(t))
        self._launch_offline()

    def _launch_offline(self):
        if not self.colocated:
            return
        self._launch_decode()
        if self.gemm_gate is not None:
            self._launch_gemm()

    def _launch_gemm(self):
        st = self.gemm_gate.read()
        a, b, c, m, n, k, tiles = self.gemm_seq[self._gemm_idx]
        fresh = st.tiles_claimed >= tiles  # this GEMM's work list finished: the next one
        if fresh:
            self._gemm_flop += 2.0 * m * n * k
            self._gemm_done += 1
            self._gemm_idx = (self._gemm_idx + 1) % len(self.gemm_seq)
            a, b, c, m, n, k, tiles = self.gemm_seq[self._gemm_idx]
        self.gemm_gate.launch_gemm(a.data_ptr(), b.data_ptr(), c.data_ptr(), m, n, k, ctas=self.gemm_ctas,
                                   stream=self.gemm_stream.cuda_stream, fresh=fresh)

    def _launch_decode(self):
        if self.offline_ctas < 0:
            return
        st = self.gate.read()
        total = self._offline_tiles_total()
        if total and st.tiles_claimed >= total:  # work list exhausted: start another pass
            self._harvest += st.tiles_done
            self.gate.reset_work()
        self.gate.launch_offline(self.pool, None, None, 0, 0, None, stream=self.off_stream.cuda_stream,
                                 tile_bytes=self.tile_bytes, ctas=self.offline_ctas)

    def _offline_tiles_total(self):
        return self._off_pages * (-(-self.pool.page_bytes // self.tile_bytes)) if self.colocated else 0

    # ------------------------------------------------------------------ memory (sim.cpp)
    def _acquire_online_pages(self, need, now):
        """sim.cpp:469-511 + 535-556: reservation growth from free handles, then a fused
        device reclaim for the shortfall; pressure growth after the charge."""
        P = self.pool
        hsz = P.handle_size_pages()
        deficit = P.online_used_pages() + need - P.online_capacity_pages()
        if deficit > 0:
            k = -(-deficit // hsz)
            from_free = min(k, P.free_handles())
            if from_free:
                P.online_grow(from_free, now)
            deficit -= from_free * hsz
        if deficit > 0:
            self.resctl.record_pressure(now)
            k = min(-(-deficit // hsz), P.offline_handles())
            if k:
                self._reclaim(k, now)
        P.online_use_pages(need)
        cap = P.online_capacity_pages()
        if cap and P.online_used_pages() / cap >= self.resctl.params().pressure_threshold:
            self.resctl.record_pressure(now)
            h = P.online_handles()
            want = self.resctl.grow_target(h, P.total_handles()) - h
            from_free = min(max(want, 0), P.free_handles())
            if from_free:
                P.online_grow(from_free, now)
            want -= from_free
            if want > 0 and P.offline_handles():
                self._reclaim(min(want, P.offline_handles()), now)

    def _reclaim(self, k, now):
        op = self.res.reclaims
        self.res.log.add(now, "reclaim_request", gpu=0, handles=int(k), op=op, purpose="shortfall")
        t_r = time.perf_counter()
        nh, ne, npg = self.pool.reclaim(k, now)
        res = self.pool.last_reclaim()
        self.res.log.add(now, "reclaim_done", gpu=0, op=op, latency_us=int((time.perf_counter() - t_r) * 1e6),
                         handle_ids=list(res.handles))
        for r in res.evicted_requests:
            self.res.log.add(now, "evicted", request_id=int(r), gpu=0, recompute_tokens=int(self._off_cost.get(r, 0)))
        self.res.reclaims += 1
        self.res.reclaimed_handles += nh
        for r in res.evicted_requests:  # evicted-waiting -> re-admitted when memory frees
            self._evicted.append(r)
            self._off_pages -= self._off_live.pop(r, 0)

    def _readmit_offline(self, now):
        """sim.cpp:730-753 admit_offline: resume evicted requests first."""
        P = self.pool
        while self._evicted:
            r = self._evicted[0]
            pages = self._off_req_pages[r]
            if not P.offline_reserve(r, pages, now):
                break
            self._evicted.pop(0)
            self._off_live[r] = pages
            self._off_pages += pages
        if self._off_live:
            P.set_costs({r: self._off_cost[r] for r in self._off_live})

    # ------------------------------------------------------------------------ main loop
    def run(self, trace: List[OnlineReq], offline_reqs=(), horizon_s: float = 30.0,
            plan: Optional[list] = None, admit_margin_us: int = 0) -> RunResult:
        """plan=None: the serving loop schedules (FIFO prefill-first, whole-batch decode) and the
        result records, per prefill, (request, decode iterations completed before it) in res.plan.
        plan=<a recorded list>: prefills happen in the recorded order at the recorded decode
        counts (never before the request's arrival; if it arrives later than in the recording the
        prefill goes at the first boundary after it), so a paired run differs from its baseline
        only in how long each step takes -- not in which decode iterations a prefill happened to
        fall between (a wall-clock loop flips that on microseconds of jitter, moving a request's
        TPOT by several ms).  admit_margin_us (recording runs): while a batch is decoding, a
        request is prefilled only at a boundary at least this long after its arrival, so a replay
        whose clock runs a little ahead of the recording still finds it arrived."""
        m = self.model
        self.res = RunResult({}, {}, 0.0)
        pi = 0  # next planned prefill
        n_decodes = 0  # decode iterations so far (the replay clock)
        by_rid = {}
        self._evicted, self._off_live, self._off_req_pages, self._off_cost = [], {}, {}, {}
        self._off_pages = 0
        self._harvest = 0
        self._gemm_flop, self._gemm_done, self._gemm_idx = 0.0, 0, 0
        reqs = [OnlineReq(r.rid, r.arrival_us, r.prompt, r.output) for r in trace]
        by_rid = {r.rid: r for r in reqs}
        log = self.res.log
        log.add(0, "run_meta", scenario="realtime_spike", preset="valve" if self.colocated else "standalone",
                seed=0, gpus=1, horizon_us=int(horizon_s * 1e6), online_fingerprint=trace_fingerprint(trace),
                offline_fingerprint="0x%016x" % len(offline_reqs))
        busy_since = 0
        preempt_rids = []
        if self.colocated:
            P = self.pool
            P.online_grow(-(-P.total_handles() // 10), 0)
            for rid, pages, cost in offline_reqs:
                self._off_req_pages[rid] = pages
                self._off_cost[rid] = cost
                if P.offline_reserve(rid, pages, 0):
                    self._off_live[rid] = pages
                    self._off_pages += pages
            P.set_costs({r: self._off_cost[r] for r in self._off_live})
            P.fill_pages()
            self.gate.reset_work()
            if self.gemm_gate is not None:
                self.gemm_gate.reset_work()
            self._launch_offline()
        queue: List[OnlineReq] = []
        decoding: List[OnlineReq] = []
        caches: Dict[int, int] = {}  # request -> KV slot
        lens: Dict[int, int] = {}
        nxt = 0
        busy = False
        pending_wait = None
        wait_events = []
        torch.cuda.synchronize()
        import gc

        gc.collect()
        gc_was = gc.isenabled()
        gc.disable()  # a generation-2 collection in the loop is a 10-100 ms stall on either arm
        t0 = time.perf_counter()
        now_us = lambda: int((time.perf_counter() - t0) * 1e6)  # noqa: E731
        while True:
            now = now_us()
            if now > horizon_s * 1e6:
                break
            if self.colocated:
                self._fire_timers(now)
            while nxt < len(reqs) and reqs[nxt].arrival_us <= now:
                r = reqs[nxt]
                log.add(r.arrival_us, "arrival", **{"class": "online"}, request_id=r.rid, gpu=0,
                        prompt_tokens=r.prompt, output_tokens=r.output)
                queue.append(r)
                nxt += 1
            act = None  # next action: ("prefill", rid) / ("decode", batch size); None = idle
            if plan is None:
                if queue and (not decoding or queue[0].arrival_us <= now - admit_margin_us):
                    act = ("prefill", queue[0].rid)
                elif decoding:
                    act = ("decode", len(decoding))
                finished = act is None and nxt >= len(reqs)
            else:
                # prefill the next planned request at the decode count it had in the recording
                # (or at the first boundary after its arrival if this run got there earlier)
                finished = pi >= len(plan) and not decoding
                if pi < len(plan):
                    rid, k = plan[pi]
                    if by_rid[rid].arrival_us <= now and (n_decodes >= k or not decoding):
                        act = ("prefill", rid)
                if act is None and decoding:
                    act = ("decode", len(decoding))
            if act is None:
                if busy:  # idle edge (sim.cpp:371-380)
                    busy = False
                    log.add(now, "busy", gpu=0, **{"class": "online"}, start_us=busy_since, end_us=now)
                    if self.colocated:
                        self.channel.note_all_idle(now)
                        self._readmit_offline(now)
                if finished:
                    break
                if self.colocated and self.channel.offline_compute_allowed():
                    # the offline engine's next iteration: a pass over its KV finished -> relaunch
                    if self.offline_ctas >= 0 and self.gate.read().live_ctas == 0:
                        self._launch_decode()
                    if self.gemm_gate is not None and self.gemm_gate.read().live_ctas == 0:
                        self._launch_gemm()
                time.sleep(50e-6)
                continue
            if act[0] == "prefill":
                self.res.plan.append((act[1], n_decodes))
                pi += 1
            else:
                n_decodes += 1
            if not busy:  # busy edge: raise + wait for the offline CTAs to retire (sim.cpp:362-369)
                busy = True
                busy_since = now
                if self.colocated:
                    log.add(now, "disable_issued", effective_us=now, cause="busy")
                    self.channel.note_busy(now)
                    self._fire_timers(now)
                    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    e0.record(self.online_stream)
                    self.gate.wait_quiesced(self.channel.disables_issued(), self.online_stream.cuda_stream)
                    e1.record(self.online_stream)
                    pending_wait = (e0, e1)  # charged to the request this edge admits
                    self.res.disables = self.channel.disables_issued()
            if act[0] == "prefill":  # prefill the queue head (or the planned request)
                r = by_rid[act[1]]
                queue.remove(r)
                need = -(-r.prompt // self.page_tokens)
                if self.colocated:
                    ta = time.perf_counter()
                    self._acquire_online_pages(need, now)
                    self.res.mech_ttft_us[r.rid] = (time.perf_counter() - ta) * 1e6
                    if pending_wait is not None:
                        wait_events.append((r.rid, pending_wait))
                        preempt_rids.append((now, r.rid))
                        pending_wait = None
                r.pages = need
                caches[r.rid] = m.alloc()
                toks = torch.randint(0, m.s.vocab, (r.prompt,), device=m.device)
                t_it = now_us()
                log.add(t_it, "prefill_start", **{"class": "online"}, request_id=r.rid, gpu=0, tokens=r.prompt)
                m.prefill(toks, caches[r.rid])
                lens[r.rid] = r.prompt
                self.online_stream.synchronize()  # never a device-wide sync: a gated launch may be queued
                t_pe = now_us()
                log.add(t_pe, "prefill_end", **{"class": "online"}, request_id=r.rid, gpu=0)
                self.res.prefill_us.append(t_pe - t_it)
                decoding.append(r)
                continue
            # one decode iteration over the batch
            need_by = []
            for r in decoding:
                tok_after = r.prompt + len(r.emits) + 1
                need_by.append(max(0, -(-tok_after // self.page_tokens) - r.pages))
            if self.colocated and sum(need_by):
                ta = time.perf_counter()
                self._acquire_online_pages(sum(need_by), now)
                dt = (time.perf_counter() - ta) * 1e6
                for r in decoding:  # the whole batch waits for the charge
                    self.res.mech_tpot_us[r.rid] = self.res.mech_tpot_us.get(r.rid, 0.0) + dt
            for r, nb in zip(decoding, need_by):
                r.pages += nb
            toks = torch.randint(0, m.s.vocab, (len(decoding),), device=m.device)
            t_it = now_us()
            m.decode(toks, [caches[r.rid] for r in decoding], [lens[r.rid] for r in decoding])
            self.online_stream.synchronize()  # never a device-wide sync: a gated launch may be queued
            t_emit = now_us()
            self.res.decode_iter_us.append(t_emit - t_it)
            done = []
            for r in decoding:
                lens[r.rid] += 1
                r.emits.append(t_emit)
                if len(r.emits) == 1:
                    r.first_us = t_emit
                    log.add(t_emit, "first_token", **{"class": "online"}, request_id=r.rid, gpu=0)
                if len(r.emits) == r.output:
                    done.append(r)
            for r in done:
                decoding.remove(r)
                m.free(caches.pop(r.rid))
                if self.colocated:
                    self.pool.online_free_pages(r.pages)
                if r.output > 1:
                    self.res.tpot_us[r.rid] = (r.emits[-1] - r.emits[0]) / (r.output - 1)
                self.res.ttft_us[r.rid] = r.first_us - r.arrival_us
                log.add(t_emit, "done", **{"class": "online"}, request_id=r.rid, gpu=0, tokens=len(r.emits),
                        first_token_us=r.emits[0], last_token_us=r.emits[-1], digest="0x0000000000000000")
        self.online_stream.synchronize()  # never a device-wide sync: a gated launch may be queued
        self.res.wall_s = time.perf_counter() - t0
        if gc_was:
            gc.enable()
        if busy:
            log.add(now_us(), "busy", gpu=0, **{"class": "online"}, start_us=busy_since, end_us=now_us())
        for (t_adm, _), (rid, (e0, e1)) in zip(preempt_rids, wait_events):
            self.res.quiesce_wait_us.append(e0.elapsed_time(e1) * 1e3)
            log.add(t_adm, "preempt_wait", gpu=0, request_id=rid, delay_us=int(round(self.res.quiesce_wait_us[-1])))
            self.res.mech_ttft_us[rid] = self.res.mech_ttft_us.get(rid, 0.0) + self.res.quiesce_wait_us[-1]
        if self.colocated:
            gen = self.channel.disables_issued() + 1000
            self.gate.raise_(gen)
            self.gate.wait_quiesced(gen)
            # not a device-wide sync here: an offline launch already queued behind "gate open"
            # would wait for the release below forever
            torch.cuda.ExternalStream(self.gate.stream).synchronize()
            self.res.offline_tiles = self._harvest + self.gate.read().tiles_done
            self.res.offline_bytes = self.res.offline_tiles * self.tile_bytes
            if self.gemm_gate is not None:
                _, _, _, m, n, k, tiles = self.gemm_seq[self._gemm_idx]
                part = self.gemm_gate.read().tiles_done
                self.res.offline_gemm_tiles = part
                self.res.offline_gemm_flop = self._gemm_flop + part * 2.0 * m * n * k / tiles
                self.res.offline_gemms_done = self._gemm_done + part / tiles
            self.gate.release(gen)
            torch.cuda.synchronize()
        return self.res


def paired_increase(base: Dict[int, float], other: Dict[int, float]):
    """metrics.cpp:49-65: mean and max of per-request % increases over paired requests."""
    pcts = [(other[i] - b) / b * 100.0 for i, b in sorted(base.items()) if i in other and b > 0]
    if not pcts:
        return {"mean_pct": None, "max_pct": None, "pairs": 0}
    return {"mean_pct": sum(pcts) / len(pcts), "max_pct": max(pcts), "pairs": len(pcts)}


def offline_population(seed: int, n: int, page_tokens: int = 16):
    """Qwen2-7B offline requests: prompt 2000-4000, output 100-200."""
    rng = random.Random(seed)
    out = []
    for r in range(n):
        inp, outp = rng.randint(2000, 4000), rng.randint(100, 200)
        out.append((r, math.ceil((inp + outp) / page_tokens), inp + rng.randint(0, outp)))
    return out


def warm_shapes(model: OnlineModel, trace: List[OnlineReq]):
    """Run every prefill length and a spread of decode shapes of the trace once, so neither
    measured run pays first-use costs (cuBLAS heuristics, allocator growth)."""
    slot = model.alloc()
    for r in trace:
        model.prefill(torch.randint(0, model.s.vocab, (r.prompt,), device=model.device), slot)
    lens = [r.prompt for r in trace[:4]]
    for b in range(1, min(4, len(trace)) + 1):
        for extra in range(0, 16, 4):
            model.decode(torch.zeros(b, dtype=torch.long, device=model.device), [slot] * b,
                         [n + extra for n in lens[:b]])
    model.free(slot)
    torch.cuda.synchronize()


class _Clocks:
    """nvidia-smi SM clock / power samples (500 ms) over one run -- evidence for clock effects of
    the offline tenant (a tensor-heavy tenant in the gaps can push the GPU into its power cap)."""

    def __init__(self, device):
        self.device, self.rows, self.proc = device, [], None

    def __enter__(self):
        import subprocess
        import threading

        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), "--query-gpu=clocks.sm,power.draw",
                 "--format=csv,noheader,nounits", "-lms", "500"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            threading.Thread(target=self._read, daemon=True).start()
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            try:
                self.rows.append(tuple(float(x) for x in line.split(",")))
            except ValueError:
                pass

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(2)
            except Exception:
                self.proc.kill()

    def summary(self):
        if not self.rows:
            return None
        sm = sorted(r[0] for r in self.rows)
        pw = sorted(r[1] for r in self.rows)
        return {"sm_mhz_median": sm[len(sm) // 2], "sm_mhz_min": sm[0], "power_w_median": pw[len(pw) // 2],
                "power_w_max": pw[-1], "samples": len(sm)}


def _avg_runs(dicts):
    """Per-request mean over runs (requests present in every run)."""
    keys = set(dicts[0])
    for d in dicts[1:]:
        keys &= set(d)
    return {k: sum(d[k] for d in dicts) / len(dicts) for k in sorted(keys)}


def _med_runs(dicts):
    """Per-request median over runs (requests present in every run).  A wall-clock loop admits
    an arrival at the first iteration boundary after it, so a few microseconds of jitter can move
    a 45 ms prefill between two decode tokens of the batch and shift that request's TPOT by
    several ms in one run; the median over runs discards such a flip, the mean keeps 1/n of it."""
    keys = set(dicts[0])
    for d in dicts[1:]:
        keys &= set(d)
    out = {}
    for k in sorted(keys):
        v = sorted(d[k] for d in dicts)
        n = len(v)
        out[k] = v[n // 2] if n % 2 else 0.5 * (v[n // 2 - 1] + v[n // 2])
    return out


def measure_deltas(horizon=24.0, base=0.3, spike=6.0, period=8.0, width=1.0, handles=64, seed=2604,
                   output=(8, 12), prompt=(2500, 3500), layers=32, device=0, offline_ctas=0, repeats=1,
                   offline_gemm=None, offline_gemm_ctas: int = 0, replay: bool = True,
                   log_dir: Optional[str] = None):
    """Paired standalone vs colocated run of one online trace (default: the pair_06 shape --
    spike base 0.3/s, 6/s for 1 s every 8 s, prompt 2500-3500, output 8-12 -- so the online
    lane goes idle and the offline tenant harvests the gaps).  Returns the reference's paired
    TTFT/TPOT increases (metrics.cpp:49-65) plus harvest statistics.

    Runs are interleaved A B A B ... A (`repeats` colocated runs between repeats+1 standalone
    ones): each request's latency is averaged over its standalone runs and over its colocated
    runs before pairing, which cancels clock/thermal drift and shrinks the batching-order jitter
    of a real-time loop by sqrt(repeats).  The A/A noise floor pairs the even standalone runs
    against the odd ones (the same statistic with no mechanism in it).

    log_dir: every run's events.jsonl in the reference schema (solo<i>.jsonl, colo<i>.jsonl), from
    which the reference's own metrics code recomputes the paired deltas (tests/test_realtime_logs)."""
    dev = torch.device("cuda", device)
    model = OnlineModel(ModelShape(layers=layers), dev)
    trace = spike_trace(seed, horizon, base, spike, period, width, prompt=prompt, output=output)
    warm_shapes(model, trace)
    # replay=True: an untimed standalone run records the serving loop's action sequence, and
    # every measured run (standalone and colocated) replays it -- the pairing then compares the
    # same work, action by action (see Colocation.run)
    plan = None
    if replay:  # the second of two live runs (the first one still pays first-use costs)
        for _ in range(2):
            plan = Colocation(model, None, None).run(trace, horizon_s=horizon + 30, admit_margin_us=6000).plan
    solos, colos = [], []
    clocks = {"standalone": [], "colocated": []}
    for i in range(repeats):
        with _Clocks(device) as ck:
            solos.append(Colocation(model, None, None).run(trace, horizon_s=horizon + 30, plan=plan))
        clocks["standalone"].append(ck.summary())
        pool = A.DevicePool(handles, 64, 16, device=device, slot_bytes=2 << 20, page_bytes=917504,
                            max_requests=4096, max_pages_per_request=1024)
        gate = A.Gate(device)
        colo_rt = Colocation(model, pool, gate, offline_ctas=offline_ctas, offline_gemm=offline_gemm,
                             offline_gemm_ctas=offline_gemm_ctas)
        with _Clocks(device) as ck:
            colos.append(colo_rt.run(trace, offline_population(seed, 4 * handles), horizon_s=horizon + 30, plan=plan))
        clocks["colocated"].append(ck.summary())
        del pool, gate, colo_rt
        import gc

        gc.collect()  # the channel's ctypes hooks close over the runtime: break the cycle now
        torch.cuda.synchronize()
        torch.cuda.empty_cache()
    solos.append(Colocation(model, None, None).run(trace, horizon_s=horizon + 30, plan=plan))
    if log_dir:
        import os

        os.makedirs(log_dir, exist_ok=True)
        for i, r in enumerate(solos):
            r.log.write_jsonl(os.path.join(log_dir, f"solo{i}.jsonl"))
        for i, r in enumerate(colos):
            r.log.write_jsonl(os.path.join(log_dir, f"colo{i}.jsonl"))

    base_ttft = _med_runs([s.ttft_us for s in solos])
    base_tpot = _med_runs([s.tpot_us for s in solos])
    colo_ttft = _med_runs([c.ttft_us for c in colos])
    colo_tpot = _med_runs([c.tpot_us for c in colos])
    ttft = paired_increase(base_ttft, colo_ttft)
    tpot = paired_increase(base_tpot, colo_tpot)
    # the same pairing on per-request run means (sensitive to single-run batching flips)
    ttft_mean = paired_increase(_avg_runs([s.ttft_us for s in solos]), _avg_runs([c.ttft_us for c in colos]))
    tpot_mean = paired_increase(_avg_runs([s.tpot_us for s in solos]), _avg_runs([c.tpot_us for c in colos]))
    even, odd = solos[0::2], solos[1::2]
    aa_ttft = paired_increase(_med_runs([s.ttft_us for s in even]), _med_runs([s.ttft_us for s in odd]))
    aa_tpot = paired_increase(_med_runs([s.tpot_us for s in even]), _med_runs([s.tpot_us for s in odd]))
    mech_ttft = _avg_runs([c.mech_ttft_us for c in colos]) if colos else {}
    mech_tpot = _avg_runs([c.mech_tpot_us for c in colos]) if colos else {}
    colo = colos[-1]

    def mean(d):
        return sum(d.values()) / max(1, len(d))

    out = {
        "trace": {"horizon_s": horizon, "online_requests": len(trace), "base_rate": base, "spike_rate": spike,
                  "period_s": period, "width_s": width, "prompt": list(prompt), "output": list(output),
                  "model": f"Llama-3-8B-shaped, {layers} layers, random init bf16"},
        "schedule": ("replayed: every run places each prefill at the decode count recorded by an untimed "
                     f"standalone run ({len(plan)} prefills)") if plan else "live (each run schedules on its own)",
        # prefills a run executed at another decode count than the plan's (arrival later than the
        # recording's boundary); 0 everywhere = both arms ran exactly the same schedule
        "plan_deviations": ({"standalone": [_deviations(plan, r.plan) for r in solos],
                             "colocated": [_deviations(plan, r.plan) for r in colos]} if plan else None),
        "design": f"interleaved A/B x{repeats} + A: per-request median over {repeats} colocated runs paired "
                  f"against the per-request median over {repeats + 1} standalone runs (reference pairing, "
                  f"metrics.cpp:49-65, on those per-request values)",
        "repeats": repeats,
        "ttft_delta_pct": ttft["mean_pct"], "ttft_delta_max_pct": ttft["max_pct"],
        "tpot_delta_pct": tpot["mean_pct"], "tpot_delta_max_pct": tpot["max_pct"], "pairs": ttft["pairs"],
        "ttft_delta_runmean_pct": ttft_mean["mean_pct"], "tpot_delta_runmean_pct": tpot_mean["mean_pct"],
        "aa_noise_ttft_pct": aa_ttft["mean_pct"], "aa_noise_tpot_pct": aa_tpot["mean_pct"],
        "per_run_ttft_delta_pct": [paired_increase(base_ttft, c.ttft_us)["mean_pct"] for c in colos],
        "per_run_tpot_delta_pct": [paired_increase(base_tpot, c.tpot_us)["mean_pct"] for c in colos],
        # the reference DES's view of the same quantity: only the delays the mechanism puts on
        # the critical path (preempt wait + page acquisition/reclaim), per request, over the
        # standalone latency -- free of the run-to-run jitter of the end-to-end statistic
        "ttft_attributable_pct": _attributable(mech_ttft, base_ttft, 1),
        "tpot_attributable_pct": _attributable(mech_tpot, base_tpot,
                                               {r.rid: max(1, r.output - 1) for r in trace}),
        "preempt_wait_us": {"p50": _median([w for c in colos for w in c.quiesce_wait_us]),
                            "max": max((w for c in colos for w in c.quiesce_wait_us), default=None)},
        "ttft_ms": {"standalone": mean(base_ttft) / 1e3, "colocated": mean(colo_ttft) / 1e3},
        "tpot_ms": {"standalone": mean(base_tpot) / 1e3, "colocated": mean(colo_tpot) / 1e3},
        "disables": colo.disables, "disables_per_request": colo.disables / max(1, len(trace)),
        "reclaims": colo.reclaims, "reclaimed_handles": colo.reclaimed_handles,
        "offline_ctas": offline_ctas or "default",
        "offline_gbs_harvested": colo.offline_bytes / colo.wall_s / 1e9,
        "offline_gemm": ({"shape": list(offline_gemm), "tflops_harvested": colo.offline_gemm_flop / colo.wall_s / 1e12,
                          "gemms_completed": colo.offline_gemms_done, "ctas": offline_gemm_ctas or "one per SM",
                          **({"model_tokens_per_s": colo.offline_gemms_done / (4 * 28) * offline_gemm[1] / colo.wall_s}
                             if offline_gemm[0] == "qwen2-7b" else {})}
                         if offline_gemm else None),
        "prefill_ms_median": {"standalone": _median([x for s in solos for x in s.prefill_us]) / 1e3,
                              "colocated": _median([x for c in colos for x in c.prefill_us]) / 1e3},
        "decode_iter_ms_median": {
            "standalone": _median([x for s in solos for x in s.decode_iter_us]) / 1e3,
            "colocated": _median([x for c in colos for x in c.decode_iter_us]) / 1e3},
        "wall_s": {"standalone": solos[0].wall_s, "colocated": colo.wall_s},
        "clocks_per_run": clocks,
    }
    import gc

    del model, colos, solos
    gc.collect()
    torch.cuda.synchronize()
    torch.cuda.empty_cache()
    return out


def _deviations(plan, executed):
    want = {rid: k for rid, k in plan}
    return sum(1 for rid, k in executed if want.get(rid) != k)


def _attributable(mech, base, per):
    """Mean over requests of mechanism delay / standalone latency, in %."""
    pcts = []
    for rid, b in base.items():
        if b <= 0:
            continue
        d = mech.get(rid, 0.0) / (per[rid] if isinstance(per, dict) else per)
        pcts.append(d / b * 100.0)
    return sum(pcts) / len(pcts) if pcts else None


def _median(xs):
    xs = sorted(xs)
    return xs[len(xs) // 2] if xs else float("nan")
