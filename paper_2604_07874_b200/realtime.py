"""Real-time colocation on one B200: measured online TTFT/TPOT deltas and offline harvest
(BASELINE.json configs[1] (C2) and configs[2] (C3)).

A thin runtime around the product kernels that follows the reference simulator's engines
(sim.cpp:391-1082) in wall-clock time on the device:

* online: a random-init Llama-3-8B-shaped decoder in PyTorch (bf16, cuBLAS GEMMs, never
  gated).  Its KV cache lives IN THE POOL: one 2 MiB slot = one 16-token page of all 32 layers
  (SURVEY §8 geometry), placed in the slots of online-reserved handles.  Prefill writes layer by
  layer; decode attends straight from the slots (libonline.so paged decode attention) inside a
  CUDA graph per batch bucket.
* memory (sim.cpp:469-556, 885-1082): online pages are charged against the reservation (free
  handles first, then a reclaim op of k offline handles -- device Algorithm 1 + apply_reclaim),
  pressure growth at 90 % utilisation, and the MIAD control plane (release one handle per quiet
  interval T, T adjusted per window -- sim.cpp:1054-1082).  Every reclaim op gathers its
  invalidated pages to pinned host memory under the pool's rate bound, and the online tenant
  writes a reclaimed slot only once the copy waves under the bytes it writes have been read out
  (landed tickets, cuStreamWaitValue64 per layer): shortfall -> first online write is one wave,
  not the whole copy.
* offline: the gated tile-looped kernels (a KV decode pass over the offline pages + a Qwen2-7B
  projection chain as gated tcgen05 GEMMs).  Their harvested work is converted to token-forwards
  and drives a request-level offline engine: admission into the pool (offline_reserve), FIFO
  prefill then batched decode, completion (offline_release), and the invalidation callback
  (sim.cpp:994-1050): an evicted request loses its progress and resumes by recomputing
  input + generated tokens (requests.hpp:68-69).
* lane edges drive the host ChannelController bound to the HBM gate (raise on the online stream,
  then the online stream waits for every offline CTA to retire).

Policies on the same kernels (policies.cpp:5-14): valve (channel + MIAD + Algorithm 1), valve-fifo
(FIFO selection, reclaim.cpp:69-83), channel+static (calibrated offline budget, FIFO kills,
sim.cpp:578-594), channel+prism (offline keeps its memory; online stalls), standalone.  The
reference's build_report / ttft_increase / normalized_offline_throughput (metrics.cpp:85-247)
recompute the reported numbers from the events.jsonl every run writes.
"""
from __future__ import annotations

import ctypes as C
import heapq
import math
import os
import random
import time
from collections import deque
from dataclasses import dataclass, field
from typing import Dict, List, Optional

import torch
import torch.nn.functional as F

from . import api as A

LIBONLINE = os.path.join(os.path.dirname(os.path.abspath(__file__)), "libonline.so")
PAGE_TOKENS = 16
LAYER_BYTES = 65536  # one layer of one 16-token page: K + V, 8 kv heads x 16 x 128 bf16 each
QWEN_PAGE = 917_504  # Qwen2-7B 16-token KV page (28 x 2 x 4 x 128 x 2 B x 16)
QWEN_FLOP_PER_TOKEN = 2.0 * 28 * 3584 * (4608 + 3584 + 37888 + 18944)  # projection chain


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

    @property
    def page_bytes(self) -> int:  # one 16-token page of every layer = one pool slot
        return self.layers * LAYER_BYTES


class OnlineModel:
    """Random-init (N(0, 0.02), bf16) decoder whose KV pages are pool slots.  Slot layout:
    [layer][K, V][kv head][16 tokens][128] bf16 -- layer l occupies slot bytes
    [l * 64 KiB, (l + 1) * 64 KiB), so a prefill writing layer l only needs the reclaim copy
    waves under those bytes to have been read out."""

    BUCKETS = (1, 2, 4, 8, 12, 16, 24, 32)
    MAX_PAGES = 288  # 4,608 tokens per request

    def __init__(self, shape: ModelShape, device, seed: int = 0):
        g = torch.Generator(device=device).manual_seed(seed)
        s = self.s = shape
        assert s.kv_heads * PAGE_TOKENS * s.head_dim * 2 * 2 == LAYER_BYTES and s.heads % s.kv_heads == 0

        def w(*shape_):
            return (torch.randn(*shape_, generator=g, device=device, dtype=torch.float32) * 0.02).to(torch.bfloat16)

        qkv = (s.heads + 2 * s.kv_heads) * s.head_dim
        self.layers = [dict(wqkv=w(s.d, qkv), wo=w(s.heads * s.head_dim, s.d), w13=w(s.d, 2 * s.ffn),
                            w2=w(s.ffn, s.d)) for _ in range(s.layers)]
        self.emb = w(s.vocab, s.d)
        self.lm = w(s.d, s.vocab)
        self.device = device
        self.lib = C.CDLL(LIBONLINE)
        self.lib.online_clock_probe.restype = C.c_int
        self.lib.online_clock_probe.argtypes = [C.c_void_p, C.c_int, C.c_void_p]
        self.clock_mhz = torch.zeros(1 << 16, dtype=torch.float32, device=device)  # per decode step
        self.clock_n = 0
        self.lib.online_paged_decode_attn.restype = C.c_int
        self.lib.online_paged_decode_attn.argtypes = [
            C.c_void_p, C.c_void_p, C.c_int64, C.c_int64, C.c_int64, C.c_int64, C.c_void_p, C.c_int, C.c_void_p,
            C.c_int, C.c_int, C.c_int, C.c_float, C.c_int, C.c_int, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]
        self.pps = 16
        self.splits = -(-self.MAX_PAGES // self.pps)
        B = self.BUCKETS[-1]
        dev = device
        # static decode inputs (graph inputs): tokens, write slot, write offset, lengths, block tables
        self.s_tok = torch.zeros(B, dtype=torch.long, device=dev)
        self.s_pg = torch.zeros(B, dtype=torch.long, device=dev)
        self.s_off = torch.zeros(B, dtype=torch.long, device=dev)
        self.s_len = torch.ones(B, dtype=torch.int32, device=dev)
        self.s_bt = torch.zeros(B, self.MAX_PAGES, dtype=torch.int32, device=dev)
        self.s_out = torch.zeros(B, dtype=torch.long, device=dev)
        self.part_acc = torch.empty(B * s.heads * self.splits * s.head_dim, dtype=torch.float32, device=dev)
        self.part_ml = torch.empty(B * s.heads * self.splits * 2, dtype=torch.float32, device=dev)
        self.attn_out = torch.empty(B, s.heads, s.head_dim, dtype=torch.bfloat16, device=dev)
        self.h_in = torch.empty(8 * B * (4 + self.MAX_PAGES), dtype=torch.int64).pin_memory()  # 8 chunks
        self.graphs: Dict[int, torch.cuda.CUDAGraph] = {}
        self.mempool = None
        self.P = None
        self.gpu_events = None  # list: (start, end) CUDA events of every decode graph replay

    def bind(self, pool: A.DevicePool):
        """Point the model at the pool's page store (graphs are captured against it)."""
        v = pool.view()
        assert v.slot_bytes == self.s.page_bytes, (v.slot_bytes, self.s.page_bytes)
        n = pool.total_handles() * pool.handle_size_pages()

        class _Arr:
            __cuda_array_interface__ = {"shape": (n * v.slot_bytes // 256, 128), "typestr": "<f2",
                                        "data": (v.pages, False), "version": 3}

        rows = torch.as_tensor(_Arr(), device=self.device)  # fp16 view of the bytes
        assert rows.data_ptr() == v.pages
        if self.P is not None and self.P.data_ptr() != v.pages:
            self.graphs.clear()
        self.P = rows.view(torch.bfloat16)  # [slots * layers * 2 * 8 * 16, 128]: one row = one token of one kv head
        self.u8 = rows.view(torch.uint8).view(n, v.slot_bytes)
        self.pages_ptr = v.pages
        self.slot_rows = self.s.layers * 2 * self.s.kv_heads * PAGE_TOKENS  # 128-dim rows per slot

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

    def _rows(self, slot, off, li, kv):
        """Row index (of 128 bf16) of token `off` of `slot`, layer li, K (0) / V (1), per kv head."""
        s = self.s
        g = torch.arange(s.kv_heads, device=self.device) * PAGE_TOKENS
        base = slot * self.slot_rows + (li * 2 + kv) * s.kv_heads * PAGE_TOKENS + off
        return base[:, None] + g[None, :]

    @torch.no_grad()
    def prefill(self, tokens, pages: List[int], wait_layer=None):
        """Prefill writing K/V layer by layer into `pages` (slots); wait_layer(li) is called
        right before layer li's KV write (landed tickets of reclaimed slots)."""
        s = self.s
        T = tokens.shape[0]
        rep = s.heads // s.kv_heads
        x = self.emb[tokens]
        t = torch.arange(T, device=self.device)
        slot = torch.tensor(pages, device=self.device, dtype=torch.long)[t // PAGE_TOKENS]
        off = t % PAGE_TOKENS
        for li, L in enumerate(self.layers):
            q, k, v = self._qkv(L, x)
            if wait_layer is not None:
                wait_layer(li)
            self.P.index_copy_(0, self._rows(slot, off, li, 0).flatten(), k.reshape(T * s.kv_heads, s.head_dim))
            self.P.index_copy_(0, self._rows(slot, off, li, 1).flatten(), v.reshape(T * s.kv_heads, s.head_dim))
            kh = k.view(T, s.kv_heads, s.head_dim).transpose(0, 1)
            vh = v.view(T, s.kv_heads, s.head_dim).transpose(0, 1)
            qh = q.view(T, s.heads, s.head_dim).transpose(0, 1).unsqueeze(0)
            o = F.scaled_dot_product_attention(qh, kh.repeat_interleave(rep, 0).unsqueeze(0),
                                               vh.repeat_interleave(rep, 0).unsqueeze(0), is_causal=True)
            x = self._mlp(L, x, o[0].transpose(0, 1).reshape(T, -1))
        return (self._rms(x[-1:]) @ self.lm).argmax(-1)

    def _decode_body(self, B):
        s = self.s
        st = torch.cuda.current_stream().cuda_stream
        x = self.emb[self.s_tok[:B]]
        pg, off = self.s_pg[:B], self.s_off[:B]
        scale = 1.0 / math.sqrt(s.head_dim)
        for li, L in enumerate(self.layers):
            q, k, v = self._qkv(L, x)
            self.P.index_copy_(0, self._rows(pg, off, li, 0).flatten(), k.reshape(B * s.kv_heads, s.head_dim))
            self.P.index_copy_(0, self._rows(pg, off, li, 1).flatten(), v.reshape(B * s.kv_heads, s.head_dim))
            qc = q.contiguous()
            rc = self.lib.online_paged_decode_attn(
                qc.data_ptr(), self.pages_ptr, s.page_bytes, li * LAYER_BYTES, LAYER_BYTES // 2,
                PAGE_TOKENS * s.head_dim * 2, self.s_bt.data_ptr(), self.MAX_PAGES, self.s_len.data_ptr(), B,
                s.heads, s.kv_heads, scale, self.splits, self.pps, self.part_acc.data_ptr(), self.part_ml.data_ptr(),
                self.attn_out.data_ptr(), C.c_void_p(st))
            assert rc == 0, f"paged decode attention failed ({rc})"
            x = self._mlp(L, x, self.attn_out[:B].reshape(B, -1))
        self.s_out[:B] = (self._rms(x) @ self.lm).argmax(-1)

    def _graph(self, B):
        g = self.graphs.get(B)
        if g is None:
            side = torch.cuda.Stream(device=self.device)
            side.wait_stream(torch.cuda.current_stream())
            with torch.cuda.stream(side), torch.no_grad():
                self._decode_body(B)  # warm-up (cuBLAS heuristics, allocator)
            torch.cuda.current_stream().wait_stream(side)
            torch.cuda.synchronize()
            if self.mempool is None:
                self.mempool = torch.cuda.graph_pool_handle()
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, pool=self.mempool), torch.no_grad():
                self._decode_body(B)
            self.graphs[B] = g
        return g

    @torch.no_grad()
    def decode(self, tokens: List[int], write_slot: List[int], pos: List[int], tables: List[List[int]],
               scratch: int):
        """One decode iteration: request b appends token tokens[b] at position pos[b] (written to
        slot write_slot[b]) and attends over its first pos[b] + 1 tokens through tables[b]."""
        n = len(tokens)
        out = []
        mp, bmax = self.MAX_PAGES, self.BUCKETS[-1]
        for ci, c0 in enumerate(range(0, n, bmax)):
            idx = list(range(c0, min(n, c0 + bmax)))
            B = next(b for b in self.BUCKETS if b >= len(idx))
            # one pinned staging region per chunk: the async H2D of chunk i may still be reading
            hv = self.h_in[ci * bmax * (4 + mp):][: B * (4 + mp)].view(B, 4 + mp)
            hv.zero_()
            for j in range(B):
                if j < len(idx):
                    i = idx[j]
                    t = tables[i]
                    hv[j, 0], hv[j, 1], hv[j, 2], hv[j, 3] = tokens[i], write_slot[i], pos[i] % PAGE_TOKENS, pos[i] + 1
                    hv[j, 4:4 + len(t)] = torch.as_tensor(t, dtype=torch.int64)
                else:  # padding row: one token in the scratch slot
                    hv[j, 1], hv[j, 3], hv[j, 4] = scratch, 1, scratch
            d = hv.to(self.device, non_blocking=True)
            self.s_tok[:B] = d[:, 0]
            self.s_pg[:B] = d[:, 1]
            self.s_off[:B] = d[:, 2]
            self.s_len[:B] = d[:, 3].to(torch.int32)
            self.s_bt[:B] = d[:, 4:].to(torch.int32)
            g = self._graph(B)
            if self.gpu_events is not None and self.clock_n < self.clock_mhz.numel():
                # SM clock at the start of the step (a 4 us probe kernel on the online stream)
                self.lib.online_clock_probe(C.c_void_p(self.clock_mhz.data_ptr()), self.clock_n,
                                            C.c_void_p(torch.cuda.current_stream().cuda_stream))
                self.clock_n += 1
            if self.gpu_events is not None:
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                g.replay()
                e1.record()
                self.gpu_events.append((e0, e1))
            else:
                g.replay()
            out.append(self.s_out[: len(idx)].clone())
        return torch.cat(out)


# ------------------------------------------------------------------------------ trace

@dataclass
class OnlineReq:
    rid: int
    arrival_us: int
    prompt: int
    output: int
    first_us: int = -1
    emits: List[int] = field(default_factory=list)
    pages: List[int] = field(default_factory=list)  # slots holding its KV, in block order


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


def offline_population(seed: int, n: int, prompt=(2000, 4000), output=(100, 200)):
    """Qwen2-7B offline backlog: (id, input, output) -- SURVEY §8d C2 (a Poisson stream at 280/s
    is a standing backlog for one GPU)."""
    rng = random.Random(seed)
    return [(r, rng.randint(*prompt), rng.randint(*output)) for r in range(n)]


# ------------------------------------------------------------------------- event log

class EventLog:
    """The reference's events.jsonl schema (log.hpp:13-59, writer log.cpp:69-217): the same
    kinds, field names and key order, so the reference's own build_report / ttft_increase /
    tpot_increase / normalized_offline_throughput (metrics.cpp:85-247) recompute the reported
    numbers from these logs (tests pin that)."""

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

    def count(self, kind: str, **match) -> int:
        return sum(1 for (_, _, k, f) in self.recs if k == kind and all(f.get(a) == b for a, b in match.items()))

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


# ------------------------------------------------------------- online pages in pool slots

class OnlinePages:
    """Physical home of the online tenant's pages: the slots of the online-reserved handles.
    The reference charges online pages as an aggregate (memory.hpp:97, sim.cpp:513-526); a real
    tenant needs the slots, so this mirrors which handles are online and which of their slots
    hold KV.  Slots whose old bytes a reclaim copy has not yet read out carry that copy's ticket
    (valve_pool_copy_ticket): a write waits for the waves under the bytes it writes.

    Free slots live in two places so allocation never scans them all: `clean` (no pending
    ticket; a max-heap, highest slot first -- releases take the lowest handle ids,
    memory.cpp:37-51) and `pending` (ticketed, usually one op's slots).  `free` is the set of
    both; heap entries of slots that left `free` are dropped lazily."""

    def __init__(self, pool: A.DevicePool, layer_bytes: int = LAYER_BYTES):
        self.pool = pool
        self.S = pool.handle_size_pages()
        self.layer_bytes = layer_bytes
        self.handles: set = set()
        self.free: set = set()
        self.clean: list = []               # heap of -slot
        self.pending: set = set()
        self.used: Dict[int, int] = {}      # slot -> request id
        self.ticket: Dict[int, tuple] = {}  # slot -> (wave_base, n_waves, wave_bytes)
        self.landed = 0

    def _free_slot(self, s):
        self.free.add(s)
        if s in self.ticket:
            self.pending.add(s)
        else:
            heapq.heappush(self.clean, -s)

    def refresh_landed(self):
        self.landed = self.pool.landed()[0]
        done = [s for s, (b, n, _) in self.ticket.items() if b + n <= self.landed]
        for s in done:
            del self.ticket[s]
            if s in self.pending:
                self.pending.discard(s)
                heapq.heappush(self.clean, -s)

    def set_tickets(self, slots, ticket):
        for s in slots:
            self.ticket[s] = ticket
            if s in self.free:
                self.pending.add(s)  # its clean heap entry is skipped on pop

    def sync_handles(self):
        ids = set(self.pool.online_handle_ids())
        for h in ids - self.handles:
            for s in range(h * self.S, (h + 1) * self.S):
                self._free_slot(s)
        for h in self.handles - ids:
            for s in range(h * self.S, (h + 1) * self.S):
                assert s not in self.used, f"online handle {h} released with live KV in slot {s}"
                self.free.discard(s)
                self.pending.discard(s)
        self.handles = ids

    def _pop_clean(self, exclude_handles=()):
        """Highest clean free slot (not in exclude_handles), or None."""
        skipped = []
        got = None
        while self.clean:
            s = -heapq.heappop(self.clean)
            if s not in self.free or s in self.ticket:
                continue  # stale entry (left the free set / got a ticket since)
            if s // self.S in exclude_handles:
                skipped.append(s)
                continue
            got = s
            self.free.discard(s)  # taken now: a duplicate heap entry of s is stale from here on
            break
        for s in skipped:
            heapq.heappush(self.clean, -s)
        return got

    def alloc(self, n: int, rid: int, exclude_handles=()) -> List[int]:
        """n free slots: clean ones first (highest first), then pending by ticket."""
        if n > len(self.free):
            raise RuntimeError(f"online slots: need {n}, have {len(self.free)}")
        if self.ticket:
            self.refresh_landed()
        pick = []
        while len(pick) < n:
            s = self._pop_clean(exclude_handles)
            if s is None:
                break
            pick.append(s)
        if len(pick) < n:
            rest = sorted((s for s in self.pending if s // self.S not in exclude_handles),
                          key=lambda s: (self.ticket[s][0], -s))[: n - len(pick)]
            if len(rest) < n - len(pick):
                for s in pick:  # not enough: give back
                    self._free_slot(s)
                raise RuntimeError(f"online slots: need {n}, have {len(pick) + len(rest)} outside {exclude_handles}")
            pick += rest
        for s in pick:
            self.free.discard(s)
            self.pending.discard(s)
            self.used[s] = rid
        return pick

    def clean_count_outside(self, handles) -> int:
        """Free slots without a pending ticket outside `handles` (O(|handles| * S))."""
        inside = sum(1 for h in handles for s in range(h * self.S, (h + 1) * self.S)
                     if s in self.free and s not in self.pending)
        return len(self.free) - len(self.pending) - inside

    def release(self, slots):
        for s in slots:
            del self.used[s]
            self._free_slot(s)

    def layer_target(self, slots, li: int) -> int:
        """Landed count a write of layer li (slot bytes [li, li+1) * layer_bytes) into `slots`
        needs: the waves covering [0, (li+1) * layer_bytes) of each pending slot (0 = none)."""
        tgt = 0
        hi = (li + 1) * self.layer_bytes
        for s in slots:
            t = self.ticket.get(s)
            if t is not None:
                base, n, wb = t
                tgt = max(tgt, base + min(n, -(-hi // wb)))
        return tgt if tgt > self.landed else 0

    def full_target(self, slots) -> int:
        tgt = 0
        for s in slots:
            t = self.ticket.get(s)
            if t is not None:
                tgt = max(tgt, t[0] + t[1])
        return tgt if tgt > self.landed else 0


# ------------------------------------------------------------------------ offline engine

@dataclass
class OffReq:
    rid: int
    input: int
    output: int
    generated: int = 0
    state: str = "waiting"   # waiting / prefill / decode / evicted / done / killed
    prefill_left: int = 0    # token-forwards of the (re)prefill still to run
    invested: int = 0        # forwards spent since the last (re)admission (lost on eviction)
    evictions: int = 0

    def recompute_cost(self) -> int:  # requests.hpp:68-69
        return self.input + self.generated


class OfflineEngine:
    """Request-level offline engine driven by the harvested GPU work (sim.cpp:730-858): FIFO
    admission into the pool (resumed requests first), prefill of recompute_cost() forwards in
    chunks interleaved with batched decode steps (one forward per request per token,
    max_offline_batch 256); completion frees the pages.  Evictions (the invalidation callback, sim.cpp:994-1050) drop the request's
    progress: it re-prefills input + generated tokens after re-admission."""

    def __init__(self, pool: A.DevicePool, backlog, log: EventLog, page_tokens=PAGE_TOKENS, max_batch=256,
                 chunk=2048):
        self.pool, self.log = pool, log
        self.chunk = chunk
        self.page_tokens = page_tokens
        self.max_batch = max_batch
        self.reqs = {rid: OffReq(rid, i, o) for rid, i, o in backlog}
        self.waiting = deque(rid for rid, _, _ in backlog)
        self.running: Dict[int, OffReq] = {}  # admitted, in prefill or decode
        self.resume: deque = deque()
        self.prefill_q: deque = deque()
        self.decoding: List[int] = []
        self.budget = -1      # static policy: max offline handles (-1 = unlimited)
        self.frozen = False   # static calibration: no admission
        self.carry = 0.0      # fractional forwards
        self.forwards = 0.0   # harvested
        self.lost = 0         # forwards thrown away by evictions / kills
        self.tokens_done = 0  # generated tokens of completed requests (metrics.cpp offline_tokens)
        self.completed = 0
        self.mark = lambda name: None  # phase stamps for the serving loop's slow-iteration log

    def pages(self, r: OffReq) -> int:
        return -(-(r.input + r.output) // self.page_tokens)

    def live(self):
        return list(self.running.values())

    def admit(self, now: int, warm: bool = False, rng: Optional[random.Random] = None) -> int:
        """Admission into the pool while it has room (sim.cpp:730-753), resumed requests first.
        warm=True (run start): the tenant is in steady state -- each admitted request has already
        prefilled and generated a random part of its output, i.e. holds input + generated tokens of
        KV, exactly what an eviction throws away (requests.hpp:68-69)."""
        if self.frozen:
            return 0
        n = 0
        for q in (self.resume, self.waiting):
            while q:
                r = self.reqs[q[0]]
                if not self.pool.offline_reserve(r.rid, self.pages(r), now, self.budget):
                    return n
                q.popleft()
                if r.state == "waiting":
                    self.log.add(now, "arrival", **{"class": "offline"}, request_id=r.rid, gpu=0,
                                 prompt_tokens=r.input, output_tokens=r.output)
                self.running[r.rid] = r
                n += 1
                if warm:
                    r.generated = rng.randrange(r.output)
                    r.state, r.prefill_left, r.invested = "decode", 0, r.input + r.generated
                    self.decoding.append(r.rid)
                else:
                    r.state, r.prefill_left, r.invested = "prefill", r.recompute_cost(), 0
                    self.prefill_q.append(r.rid)
        return n

    def costs(self):
        return {r.rid: r.recompute_cost() for r in self.running.values()}

    def advance(self, forwards: float, now: int, horizon_us: int, budget_s: float = 1e-3):
        """Spend harvested token-forwards, iteration by iteration as a continuous-batching engine
        does: one decode step of the running batch (one forward per request), then a prefill
        chunk of up to `chunk` forwards of the FIFO head(s).  Returns whether pages were freed.
        At most `budget_s` of host time per call: forwards not spent yet stay in the carry and are
        spent by the next calls (the engine's bookkeeping must never hold the serving loop)."""
        self.forwards += forwards
        total = forwards + self.carry
        f = int(total)
        frac = total - f
        deadline = time.perf_counter() + budget_s
        freed = False
        while f > 0:
            if time.perf_counter() > deadline:
                break
            progressed = False
            batch = self.decoding[: self.max_batch]
            if batch and f >= len(batch):
                f -= len(batch)
                progressed = True
                for rid in batch:
                    r = self.reqs[rid]
                    r.generated += 1
                    r.invested += 1
                    if r.generated == r.output:
                        r.state = "done"
                        self.decoding.remove(rid)
                        del self.running[rid]
                        self.mark("advance:loop")
                        self.pool.offline_release(rid)
                        self.mark("advance:release")
                        freed = True
                        if now <= horizon_us:
                            self.tokens_done += r.generated
                            self.completed += 1
                            self.log.add(now, "done", **{"class": "offline"}, request_id=rid, gpu=0,
                                         tokens=r.generated, first_token_us=-1, last_token_us=-1,
                                         digest="0x0000000000000000")
            budget = min(f, self.chunk)
            while budget > 0 and self.prefill_q:
                r = self.reqs[self.prefill_q[0]]
                use = min(budget, r.prefill_left)
                r.prefill_left -= use
                r.invested += use
                budget -= use
                f -= use
                progressed = True
                if r.prefill_left == 0:
                    self.prefill_q.popleft()
                    r.state = "decode"
                    self.decoding.append(r.rid)
            if not progressed:
                break
        self.carry = frac + f  # unspent forwards (budget reached, or nothing to run)
        return freed

    def on_evicted(self, rids, now: int, kill: bool):
        for rid in rids:
            r = self.reqs[rid]
            self.running.pop(rid, None)
            self.lost += r.invested
            if r.rid in self.prefill_q:
                self.prefill_q.remove(r.rid)
            if r.rid in self.decoding:
                self.decoding.remove(r.rid)
            r.invested = 0
            if kill:
                r.state = "killed"
                self.log.add(now, "killed", request_id=rid, gpu=0, lost_tokens=r.recompute_cost())
            else:
                r.state = "evicted"
                r.evictions += 1
                self.log.add(now, "evicted", request_id=rid, gpu=0, recompute_tokens=r.recompute_cost())
                self.resume.append(rid)


# ------------------------------------------------------------------------- the runtime

POLICIES = ("standalone", "valve", "valve-fifo", "channel+static", "channel+prism")


@dataclass
class RunResult:
    policy: str
    ttft_us: Dict[int, float]
    tpot_us: Dict[int, float]
    wall_s: float = 0.0
    disables: int = 0
    reclaims: int = 0
    reclaimed_handles: int = 0
    releases: int = 0
    interval_changes: int = 0
    pressure: int = 0
    kills: int = 0
    evictions: int = 0
    stalls: int = 0
    copy_bytes: int = 0
    copy_gbs: List[float] = field(default_factory=list)
    offline_tokens_done: int = 0
    offline_completed: int = 0
    offline_forwards: float = 0.0
    offline_lost_forwards: int = 0
    offline_decode_bytes: float = 0.0
    quiesce_wait_us: List[float] = field(default_factory=list)
    shortfall_to_write_us: List[float] = field(default_factory=list)   # reclaim issued -> first layer write allowed
    shortfall_full_copy_us: List[float] = field(default_factory=list)  # reclaim issued -> whole copy out
    decision_us: List[float] = field(default_factory=list)
    op_phase_us: Dict[str, float] = field(default_factory=dict)
    decode_iter_us: List[float] = field(default_factory=list)
    prefill_us: List[float] = field(default_factory=list)
    step_gap_us: List[float] = field(default_factory=list)  # host time between back-to-back busy steps
    decode_gpu_us: List[float] = field(default_factory=list)  # device time of each decode graph replay
    decode_sm_mhz: List[float] = field(default_factory=list)  # SM clock at the start of each replay
    decode_t_us: List[int] = field(default_factory=list)  # loop time at the start of each decode step
    busy_starts: List[int] = field(default_factory=list)  # loop time of every busy edge
    slow_iterations: List[dict] = field(default_factory=list)  # loop iterations with > 3 ms host time
    deferred_releases: int = 0  # MIAD releases postponed: no copied-out slots to move the KV into
    log: EventLog = field(default_factory=EventLog)
    plan: list = field(default_factory=list)


@dataclass
class RtConfig:
    policy: str = "valve"
    page_tokens: int = PAGE_TOKENS
    max_gap_us: int = 300                 # G of the bundled scenarios (T_cool = 2G)
    resparams: Optional[A.ReservationParams] = None
    offline_page_bytes: int = QWEN_PAGE
    decode_ctas: int = 16                 # offline KV decode pass CTAs (-1: none)
    gemm_ctas: int = 64                   # offline projection-chain CTAs (0: one per SM)
    gemm_tokens: int = 2048               # tokens per projection-chain pass
    gemm_layers: int = 28
    copy: bool = True                     # gather reclaimed pages to host (north star (a))
    copy_rate_gbs: float = 32.0           # rate bound of the reclaim copies (bytes per window)
    copy_burst_bytes: int = 64 << 20
    copy_ctas: int = 8
    copy_buffer_bytes: int = 6 << 30      # largest reclaim op's bytes; the pinned arena is twice this
    static_window_frac: float = 0.1       # scenario.hpp:51
    seed: int = 2604


def c2_resparams() -> A.ReservationParams:
    """c2_llama8b_qwen7b.json's rate-control reservation (window 5 s, t_max 1 s, target 1 per
    window) with a first release interval of 200 ms instead of 1 s, so the reservation leaves
    its initial 10 % within the first ~20 s of a 60 s trace (the reference's default T_init is
    sized for its 500 s rate_control run); everything else at the defaults (memory.hpp:103-114)."""
    p = A.ReservationParams()
    p.window_us = 5_000_000
    p.t_max_us = 1_000_000
    p.t_init_us = 200_000
    return p


class Colocation:
    """One run of one policy on a shared pool + model (the pool is reset per run)."""

    def __init__(self, model: OnlineModel, pool: A.DevicePool, cfg: RtConfig, offline_backlog=(),
                 gemm_chain=None, host_bufs=None):  # host_bufs: the pinned copy arena (api.HostBuffer)
        self.m, self.pool, self.cfg = model, pool, cfg
        self.policy = cfg.policy
        self.colocated = cfg.policy != "standalone"
        self.mem = {"valve": "our_mem", "valve-fifo": "our_mem", "channel+static": "static",
                    "channel+prism": "prism", "standalone": "our_mem"}[cfg.policy]
        self.dev = model.device
        self.online = torch.cuda.Stream(device=self.dev, priority=-1)
        self.off_stream = torch.cuda.Stream(device=self.dev)
        self.gemm_stream = torch.cuda.Stream(device=self.dev)
        self.pool_stream = torch.cuda.ExternalStream(pool.view().stream, device=self.dev)
        self.backlog = offline_backlog
        self.gemm_chain = gemm_chain  # list of (a, b, c, m, n, k, tiles)
        self.arena = host_bufs  # one pinned HostBuffer: the copies' destination ring
        self.timers: list = []
        self.seq = 0

    # ----------------------------------------------------------------- timers / channel
    def _mark(self, name):
        """Phase stamp for the slow-iteration log (no-op outside run())."""
        m = getattr(self, "_marks", None)
        if m is not None:
            m.append((name, time.perf_counter()))

    def _schedule(self, when, kind, *args):
        heapq.heappush(self.timers, (int(when), self.seq, kind, args))
        self.seq += 1

    def _fire_timers(self, now):
        while self.timers and self.timers[0][0] <= now:
            when, _, kind, args = heapq.heappop(self.timers)
            if kind == "cooldown":
                self.channel.handle_cooldown(when, args[0])
            elif kind == "toggle":
                self.channel.handle_toggle(when, args[0])
            elif kind == "tick":
                self._reservation_tick(when)
            elif kind == "window":
                self._reservation_window(when)
            elif kind == "calib":
                self._calibration_end(when)
            self._mark("timer:" + kind)

    def _on_enabled(self, t):
        self._launch_offline()

    def _log_channel(self, t, what, aux, memory_cause):
        """sim.cpp:224-249 log_channel: the channel's transitions as event records."""
        log = self.res.log
        if what == A.ChannelLog.kDisableIssued:
            log.add(t, "disable_issued", effective_us=int(aux), cause="memory" if memory_cause else "busy")
        elif what == A.ChannelLog.kDisabled:
            log.add(t, "disabled")
        elif what == A.ChannelLog.kEnableIssued:
            log.add(t, "enable_issued", effective_us=int(aux))
        elif what == A.ChannelLog.kEnabled:
            log.add(t, "enabled")
        elif what == A.ChannelLog.kCooldownScheduled:
            log.add(t, "cooldown_scheduled", expiry_us=int(aux))
        elif what == A.ChannelLog.kCooldownCancelled:
            log.add(t, "cooldown_cancelled")

    # ----------------------------------------------------------------- offline tenant
    def _offline_allowed(self):
        return self.colocated and self.channel.offline_compute_allowed() and not self.offline.frozen

    def _launch_offline(self):
        if not self._offline_allowed():
            return
        if self.cfg.decode_ctas >= 0:
            st = self.gate.read()
            if st.live_ctas == 0:
                if st.total_tiles and st.tiles_claimed >= st.total_tiles:
                    # a pass over the offline KV finished: the next iteration's work list (the rows
                    # live now -- evicted requests are gone from it, sim.cpp:994-1050)
                    self._decode_tiles += st.tiles_done
                    self.gate.reset_work()
                if self.offline.running:
                    self.gate.launch_offline(self.pool, None, None, 0, 0, None, stream=self.off_stream.cuda_stream,
                                             ctas=self.cfg.decode_ctas)
        if self.gemm_chain and self.ggate.read().live_ctas == 0:
            self._launch_gemm()

    def _launch_gemm(self):
        st = self.ggate.read()
        a, b, c, m, n, k, tiles = self.gemm_chain[self._gi]
        fresh = st.tiles_claimed >= tiles
        if fresh:
            self._gemm_done_tiles += tiles
            self._gi = (self._gi + 1) % len(self.gemm_chain)
            a, b, c, m, n, k, tiles = self.gemm_chain[self._gi]
        self.ggate.launch_gemm(a.data_ptr(), b.data_ptr(), c.data_ptr(), m, n, k, ctas=self.cfg.gemm_ctas,
                               stream=self.gemm_stream.cuda_stream, fresh=fresh)

    def _harvest(self, now, force=False):
        """Harvested projection-chain tiles -> token-forwards -> offline request progress."""
        if not self.colocated or not self.gemm_chain:
            return
        if not force and now - self._last_harvest < 20_000:
            return
        self._last_harvest = now
        st = self.ggate.read()
        self._mark("harvest:gate_read")
        cur = self.gemm_chain[self._gi]
        # tiles of the completed GEMMs of the chain + the running one's (a whole pass of the chain
        # is one forward of gemm_tokens tokens)
        flop = self._chain_flop_of(self._gemm_done_tiles + min(st.tiles_done, cur[6]))
        per_token = QWEN_FLOP_PER_TOKEN * self.cfg.gemm_layers / 28
        fwd = (flop - self._flop_accounted) / per_token if flop > self._flop_accounted else 0.0
        self._flop_accounted = max(self._flop_accounted, flop)
        freed = fwd > 0 and self.offline.advance(fwd, now, self.horizon_us)
        self._mark("harvest:advance")
        if freed and not self._busy:
            self.offline.admit(now)  # while the lane is busy, admission waits for the idle edge
            self._mark("harvest:admit")

    def _chain_flop_of(self, tiles_total):
        """FLOP of the first `tiles_total` tiles of the (cyclic) chain."""
        per_pass = sum(c[6] for c in self.gemm_chain)
        flop_pass = sum(2.0 * c[3] * c[4] * c[5] for c in self.gemm_chain)
        passes, rem = divmod(tiles_total, per_pass)
        flop = passes * flop_pass
        for c in self.gemm_chain:
            if rem <= 0:
                break
            t = min(rem, c[6])
            flop += 2.0 * c[3] * c[4] * c[5] * t / c[6]
            rem -= t
        return flop

    # ----------------------------------------------------------------- memory (sim.cpp)
    def _can_acquire(self, need) -> bool:
        """Whether the policy can give the online side `need` more pages now (else: stall)."""
        P, S = self.pool, self.pool.handle_size_pages()
        slack = P.online_capacity_pages() - P.online_used_pages() + P.free_handles() * S
        if need <= slack:
            return True
        if not self.colocated or self.mem == "prism":
            return False
        if self.mem == "static":  # sim.cpp:578-594: kill k offline handles, or stall
            return P.offline_handles() >= -(-(need - slack) // S)
        return need <= slack + P.offline_handles() * S

    def _acquire(self, need, now):
        """sim.cpp:469-511 + 535-556 for the policy (the caller checked _can_acquire)."""
        P, hsz = self.pool, self.pool.handle_size_pages()
        deficit = P.online_used_pages() + need - P.online_capacity_pages()
        if deficit > 0:
            from_free = min(-(-deficit // hsz), P.free_handles())
            if from_free:
                self._grow(from_free, now, "demand")
            deficit -= from_free * hsz
        if deficit > 0:
            k = -(-deficit // hsz)
            self.res.log.add(now, "pressure", gpu=0, used_pages=P.online_used_pages() + need,
                             capacity_pages=P.online_capacity_pages())
            self.res.pressure += 1
            if self.mem == "our_mem":
                self.resctl.record_pressure(now)
            self._reclaim(min(k, P.offline_handles()), now, "shortfall", kill=self.mem == "static")
        P.online_use_pages(need)
        self._note_static_free()
        self._pressure_growth(now)

    def _note_static_free(self):
        if self.mem == "static":
            self._static_min_free = min(self._static_min_free, self.pool.free_handles())

    def _pressure_growth(self, now):
        """sim.cpp:535-556."""
        if self.mem != "our_mem" or not self.colocated:
            return
        P = self.pool
        cap = P.online_capacity_pages()
        if cap == 0 or P.online_used_pages() / cap < self.resctl.params().pressure_threshold:
            return
        self.resctl.record_pressure(now)
        self.res.log.add(now, "pressure", gpu=0, used_pages=P.online_used_pages(), capacity_pages=cap)
        self.res.pressure += 1
        h = P.online_handles()
        want = self.resctl.grow_target(h, P.total_handles()) - h
        if want <= 0:
            return
        from_free = min(want, P.free_handles())
        if from_free:
            self._grow(from_free, now, "pressure")
        want -= from_free
        if want > 0 and P.offline_handles():
            self._reclaim(min(want, P.offline_handles()), now, "growth")

    def _grow(self, k, now, cause):
        old = self.pool.online_handles()
        self.pool.online_grow(k, now)
        self.pages.sync_handles()
        self.res.log.add(now, "reserve_change", gpu=0, old_handles=old, new_handles=self.pool.online_handles(),
                         cause=cause)
        self._note_static_free()

    def _quiesce_order_pool(self, now):
        """The remap must not overtake the offline CTAs: the channel is disabled (the gate is
        raised on the online stream) and the pool stream waits for that stream's quiesce wait."""
        self.channel.ensure_disabled(now)
        gen = self.channel.disables_issued()
        if self._waited_gen != gen:
            self.gate.wait_quiesced(gen, self.online.cuda_stream)
            self._waited_gen = gen
        ev = torch.cuda.Event()
        ev.record(self.online)
        self.pool_stream.wait_event(ev)

    def _reclaim(self, k, now, purpose, kill=False):
        """Reclaim k handles as ops no larger than the pinned copy buffer allows."""
        hb = self.pool.handle_size_pages() * self.cfg.offline_page_bytes
        k_max = max(1, self.cfg.copy_buffer_bytes // hb)
        while k > 0:
            self._reclaim_op(min(k, k_max), now, purpose, kill)
            k -= k_max

    def _reclaim_op(self, k, now, purpose, kill):
        """One reclaim op (sim.cpp:885-992): quiesce-ordered fused device decision (Algorithm 1;
        FIFO for valve-fifo and the static kills), the invalidation callback, then the
        rate-bounded gather copy of the invalidated pages, whose slots carry the copy's ticket."""
        op = self.res.reclaims
        self.res.log.add(now, "reclaim_request", gpu=0, handles=int(k), op=op, purpose=purpose)
        ph = self.res.op_phase_us
        t0 = time.perf_counter()
        self._harvest(now, force=True)
        if self.offline.running:
            self.pool.set_costs(self.offline.costs())  # Cost(r) of the residents now (sim.cpp:877-883)
        t1 = time.perf_counter()
        self._quiesce_order_pool(now)
        mode = 1 if (kill or self.policy == "valve-fifo") else 0
        old_h = self.pool.online_handles()
        td = time.perf_counter()
        nh, ne, npg = self.pool.reclaim(k, now, mode)
        t3 = time.perf_counter()
        self.res.decision_us.append((t3 - td) * 1e6)
        res = self.pool.last_reclaim()
        t4 = time.perf_counter()
        for key, a_, b_ in (("costs", t0, t1), ("order", t1, td), ("decision", td, t3), ("result", t3, t4)):
            ph[key] = ph.get(key, 0.0) + (b_ - a_) * 1e6
        self._mark("reclaim:decision")
        if self.cfg.copy and not kill and npg:
            total, _ = self.pool.last_copy_layout()
            off = self._arena_alloc(total)
            self._mark("reclaim:arena")
            self.pool.reclaim_copy_start(self.arena.ptr + off, total, A.copy_params(
                ctas=self.cfg.copy_ctas, rate_bytes_per_s=self.cfg.copy_rate_gbs * 1e9,
                burst_bytes=self.cfg.copy_burst_bytes))
            ticket = self.pool.copy_ticket()
            self.pages.set_tickets([p for r in res.evicted_requests for p in res.physical_pages[r]], ticket)
            self._copies.append((op, off, total))
            self.res.copy_bytes += total
            if purpose == "shortfall":
                # when could the waiting online request write its first layer (wave 0 out) and
                # when was the whole op out -- observed on a side stream, converted at the end
                base, n, _ = ticket
                e1, e2 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                self.pool.wait_landed(base + 1, self.observer.cuda_stream)
                e1.record(self.observer)
                self.pool.wait_landed(base + n, self.observer.cuda_stream)
                e2.record(self.observer)
                self._shortfall_marks.append((t0, e1, e2))
        t5 = time.perf_counter()
        self.pages.sync_handles()
        t6 = time.perf_counter()
        ph["copy_start"] = ph.get("copy_start", 0.0) + (t5 - t4) * 1e6
        ph["sync_handles"] = ph.get("sync_handles", 0.0) + (t6 - t5) * 1e6
        lat = int((t6 - t0) * 1e6)
        self.res.log.add(now, "reclaim_done", gpu=0, op=op, latency_us=lat, handle_ids=list(res.handles))
        self.res.log.add(now, "reserve_change", gpu=0, old_handles=old_h, new_handles=self.pool.online_handles(),
                         cause="pressure" if purpose == "growth" else "demand")
        for r in res.evicted_requests:
            self.res.log.add(now, "invalidation", request_id=int(r), gpu=0,
                             invalidated_page_ids=[int(p) for p in res.invalidated_pages[r]])
        self.offline.on_evicted([int(r) for r in res.evicted_requests], now, kill)
        self.res.reclaims += 1
        self.res.reclaimed_handles += nh
        if kill:
            self.res.kills += ne
        else:
            self.res.evictions += ne

    def _arena_alloc(self, nbytes: int) -> int:
        """Destination of the next copy in the pinned arena, used as a FIFO byte ring: at most
        VALVE_COPY_RING copies in flight and no overlap with an in-flight copy's bytes; only when
        the ring is full does the host wait (for the oldest copy) -- never per op."""
        size = self.arena.nbytes
        assert nbytes <= size, "reclaim op larger than the pinned copy arena"
        while True:
            if len(self._copies) >= A.COPY_RING:
                self._complete_copy()
                continue
            if not self._copies:
                return 0
            head_off = self._copies[0][1]
            tail_end = self._copies[-1][1] + self._copies[-1][2]
            # (a non-wrapped ring has tail_end > head_off; tail_end == head_off is a wrapped, full ring)
            if tail_end > head_off:  # in-flight bytes [head_off, tail_end): free tail, then wrap to 0
                if tail_end + nbytes <= size:
                    return tail_end
                if nbytes <= head_off:
                    return 0
            elif tail_end + nbytes <= head_off:  # wrapped: free gap [tail_end, head_off)
                return tail_end
            self._complete_copy()

    def _complete_copy(self):
        self._copies.pop(0)
        st = self.pool.reclaim_copy_wait()
        if st.kernel_ms > 0:
            self.res.copy_gbs.append(st.bytes / st.kernel_ms / 1e6)

    def _reservation_tick(self, t):
        """sim.cpp:1054-1069: release one handle per quiet interval."""
        P = self.pool
        if self.resctl.release_due(t, P.online_handles()):
            old = P.online_handles()
            if self._release_online(1) > 0:
                self.res.log.add(t, "reserve_change", gpu=0, old_handles=old, new_handles=P.online_handles(),
                                 cause="release")
                self.res.releases += 1
                if not self._busy:  # the offline engine admits at its next iteration
                    self.offline.admit(t)
                    self._launch_offline()
        self.resctl.note_tick(t)
        self._schedule(t + self.resctl.interval(), "tick")

    def _release_online(self, k) -> int:
        """online_release(k) (memory.cpp:37-51 releases the lowest-id online handles): first move
        any online KV out of those handles (a device copy of the slot on the online stream), so
        the slots the reference's aggregate accounting gives back are really empty."""
        P, S = self.pool, self.pool.handle_size_pages()
        n_on, used = P.online_handles(), P.online_used_pages()
        r = max(0, min(k, n_on - (-(-used // S))))
        if r == 0:
            return 0
        going = sorted(self.pages.handles)[:r]
        move = [s for h in going for s in range(h * S, (h + 1) * S) if s in self.pages.used]
        if move:
            # move the KV out of the handles going back -- only into slots whose old bytes are
            # already out (no ticket): a release must never make the online lane wait for a copy;
            # if there are not enough such slots the release waits for a later tick
            if self.pages.ticket:
                self.pages.refresh_landed()
            if self.pages.clean_count_outside(set(going)) < len(move):
                self.res.deferred_releases += 1
                return 0
            dst = self.pages.alloc(len(move), -2, exclude_handles=set(going))
            with torch.cuda.stream(self.online):
                # slot-to-slot device copies: no temporary (a fresh 2 MiB x n allocation can make
                # the caching allocator call cudaMalloc, which waits for the running reclaim copies)
                for a_, b_ in zip(move, dst):
                    self.m.u8[b_].copy_(self.m.u8[a_])
            for s, d in zip(move, dst):
                rid = self.pages.used.pop(s)
                self.pages.used[d] = rid
                if rid < 0:
                    self._scratch = d
                else:
                    req = self._by_rid[rid]
                    req.pages[req.pages.index(s)] = d
            self.online.synchronize()
            self._mark("release:move")
        got = P.online_release(r)
        self._mark("release:pool")
        assert got == r, (got, r)
        self.pages.sync_handles()
        return got

    def _reservation_window(self, t):
        """sim.cpp:1071-1082."""
        old = self.resctl.interval()
        new = self.resctl.window_tick(t)
        if new != old:
            self.res.log.add(t, "interval_change", gpu=0, old_us=old, new_us=new)
            self.res.interval_changes += 1
        self._schedule(t + self.resctl.params().window_us, "window")

    def _calibration_end(self, t):
        """sim.cpp on_calibration_end: the static offline budget = min free handles seen."""
        self.offline.budget = self._static_min_free
        self.offline.frozen = False
        self.res.log.add(t, "static_limit", gpu=0, handles=self._static_min_free)
        self.offline.admit(t, warm=True, rng=random.Random(self.cfg.seed))
        self._launch_offline()

    # ----------------------------------------------------------------- online page writes
    def _wait_layer_fn(self, slots):
        """wait_layer(li) for a prefill into `slots`: the online stream waits for the copy waves
        under layer li's bytes of every slot with a pending ticket (one memop per layer at most)."""
        pending = [s for s in slots if s in self.pages.ticket]
        if not pending:
            return None
        state = {"t": 0}

        def wait(li):
            tgt = self.pages.layer_target(pending, li)
            if tgt > state["t"]:
                self.pool.wait_landed(tgt, self.online.cuda_stream)
                state["t"] = tgt
        return wait

    # ------------------------------------------------------------------------ main loop
    def run(self, trace: List[OnlineReq], horizon_s: float, plan: Optional[list] = None,
            admit_margin_us: int = 0, tail_s: float = 30.0) -> RunResult:
        """plan=None: the serving loop schedules (FIFO prefill-first, whole-batch decode) and
        records, per prefill, (request, decode iterations completed before it) in res.plan.
        plan=<recorded>: prefills happen in the recorded order at the recorded decode counts
        (never before the request's arrival), so a paired run differs from its baseline only in
        how long each step takes."""
        m, P, cfg = self.m, self.pool, self.cfg
        self.res = RunResult(self.policy, {}, {})
        m.gpu_events = []
        m.clock_n = 0
        log = self.res.log
        self.horizon_us = int(horizon_s * 1e6)
        P.reset()
        self.pages = OnlinePages(P)
        self.offline = OfflineEngine(P, self.backlog if self.colocated else [], log)
        self.offline.mark = self._mark
        self.observer = torch.cuda.Stream(device=self.dev)
        self._copies, self._shortfall_marks = [], []
        self._waited_gen = -1
        self._decode_tiles = 0
        self._gi, self._gemm_done_tiles, self._flop_accounted, self._last_harvest = 0, 0, 0.0, 0
        self._static_min_free = P.total_handles()
        reqs = [OnlineReq(r.rid, r.arrival_us, r.prompt, r.output) for r in trace]
        self._by_rid = by_rid = {r.rid: r for r in reqs}
        log.add(0, "run_meta", scenario="realtime_c2", preset=self.policy, seed=0, gpus=1,
                horizon_us=self.horizon_us, online_fingerprint=trace_fingerprint(trace),
                offline_fingerprint="0x%016x" % len(self.backlog))
        # initial online reserve ceil(0.1 * total) (sim.cpp:118-121, 207-210)
        P.online_grow(-(-P.total_handles() // 10), 0)
        self.pages.sync_handles()
        self._scratch = self.pages.alloc(1, -1)[0]  # decode padding rows write here
        P.online_use_pages(1)
        self.gate = self.ggate = self.channel = None
        if self.colocated:
            self.gate = A.Gate(self.dev.index or 0)
            if self.gemm_chain:
                self.ggate = A.Gate(self.dev.index or 0)
                self.gate.attach_peers([self.ggate])  # one raise quiesces both offline kernels
            hooks = A.Hooks(schedule=lambda when, gen, cd: self._schedule(when, "cooldown" if cd else "toggle", gen),
                            on_disabled=lambda t: None, on_enabled=self._on_enabled, log=self._log_channel)
            # real time: the gate takes effect at issue (raised on the online stream, which then
            # waits for the quiesce), so the modelled toggle latency is 0 (channel.cpp:13-20)
            self.channel = A.ChannelController(0, A.CooldownPolicy(cfg.max_gap_us).cooldown_us(), hooks,
                                               gate=self.gate, gate_stream=self.online.cuda_stream)
            self.resctl = A.ReservationController(cfg.resparams or c2_resparams())
            if self.mem == "our_mem":
                rp = self.resctl.params()
                self._schedule(rp.t_init_us, "tick")
                self._schedule(rp.window_us, "window")
            if self.mem == "static":
                self.offline.frozen = True
                self._schedule(int(round(self.horizon_us * cfg.static_window_frac)), "calib")
            self.offline.admit(0, warm=True, rng=random.Random(cfg.seed))
            P.fill_pages()
            self.gate.reset_work()
            if self.ggate:
                self.ggate.reset_work()
            self._launch_offline()
        queue: List[OnlineReq] = []
        decoding: List[OnlineReq] = []
        lens: Dict[int, int] = {}
        last_tok: Dict[int, int] = {}
        nxt, pi, n_decodes = 0, 0, 0
        busy, busy_since, stalled = False, 0, False
        self._busy = False
        pending_wait = None
        last_end = None
        wait_events = []
        torch.cuda.synchronize()
        import gc

        gc.collect()
        gc_was = gc.isenabled()
        gc.disable()  # a generation-2 collection in the loop is a 10-100 ms stall on either arm
        t0 = time.perf_counter()
        self._t0 = t0
        now_us = lambda: int((time.perf_counter() - t0) * 1e6)  # noqa: E731
        stop_us = int((horizon_s + tail_s) * 1e6)
        pc = time.perf_counter
        marks = self._marks = []  # (phase, perf_counter) of this loop iteration, for the slow-iteration log

        def slow_check(where):
            # an iteration that spent > 3 ms of host time before its step (or before going idle)
            if marks and pc() - marks[0][1] > 3e-3:
                self.res.slow_iterations.append(
                    {"t_us": int((marks[0][1] - t0) * 1e6), "where": where,
                     "phases_us": [[marks[i][0], int((marks[i][1] - marks[i - 1][1]) * 1e6)]
                                   for i in range(1, len(marks)) if marks[i][1] - marks[i - 1][1] > 2e-4],
                     "total_us": int((pc() - marks[0][1]) * 1e6)})

        while True:
            marks.clear()
            marks.append(("top", pc()))
            now = now_us()
            if now > stop_us:
                break
            if self.colocated:
                self._fire_timers(now)
                marks.append(("timers", pc()))
                if not busy:  # gated while busy: nothing to harvest
                    self._harvest(now)
                    marks.append(("harvest", pc()))
            while nxt < len(reqs) and reqs[nxt].arrival_us <= now:
                r = reqs[nxt]
                log.add(r.arrival_us, "arrival", **{"class": "online"}, request_id=r.rid, gpu=0,
                        prompt_tokens=r.prompt, output_tokens=r.output)
                queue.append(r)
                nxt += 1
            act = None
            if plan is None:
                if queue and (not decoding or queue[0].arrival_us <= now - admit_margin_us):
                    act = ("prefill", queue[0].rid)
                elif decoding:
                    act = ("decode", len(decoding))
                finished = act is None and nxt >= len(reqs)
            else:
                # exact replay: the planned prefill goes after exactly the recorded number of decode
                # iterations; if its request has not arrived yet the loop waits for it (spinning
                # while a batch is decoding: the lane stays busy), so both arms of a pair run the
                # same batches in the same order and differ only in step durations
                finished = pi >= len(plan) and not decoding
                spin = False
                if pi < len(plan) and (n_decodes >= plan[pi][1] or not decoding):
                    rid = plan[pi][0]
                    if by_rid[rid].arrival_us <= now:
                        act = ("prefill", rid)
                    elif decoding:
                        spin = True
                elif decoding:
                    act = ("decode", len(decoding))
                if spin:
                    continue
            # page demand of the action (sim.cpp:469-511); a policy that cannot supply it stalls
            need, need_by = 0, []
            if act is not None:
                if act[0] == "prefill":
                    need = -(-by_rid[act[1]].prompt // cfg.page_tokens)
                else:
                    need_by = [max(0, -(-(lens[r.rid] + 1) // cfg.page_tokens) - len(r.pages)) for r in decoding]
                    need = sum(need_by)
                if need and not self._can_acquire(need):
                    if not stalled:
                        stalled = True
                        self.res.stalls += 1
                        log.add(now, "stall", gpu=0, **{"class": "online"}, reason="memory")
                    act = None
            if act is None:
                if busy:  # idle edge (sim.cpp:371-380)
                    busy = self._busy = False
                    log.add(now, "busy", gpu=0, **{"class": "online"}, start_us=busy_since, end_us=now)
                    if self.colocated:
                        self.channel.note_all_idle(now)
                        self._fire_timers(now)
                        self._harvest(now, force=True)
                        self.offline.admit(now)
                if finished and not stalled:
                    break
                marks.append(("idle_edge", pc()))
                if self.colocated and self._offline_allowed():
                    self._launch_offline()
                    if stalled:
                        self.offline.admit(now)
                marks.append(("launch_offline", pc()))
                slow_check("idle")
                time.sleep(50e-6)
                continue
            stalled = False
            gap_from = last_end if busy else None
            if act[0] == "prefill":
                self.res.plan.append((act[1], n_decodes))
                pi += 1
            else:
                n_decodes += 1
            if not busy:  # busy edge: raise + wait for the offline CTAs to retire (sim.cpp:362-369)
                busy = self._busy = True
                busy_since = now
                self.res.busy_starts.append(now)
                if self.colocated:
                    self._harvest(now, force=True)
                    self.channel.note_busy(now)
                    self._fire_timers(now)
                    gen = self.channel.disables_issued()
                    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    e0.record(self.online)
                    self.gate.wait_quiesced(gen, self.online.cuda_stream)
                    self._waited_gen = gen
                    e1.record(self.online)
                    pending_wait = (e0, e1)
                    self.res.disables = self.channel.disables_issued()
                marks.append(("busy_edge", pc()))
            if act[0] == "prefill":
                r = by_rid[act[1]]
                queue.remove(r)
                self._acquire(need, now)
                marks.append(("acquire", pc()))
                r.pages = self.pages.alloc(need, r.rid)
                marks.append(("alloc", pc()))
                if pending_wait is not None:
                    wait_events.append((now, r.rid, pending_wait))
                    pending_wait = None
                toks = torch.randint(0, m.s.vocab, (r.prompt,), device=self.dev)
                marks.append(("tokens", pc()))
                slow_check("prefill")
                t_it = now_us()
                if gap_from is not None:
                    self.res.step_gap_us.append(t_it - gap_from)
                log.add(t_it, "prefill_start", **{"class": "online"}, request_id=r.rid, gpu=0, tokens=r.prompt)
                with torch.cuda.stream(self.online):
                    tok = m.prefill(toks, r.pages, self._wait_layer_fn(r.pages))
                self.online.synchronize()
                lens[r.rid] = r.prompt
                last_tok[r.rid] = int(tok.item())
                t_pe = last_end = now_us()
                log.add(t_pe, "prefill_end", **{"class": "online"}, request_id=r.rid, gpu=0)
                self.res.prefill_us.append(t_pe - t_it)
                decoding.append(r)
                continue
            # one decode iteration over the batch
            if need:
                self._acquire(need, now)
                marks.append(("acquire", pc()))
            new_slots = []
            for r, nb in zip(decoding, need_by):
                if nb:
                    sl = self.pages.alloc(nb, r.rid)
                    r.pages += sl
                    new_slots += sl
            if new_slots:
                tgt = self.pages.full_target(new_slots)
                if tgt:
                    self.pool.wait_landed(tgt, self.online.cuda_stream)
            marks.append(("alloc", pc()))
            slow_check("decode")
            t_it = now_us()
            self.res.decode_t_us.append(t_it)
            if gap_from is not None:
                self.res.step_gap_us.append(t_it - gap_from)
            with torch.cuda.stream(self.online):
                out = m.decode([last_tok[r.rid] for r in decoding],
                               [r.pages[lens[r.rid] // cfg.page_tokens] for r in decoding],
                               [lens[r.rid] for r in decoding], [r.pages for r in decoding], self._scratch)
            self.online.synchronize()
            t_emit = last_end = now_us()
            self.res.decode_iter_us.append(t_emit - t_it)
            done = []
            for r, o in zip(decoding, out.tolist()):
                lens[r.rid] += 1
                last_tok[r.rid] = o
                r.emits.append(t_emit)
                if len(r.emits) == 1:
                    r.first_us = t_emit
                    log.add(t_emit, "first_token", **{"class": "online"}, request_id=r.rid, gpu=0)
                if len(r.emits) == r.output:
                    done.append(r)
            for r in done:
                decoding.remove(r)
                self.pages.release(r.pages)
                P.online_free_pages(len(r.pages))
                if r.output > 1:
                    self.res.tpot_us[r.rid] = (r.emits[-1] - r.emits[0]) / (r.output - 1)
                self.res.ttft_us[r.rid] = r.first_us - r.arrival_us
                log.add(t_emit, "done", **{"class": "online"}, request_id=r.rid, gpu=0, tokens=len(r.emits),
                        first_token_us=r.emits[0], last_token_us=r.emits[-1], digest="0x0000000000000000")
        self.online.synchronize()
        self.res.wall_s = time.perf_counter() - t0
        self.res.decode_gpu_us = [a.elapsed_time(b) * 1e3 for a, b in m.gpu_events]
        self.res.decode_sm_mhz = m.clock_mhz[: m.clock_n].tolist()
        m.gpu_events = None
        end = now_us()
        if gc_was:
            gc.enable()
        if busy:
            log.add(end, "busy", gpu=0, **{"class": "online"}, start_us=busy_since, end_us=end)
        for t_adm, rid, (e0, e1) in wait_events:
            self.res.quiesce_wait_us.append(e0.elapsed_time(e1) * 1e3)
            log.add(t_adm, "preempt_wait", gpu=0, request_id=rid, delay_us=int(round(self.res.quiesce_wait_us[-1])))
        if self.colocated:
            self._shutdown_offline(end)
        return self.res

    def _shutdown_offline(self, end):
        """Stop the tenant without running its remaining work: raise, wait for the quiesce, drop
        the work lists (queued launches retire at once), release, drain the copies."""
        self._harvest(end, force=True)
        gen = self.channel.disables_issued() + 1000
        self.gate.raise_(gen, self.online.cuda_stream)
        self.gate.wait_quiesced(gen, self.online.cuda_stream)
        self.online.synchronize()
        self.res.offline_decode_bytes = (self._decode_tiles + self.gate.read().tiles_done) * 16384.0
        self.gate.cancel_work()
        if self.ggate:
            self.ggate.cancel_work()
        self.gate.release(gen, self.online.cuda_stream)
        while self._copies:
            self._complete_copy()
        torch.cuda.synchronize()
        # host instant <-> event timeline: one anchor event recorded now
        anchor = torch.cuda.Event(enable_timing=True)
        anchor.record(self.observer)
        anchor.synchronize()
        t_anchor = time.perf_counter()
        for t_issue, e1, e2 in self._shortfall_marks:
            self.res.shortfall_to_write_us.append((t_anchor - t_issue) * 1e6 - e1.elapsed_time(anchor) * 1e3)
            self.res.shortfall_full_copy_us.append((t_anchor - t_issue) * 1e6 - e2.elapsed_time(anchor) * 1e3)
        o = self.offline
        self.res.offline_tokens_done, self.res.offline_completed = o.tokens_done, o.completed
        self.res.offline_forwards, self.res.offline_lost_forwards = o.forwards, o.lost
        self.gate = self.ggate = self.channel = None


# ------------------------------------------------------------------------ measurement

def paired_increase(base: Dict[int, float], other: Dict[int, float]):
    """metrics.cpp:49-65: mean and max of per-request % increases over paired requests."""
    pcts = [(other[i] - b) / b * 100.0 for i, b in sorted(base.items()) if i in other and b > 0]
    if not pcts:
        return {"mean_pct": None, "max_pct": None, "pairs": 0}
    return {"mean_pct": sum(pcts) / len(pcts), "max_pct": max(pcts), "pairs": len(pcts)}


def qwen_chain(device, tokens: int, layers: int = 28, seed: int = 7):
    """A random-init Qwen2-7B's projection chain over `tokens` tokens: per layer qkv (4608),
    o (3584), gate/up (2 x 18944), down (18944 -> 3584) as gated tcgen05 GEMMs."""
    g = torch.Generator(device=device).manual_seed(seed)

    def rnd(*shape, scale=1.0):
        return (torch.randn(*shape, device=device, generator=g) * scale).to(torch.bfloat16)

    d, qkv, ffn = 3584, 4608, 18944
    x, act = rnd(tokens, d), rnd(tokens, ffn)
    outs = {n: torch.empty(tokens, n, device=device, dtype=torch.bfloat16) for n in (qkv, d, 2 * ffn)}
    chain = []
    for _ in range(layers):
        for (a, n, k) in ((x, qkv, d), (x, d, d), (x, 2 * ffn, d), (act, d, ffn)):
            chain.append((a, rnd(n, k, scale=0.02), outs[n], tokens, n, k))
    return [(a, b, c, mm, n, k, (mm // (256 if mm % 256 == 0 else 128)) * (n // 256)) for (a, b, c, mm, n, k) in chain]


def warm(model: OnlineModel, pool: A.DevicePool, trace: List[OnlineReq]):
    """Every prefill length of the trace and every decode batch bucket once (cuBLAS heuristics,
    graph capture), so no measured run pays first-use costs."""
    pool.reset()
    S = pool.handle_size_pages()
    pool.online_grow(pool.total_handles(), 0)
    slots = list(range(min(pool.total_handles() * S, 300)))
    for plen in sorted({r.prompt for r in trace})[:: max(1, len(trace) // 24)]:
        model.prefill(torch.randint(0, model.s.vocab, (plen,), device=model.device),
                      slots[: -(-plen // PAGE_TOKENS)])
    for B in model.BUCKETS:
        model.decode([0] * B, [slots[1]] * B, [40] * B, [slots[:3]] * B, slots[0])
    torch.cuda.synchronize()
    pool.reset()


class _Clocks:
    """nvidia-smi SM clock / power samples (500 ms) over one run."""

    def __init__(self, device):
        self.device, self.rows, self.proc = device, [], None

    def __enter__(self):
        import subprocess
        import threading

        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), "--query-gpu=clocks.sm,power.draw,temperature.gpu,temperature.memory,clocks.mem",
                 "--format=csv,noheader,nounits", "-lms", "500"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            threading.Thread(target=self._read, daemon=True).start()
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            vals = []
            for x in line.split(","):
                try:
                    vals.append(float(x))
                except ValueError:  # "[N/A]" on boards without a memory sensor
                    vals.append(float("nan"))
            if len(vals) >= 2 and vals[0] == vals[0]:
                self.rows.append(tuple(vals))

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
        out = {"sm_mhz_median": sm[len(sm) // 2], "sm_mhz_min": sm[0], "power_w_median": pw[len(pw) // 2],
               "power_w_max": pw[-1], "samples": len(sm)}
        for i, key in ((2, "gpu_temp_c"), (3, "mem_temp_c"), (4, "mem_mhz")):
            v = sorted(r[i] for r in self.rows if len(r) > i and r[i] == r[i])
            if v:
                out[key + "_median"], out[key + "_max"] = v[len(v) // 2], v[-1]
        return out


def _med_runs(dicts):
    """Per-request median over runs (requests present in every run)."""
    keys = set(dicts[0])
    for d in dicts[1:]:
        keys &= set(d)
    out = {}
    for k in sorted(keys):
        v = sorted(d[k] for d in dicts)
        n = len(v)
        out[k] = v[n // 2] if n % 2 else 0.5 * (v[n // 2 - 1] + v[n // 2])
    return out


def _pct(xs, p):
    xs = sorted(xs)
    return xs[min(len(xs) - 1, int(round(p / 100 * (len(xs) - 1))))] if xs else None


def _deviations(plan, executed):
    want = {rid: k for rid, k in plan}
    return sum(1 for rid, k in executed if want.get(rid) != k)


def measure(horizon=60.0, base=2.0, spike=20.0, period=6.0, width=1.0, prompt=(2000, 4000), output=(32, 128),
            handles=0, seed=2604, layers=32, device=0, repeats=2, policies=("valve-fifo", "channel+static",
                                                                          "channel+prism"),
            cfg: Optional[RtConfig] = None, log_dir: Optional[str] = None, tail_s=30.0):
    """BASELINE C2 trace (spike online: base 2/s, 20/s for 1 s every 6 s, prompt 2000-4000,
    output 32-128, >= 60 s; Qwen2-7B offline backlog) on a pool of `handles` 128 MiB handles (0:
    as many as fit, at most 1,024), C3's MIAD reservation resizing and rate-bounded copies.

    Runs: repeats+1 standalone and `repeats` valve runs interleaved (A B A B .. A), then one run of
    each extra policy.  Every run replays the action sequence recorded by an untimed standalone
    run, so arms differ only in how long each step takes.  TTFT/TPOT deltas pair per-request
    medians (metrics.cpp:49-65); the A/A noise floor pairs the even standalone runs against the
    odd ones.  Normalized offline throughput = offline tokens / channel+prism's
    (metrics.cpp:243-247)."""
    dev = torch.device("cuda", device)
    torch.cuda.set_device(dev)
    cfg = cfg or RtConfig()
    shape = ModelShape(layers=layers)
    model = OnlineModel(shape, dev)
    chain = qwen_chain(dev, cfg.gemm_tokens, cfg.gemm_layers) if cfg.gemm_ctas >= 0 else None
    torch.cuda.synchronize()
    if not handles:
        free, _ = torch.cuda.mem_get_info(dev)
        handles = int(min(1024, (free - 6e9) // (64 * shape.page_bytes)))
    pool = A.DevicePool(handles, 64, PAGE_TOKENS, device=device, slot_bytes=shape.page_bytes,
                        page_bytes=min(cfg.offline_page_bytes, shape.page_bytes), max_requests=4096,
                        max_pages_per_request=512)
    cfg.offline_page_bytes = min(cfg.offline_page_bytes, shape.page_bytes)
    model.bind(pool)
    trace = spike_trace(seed, horizon, base, spike, period, width, prompt=prompt, output=output)
    backlog = offline_population(seed + 1, 20 * handles)
    bufs = A.HostBuffer(2 * cfg.copy_buffer_bytes)
    warm(model, pool, trace)
    plan = None
    for _ in range(2):  # the second of two live standalone runs (the first pays first-use costs)
        plan = Colocation(model, pool, RtConfig(policy="standalone")).run(trace, horizon, admit_margin_us=6000,
                                                                          tail_s=tail_s).plan

    def one(policy):
        c = RtConfig(**{**cfg.__dict__, "policy": policy})
        with _Clocks(device) as ck:
            r = Colocation(model, pool, c, backlog, chain, bufs).run(trace, horizon, plan=plan, tail_s=tail_s)
        r.clocks = ck.summary()
        torch.cuda.synchronize()
        return r

    solos, colos, extra = [], [], {}
    for _ in range(repeats):
        solos.append(one("standalone"))
        colos.append(one(cfg.policy if cfg.policy != "standalone" else "valve"))
    solos.append(one("standalone"))
    for pol in policies:
        extra[pol] = one(pol)
    runs = {"solo": solos, "colo": colos, **{pol.replace("+", "_"): [r] for pol, r in extra.items()}}
    if log_dir:
        os.makedirs(log_dir, exist_ok=True)
        import json

        for name, rs in runs.items():
            for i, r in enumerate(rs):
                r.log.write_jsonl(os.path.join(log_dir, f"{name}{i}.jsonl"))
                with open(os.path.join(log_dir, f"{name}{i}_steps.json"), "w") as f:  # per-step device times
                    json.dump({"decode_gpu_us": [round(x, 1) for x in r.decode_gpu_us],
                               "decode_sm_mhz": [round(x) for x in r.decode_sm_mhz],
                               "decode_t_us": r.decode_t_us, "busy_starts": r.busy_starts,
                               "decode_iter_us": r.decode_iter_us, "prefill_us": r.prefill_us}, f)

    base_ttft, base_tpot = _med_runs([s.ttft_us for s in solos]), _med_runs([s.tpot_us for s in solos])
    even, odd = solos[0::2], solos[1::2]
    aa_ttft = paired_increase(_med_runs([s.ttft_us for s in even]), _med_runs([s.ttft_us for s in odd]))
    aa_tpot = paired_increase(_med_runs([s.tpot_us for s in even]), _med_runs([s.tpot_us for s in odd]))

    def arm(rs):
        ttft = paired_increase(base_ttft, _med_runs([r.ttft_us for r in rs]))
        tpot = paired_increase(base_tpot, _med_runs([r.tpot_us for r in rs]))
        r = rs[-1]
        q = [w for x in rs for w in x.quiesce_wait_us]
        sf = [w for x in rs for w in x.shortfall_to_write_us]
        sc = [w for x in rs for w in x.shortfall_full_copy_us]
        return {
            "ttft_delta_pct": ttft["mean_pct"], "tpot_delta_pct": tpot["mean_pct"], "pairs": ttft["pairs"],
            "per_run_ttft_delta_pct": [paired_increase(base_ttft, x.ttft_us)["mean_pct"] for x in rs],
            "per_run_tpot_delta_pct": [paired_increase(base_tpot, x.tpot_us)["mean_pct"] for x in rs],
            "offline_tokens_per_s": r.offline_tokens_done / horizon, "offline_completed": r.offline_completed,
            "offline_forwards_per_s": r.offline_forwards / r.wall_s,
            "offline_lost_forward_frac": (r.offline_lost_forwards / r.offline_forwards) if r.offline_forwards else None,
            "offline_decode_gbs": r.offline_decode_bytes / r.wall_s / 1e9,
            "disables": r.disables, "disables_per_request": r.disables / max(1, len(trace)),
            "reclaims": r.reclaims, "reclaimed_handles": r.reclaimed_handles, "evictions": r.evictions,
            "kills": r.kills, "releases": r.releases, "deferred_releases": r.deferred_releases,
            "interval_changes": r.interval_changes,
            "pressure_events": r.pressure, "stalls": r.stalls,
            "copy_gb": r.copy_bytes / 1e9, "copy_gbs_mean": (sum(r.copy_gbs) / len(r.copy_gbs)) if r.copy_gbs else None,
            "decision_us_p50": _pct([d for x in rs for d in x.decision_us], 50),
            "slow_iterations": {"n": sum(len(x.slow_iterations) for x in rs),
                                "worst": sorted((w for x in rs for w in x.slow_iterations), key=lambda w: -w["total_us"])[:5]},
            "decode_iter_ms_mean": sum(d for x in rs for d in x.decode_iter_us) / max(1, sum(len(x.decode_iter_us) for x in rs)) / 1e3,
            "step_gap_us_mean": sum(d for x in rs for d in x.step_gap_us) / max(1, sum(len(x.step_gap_us) for x in rs)),
            "decode_gpu_ms_mean": sum(d for x in rs for d in x.decode_gpu_us) / max(1, sum(len(x.decode_gpu_us) for x in rs)) / 1e3,
            "decode_sm_mhz_mean": sum(d for x in rs for d in x.decode_sm_mhz) / max(1, sum(len(x.decode_sm_mhz) for x in rs)),
            "step_gap_us_p99": _pct([d for x in rs for d in x.step_gap_us], 99),
            "op_host_us_mean": {k: v / max(1, r.reclaims) for k, v in r.op_phase_us.items()},
            "quiesce_wait_us": {"p50": _pct(q, 50), "p99": _pct(q, 99), "max": max(q) if q else None, "n": len(q)},
            "shortfall_to_first_write_us": {"p50": _pct(sf, 50), "p99": _pct(sf, 99), "n": len(sf)},
            "shortfall_to_full_copy_us": {"p50": _pct(sc, 50), "p99": _pct(sc, 99), "n": len(sc)},
            "plan_deviations": [_deviations(plan, x.plan) for x in rs],
            "wall_s": r.wall_s, "clocks": [x.clocks for x in rs],
        }

    out = {
        "trace": {"horizon_s": horizon, "online_requests": len(trace), "base_rate": base, "spike_rate": spike,
                  "period_s": period, "width_s": width, "prompt": list(prompt), "output": list(output),
                  "model": f"Llama-3-8B-shaped, {layers} layers, random init bf16, KV in pool slots"},
        "pool_handles": handles, "page_bytes_online": shape.page_bytes, "page_bytes_offline": cfg.offline_page_bytes,
        "copy_rate_bound_gbs": cfg.copy_rate_gbs if cfg.copy else None,
        "reservation": {k: getattr(cfg.resparams or c2_resparams(), k) for k in ("window_us", "t_max_us", "t_min_us",
                                                                              "t_init_us", "delta_us", "alpha", "beta")},
        "schedule": f"replayed: every run places each prefill at the decode count recorded by an untimed "
                    f"standalone run ({len(plan)} prefills)",
        "design": f"A B x{repeats} + A (standalone / {colos[0].policy}); per-request medians paired (metrics.cpp:49-65)",
        "aa_noise_ttft_pct": aa_ttft["mean_pct"], "aa_noise_tpot_pct": aa_tpot["mean_pct"],
        "standalone": {"ttft_ms_mean": sum(base_ttft.values()) / max(1, len(base_ttft)) / 1e3,
                       "tpot_ms_mean": sum(base_tpot.values()) / max(1, len(base_tpot)) / 1e3,
                       "decode_iter_ms_p50": _pct([x for s in solos for x in s.decode_iter_us], 50) / 1e3,
                       "prefill_ms_p50": _pct([x for s in solos for x in s.prefill_us], 50) / 1e3,
                       "decode_iter_ms_mean": sum(d for x in solos for d in x.decode_iter_us) / max(1, sum(len(x.decode_iter_us) for x in solos)) / 1e3,
                       "step_gap_us_mean": sum(d for x in solos for d in x.step_gap_us) / max(1, sum(len(x.step_gap_us) for x in solos)),
                       "decode_gpu_ms_mean": sum(d for x in solos for d in x.decode_gpu_us) / max(1, sum(len(x.decode_gpu_us) for x in solos)) / 1e3,
                       "decode_sm_mhz_mean": sum(d for x in solos for d in x.decode_sm_mhz) / max(1, sum(len(x.decode_sm_mhz) for x in solos)),
                       "step_gap_us_p99": _pct([d for x in solos for d in x.step_gap_us], 99),
                       "plan_deviations": [_deviations(plan, x.plan) for x in solos],
                       "slow_iterations": {"n": sum(len(x.slow_iterations) for x in solos),
                                           "worst": sorted((w for x in solos for w in x.slow_iterations),
                                                           key=lambda w: -w["total_us"])[:5]},
                       "clocks": [x.clocks for x in solos]},
        colos[0].policy: arm(colos),
        **{pol: arm([r]) for pol, r in extra.items()},
    }
    prism = extra.get("channel+prism")
    if prism is not None and prism.offline_tokens_done > 0:
        for pol in [colos[0].policy, *extra]:
            rs = colos if pol == colos[0].policy else [extra[pol]]
            out[pol]["normalized_offline_throughput"] = rs[-1].offline_tokens_done / prism.offline_tokens_done
    fifo = extra.get("valve-fifo")
    if fifo is not None:
        v, f = colos[-1], fifo
        lv = v.offline_lost_forwards / v.offline_forwards if v.offline_forwards else None
        lf = f.offline_lost_forwards / f.offline_forwards if f.offline_forwards else None
        out["policy_contrast"] = {
            "lost_forward_frac": {"algorithm1": lv, "fifo": lf},
            "offline_tokens": {"algorithm1": v.offline_tokens_done, "fifo": f.offline_tokens_done},
            "throughput_loss_reduction_pct": (1 - lv / lf) * 100 if lv is not None and lf else None,
        }
    del model, pool, bufs
    import gc

    gc.collect()
    torch.cuda.synchronize()
    torch.cuda.empty_cache()
    return out
