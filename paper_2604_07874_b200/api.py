"""Python mirror of the reference runtime API (colosim, /root/reference/proj/include/colosim),
bound to the C ABI of include/valve_cuda.h.

Names, argument meaning and error behaviour follow the reference so tests read like its
doctest suites (tests/test_memory.cpp, test_reclaim.cpp, test_channel.cpp):

    MemoryPool                memory.hpp:19-98
    ReservationParams/-Controller  memory.hpp:103-146
    ReclaimHandle/Instance, evicted_cost, selective/fifo/oracle_reclaim   reclaim.hpp:12-37
    ChannelController, CooldownPolicy, ChannelLog   channel.hpp:12-80

C++ exception types map to Python ones with the same hierarchy
(invalid_argument / out_of_range are logic_errors):

    InvalidArgument(LogicError, ValueError)   std::invalid_argument
    OutOfRange(LogicError, IndexError)        std::out_of_range
    LogicError                                std::logic_error
    ValveRuntimeError(RuntimeError)           std::runtime_error
    CudaError(RuntimeError)                   CUDA failure

The default backend is libvalve.so (sm_100a kernels).  `Backend` exists so the test suite
can drive the CPU checkers in oracle/ through the *same* wrapper; nothing in this package
constructs such a backend.
"""
from __future__ import annotations

import ctypes as C
import itertools
import os
from dataclasses import dataclass, field
from typing import Callable, Dict, List, Optional, Sequence

_HERE = os.path.dirname(os.path.abspath(__file__))
LIBVALVE = os.path.join(_HERE, "libvalve.so")
COPY_RING = 8  # VALVE_COPY_RING (valve_cuda.h): reclaim copies in flight per pool


class LogicError(Exception):
    """std::logic_error"""


class InvalidArgument(LogicError, ValueError):
    """std::invalid_argument"""


class OutOfRange(LogicError, IndexError):
    """std::out_of_range"""


class ValveRuntimeError(RuntimeError):
    """std::runtime_error"""


class CudaError(RuntimeError):
    """CUDA failure inside the library"""


_EXC = {1: InvalidArgument, 2: LogicError, 3: ValveRuntimeError, 4: CudaError, 5: OutOfRange}

i32, i64, u32, dbl = C.c_int32, C.c_int64, C.c_uint32, C.c_double
P = C.POINTER


class _ResParams(C.Structure):
    _fields_ = [("alpha", dbl), ("beta", dbl), ("t_init_us", i64), ("delta_us", i64),
                ("t_min_us", i64), ("t_max_us", i64), ("window_us", i64),
                ("target_per_window", dbl), ("h_min", i32), ("pressure_threshold", dbl)]


_SCHED = C.CFUNCTYPE(None, C.c_void_p, i64, i64, C.c_int)
_ONT = C.CFUNCTYPE(None, C.c_void_p, i64)
_LOG = C.CFUNCTYPE(None, C.c_void_p, i64, C.c_int, i64, C.c_int)


class _Hooks(C.Structure):
    _fields_ = [("user", C.c_void_p), ("schedule", _SCHED), ("on_disabled", _ONT),
                ("on_enabled", _ONT), ("log", _LOG)]


class Backend:
    """A loaded shared library exposing the pool/selection/controller C API with `prefix`."""

    def __init__(self, path: str, prefix: str, device_arg: bool, name: str):
        if not os.path.exists(path):
            raise ImportError(f"{name}: {path} is missing -- run __graft_entry__.build()")
        self.lib = C.CDLL(path)
        self.prefix = prefix
        self.device_arg = device_arg  # valve_select / valve_evicted_cost take a device ordinal
        self.name = name
        self._declare()

    def fn(self, name):
        return getattr(self.lib, self.prefix + name)

    def _declare(self):
        L, p = self.lib, self.prefix
        sig = {
            "last_error": (C.c_char_p, []),
            "pool_create": (C.c_int, [C.c_int, C.c_int, C.c_int, P(C.c_void_p)]),
            "pool_destroy": (None, [C.c_void_p]),
            "pool_counts": (C.c_int, [C.c_void_p, P(i64)]),
            "pool_online_grow": (C.c_int, [C.c_void_p, C.c_int, i64]),
            "pool_online_release": (C.c_int, [C.c_void_p, C.c_int, P(C.c_int)]),
            "pool_online_use_pages": (C.c_int, [C.c_void_p, i64]),
            "pool_online_free_pages": (C.c_int, [C.c_void_p, i64]),
            "pool_offline_reserve": (C.c_int, [C.c_void_p, i64, C.c_int, i64, C.c_int, P(C.c_int)]),
            "pool_offline_release": (C.c_int, [C.c_void_p, i64]),
            "pool_requests_on_handle": (C.c_int, [C.c_void_p, C.c_int, P(i64), C.c_int, P(C.c_int)]),
            "pool_handles_of_request": (C.c_int, [C.c_void_p, i64, P(C.c_int), C.c_int, P(C.c_int)]),
            "pool_offline_pages_of": (C.c_int, [C.c_void_p, i64, P(C.c_int)]),
            "pool_snapshot": (C.c_int, [C.c_void_p, P(C.c_int), P(i64), P(C.c_int), P(i64), C.c_int,
                                        C.c_int, P(C.c_int), P(C.c_int)]),
            "pool_apply_reclaim": (C.c_int, [C.c_void_p, P(C.c_int), C.c_int, i64, P(C.c_int),
                                             P(C.c_int), P(i64), P(C.c_int), P(C.c_int), P(i64),
                                             P(C.c_int), P(C.c_int), C.c_int, C.c_int, P(C.c_int)]),
            "pool_handle_state": (C.c_int, [C.c_void_p, C.c_int, P(C.c_int)]),
            "pool_handle_mapped_at": (C.c_int, [C.c_void_p, C.c_int, P(i64)]),
            "pool_check_invariants": (C.c_int, [C.c_void_p]),
            "pool_block_table": (C.c_int, [C.c_void_p, i64, P(C.c_int), C.c_int, P(C.c_int)]),
            "resparams_default": (None, [P(_ResParams)]),
            "resctl_create": (C.c_int, [P(_ResParams), P(C.c_void_p)]),
            "resctl_destroy": (None, [C.c_void_p]),
            "resctl_interval": (i64, [C.c_void_p]),
            "resctl_pressure_events": (i64, [C.c_void_p]),
            "resctl_grow_target": (C.c_int, [C.c_void_p, C.c_int, C.c_int]),
            "resctl_record_pressure": (None, [C.c_void_p, i64]),
            "resctl_release_due": (C.c_int, [C.c_void_p, i64, C.c_int]),
            "resctl_note_tick": (None, [C.c_void_p, i64]),
            "resctl_window_tick": (i64, [C.c_void_p, i64]),
            "resctl_pressure_in_window": (i64, [C.c_void_p, i64]),
            "channel_create": (C.c_int, [i64, i64, P(_Hooks), P(C.c_void_p)]),
            "channel_destroy": (None, [C.c_void_p]),
            "channel_state": (C.c_int, [C.c_void_p]),
            "channel_offline_compute_allowed": (C.c_int, [C.c_void_p]),
            "channel_disables_issued": (i64, [C.c_void_p]),
            "channel_pending_effective": (i64, [C.c_void_p]),
            "channel_note_busy": (None, [C.c_void_p, i64]),
            "channel_note_all_idle": (None, [C.c_void_p, i64]),
            "channel_ensure_disabled": (i64, [C.c_void_p, i64]),
            "channel_handle_toggle": (None, [C.c_void_p, i64, i64]),
            "channel_handle_cooldown": (None, [C.c_void_p, i64, i64]),
        }
        sel = [C.c_int, P(C.c_int), P(i64), P(C.c_int), P(i64), C.c_int, P(i64), P(i64), C.c_int,
               C.c_int, P(C.c_int), P(C.c_int)]
        ec = [C.c_int, P(C.c_int), P(C.c_int), P(i64), C.c_int, P(i64), P(i64), P(C.c_int),
              C.c_int, P(i64)]
        if self.device_arg:
            sel = [C.c_int] + sel
            ec = [C.c_int] + ec
        sig["select"] = (C.c_int, sel)
        sig["evicted_cost"] = (C.c_int, ec)
        for name, (res, args) in sig.items():
            f = getattr(L, p + name)
            f.restype = res
            f.argtypes = args

    def check(self, rc: int):
        if rc:
            msg = self.fn("last_error")().decode(errors="replace")
            raise _EXC.get(rc, ValveRuntimeError)(msg)


_VALVE: Optional[Backend] = None


def valve_backend() -> Backend:
    """The product backend (libvalve.so).  Raises ImportError if it was not built."""
    global _VALVE
    if _VALVE is None:
        _VALVE = Backend(LIBVALVE, "valve_", True, "libvalve")
        _declare_valve_extras(_VALVE.lib)
    return _VALVE


def _arr(ctype, n):
    return (ctype * max(int(n), 1))()


def _ptr(a, ctype):
    if hasattr(a, "ctypes") and hasattr(a, "dtype"):  # numpy array
        return a.ctypes.data_as(P(ctype))
    return C.cast(a, P(ctype))


def _np():
    import numpy

    return numpy


def _np_empty(n, dtype):
    return _np().empty(max(int(n), 1), dtype=dtype)


# ---------------------------------------------------------------------------- reclaim types

@dataclass
class ReclaimHandle:
    """reclaim.hpp:12-16"""
    id: int = 0
    mapped_at: int = 0
    requests: List[int] = field(default_factory=list)


@dataclass
class ReclaimInstance:
    """reclaim.hpp:18-21 (cost: request id -> recompute cost)"""
    handles: List[ReclaimHandle] = field(default_factory=list)
    cost: Dict[int, int] = field(default_factory=dict)


@dataclass
class ReclaimResult:
    """memory.hpp:64-68"""
    handles: List[int]
    evicted_requests: List[int]
    invalidated_pages: Dict[int, List[int]]
    # B200 additions, aligned with invalidated_pages[req]: physical page, block index
    physical_pages: Dict[int, List[int]] = field(default_factory=dict)
    block_index: Dict[int, List[int]] = field(default_factory=dict)


def _csr(inst: ReclaimInstance):
    np = _np()
    hs = inst.handles
    n = len(hs)
    ids = np.fromiter((h.id for h in hs), np.int32, n) if n else _np_empty(0, np.int32)
    mapped = np.fromiter((h.mapped_at for h in hs), np.int64, n) if n else _np_empty(0, np.int64)
    off = np.zeros(n + 1, np.int32)
    if n:
        np.cumsum(np.fromiter((len(h.requests) for h in hs), np.int32, n), out=off[1:])
    reqs = np.fromiter(itertools.chain.from_iterable(h.requests for h in hs), np.int64, int(off[n]))
    if not len(reqs):
        reqs = _np_empty(0, np.int64)
    keys = sorted(inst.cost)
    m = len(keys)
    ck = np.array(keys, np.int64) if m else _np_empty(0, np.int64)
    cv = np.fromiter((inst.cost[k] for k in keys), np.int64, m) if m else _np_empty(0, np.int64)
    return n, ids, mapped, off, reqs, m, ck, cv


def _select(inst: ReclaimInstance, k: int, mode: int, backend: Optional[Backend], device: int):
    b = backend or valve_backend()
    n, ids, mapped, off, reqs, m, ck, cv = _csr(inst)
    out = _arr(C.c_int, max(n, 1))
    nout = C.c_int(0)
    args = [n, _ptr(ids, C.c_int), _ptr(mapped, i64), _ptr(off, C.c_int), _ptr(reqs, i64), m,
            _ptr(ck, i64), _ptr(cv, i64), int(k), mode, _ptr(out, C.c_int), C.byref(nout)]
    if b.device_arg:
        args = [device] + args
    b.check(b.fn("select")(*args))
    return [out[i] for i in range(nout.value)]


def selective_reclaim(inst: ReclaimInstance, k: int, *, backend: Optional[Backend] = None,
                      device: int = 0) -> List[int]:
    """reclaim.hpp:32-35 -- Algorithm 1 (greedy marginal-cost rounds, smallest-id ties)."""
    return _select(inst, k, 0, backend, device)


def fifo_reclaim(inst: ReclaimInstance, k: int, *, backend: Optional[Backend] = None,
                 device: int = 0) -> List[int]:
    """reclaim.hpp:37-38"""
    return _select(inst, k, 1, backend, device)


def oracle_reclaim(inst: ReclaimInstance, k: int, *, backend: Optional[Backend] = None,
                   device: int = 0) -> List[int]:
    """reclaim.hpp:40-42 (exhaustive; <= 20 handles)"""
    return _select(inst, k, 2, backend, device)


def evicted_cost(inst: ReclaimInstance, handle_ids: Sequence[int], *,
                 backend: Optional[Backend] = None, device: int = 0) -> int:
    """reclaim.hpp:28-30"""
    b = backend or valve_backend()
    n, ids, mapped, off, reqs, m, ck, cv = _csr(inst)
    pick = _arr(C.c_int, len(handle_ids))
    for i, h in enumerate(handle_ids):
        pick[i] = int(h)
    out = i64(0)
    args = [n, _ptr(ids, C.c_int), _ptr(off, C.c_int), _ptr(reqs, i64), m, _ptr(ck, i64),
            _ptr(cv, i64), _ptr(pick, C.c_int), len(handle_ids), C.byref(out)]
    if b.device_arg:
        args = [device] + args
    b.check(b.fn("evicted_cost")(*args))
    return out.value


# ------------------------------------------------------------------------------ memory pool

class HandleState:
    """memory.hpp:21"""
    kFree, kOnlineReserved, kOfflineMapped = 0, 1, 2


class MemoryPool:
    """memory.hpp:19-98 on the device (or a CPU checker when `backend` is given)."""

    HandleState = HandleState

    def __init__(self, total_handles: int, handle_size_pages: int, page_size_tokens: int, *,
                 backend: Optional[Backend] = None, config: Optional[dict] = None):
        self._b = backend or valve_backend()
        self._h = C.c_void_p()
        if config is not None:
            if self._b.prefix != "valve_":
                raise InvalidArgument("config= is a device-pool option")
            cfg = PoolConfig()
            self._b.lib.valve_pool_config_default(C.byref(cfg))
            cfg.total_handles, cfg.handle_size_pages = total_handles, handle_size_pages
            cfg.page_size_tokens = page_size_tokens
            for k, v in config.items():
                setattr(cfg, k, v)
            self._b.check(self._b.lib.valve_pool_create_ex(C.byref(cfg), C.byref(self._h)))
        else:
            self._b.check(self._b.fn("pool_create")(total_handles, handle_size_pages,
                                                    page_size_tokens, C.byref(self._h)))
        self._hsz = handle_size_pages
        self._total = total_handles
        self._tok = page_size_tokens

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value:
            self._b.fn("pool_destroy")(h)
            self._h = C.c_void_p()

    close = __del__

    @property
    def handle(self):
        return self._h

    def _f(self, name, *args):
        self._b.check(self._b.fn(name)(self._h, *args))

    def _counts(self):
        out = _arr(i64, 5)
        self._f("pool_counts", _ptr(out, i64))
        return [out[i] for i in range(5)]

    # memory.hpp:25-41
    def total_handles(self) -> int:
        return self._total

    def handle_size_pages(self) -> int:
        return self._hsz

    def page_size_tokens(self) -> int:
        return self._tok

    def free_handles(self) -> int:
        return self._counts()[0]

    def online_handles(self) -> int:
        return self._counts()[1]

    def offline_handles(self) -> int:
        return self._counts()[2]

    def quarantine_page_id(self) -> int:
        return self._total * self._hsz

    def online_used_pages(self) -> int:
        return self._counts()[3]

    def online_capacity_pages(self) -> int:
        return self._counts()[4]

    # memory.hpp:43-59
    def online_grow(self, k: int, t: int) -> None:
        self._f("pool_online_grow", int(k), int(t))

    def online_release(self, k: int) -> int:
        r = C.c_int(0)
        self._f("pool_online_release", int(k), C.byref(r))
        return r.value

    def online_use_pages(self, n: int) -> None:
        self._f("pool_online_use_pages", int(n))

    def online_free_pages(self, n: int) -> None:
        self._f("pool_online_free_pages", int(n))

    def offline_reserve(self, req: int, pages: int, t: int, max_offline_handles: int = -1) -> bool:
        ok = C.c_int(0)
        self._f("pool_offline_reserve", int(req), int(pages), int(t), int(max_offline_handles),
                C.byref(ok))
        return bool(ok.value)

    def offline_release(self, req: int) -> None:
        self._f("pool_offline_release", int(req))

    def requests_on_handle(self, handle: int) -> List[int]:
        n = C.c_int(0)
        out = _arr(i64, self._hsz)
        self._f("pool_requests_on_handle", int(handle), _ptr(out, i64), self._hsz, C.byref(n))
        return [out[i] for i in range(n.value)]

    def handles_of_request(self, req: int) -> List[int]:
        n = C.c_int(0)
        out = _arr(C.c_int, self._total)
        self._f("pool_handles_of_request", int(req), _ptr(out, C.c_int), self._total, C.byref(n))
        return [out[i] for i in range(n.value)]

    def offline_pages_of(self, req: int) -> int:
        r = C.c_int(0)
        self._f("pool_offline_pages_of", int(req), C.byref(r))
        return r.value

    def snapshot(self) -> ReclaimInstance:
        """memory.hpp:62 (costs attached by the caller)"""
        nh, nr = C.c_int(0), C.c_int(0)
        self._f("pool_snapshot", None, None, None, None, 0, 0, C.byref(nh), C.byref(nr))
        np = _np()
        ids, mapped = _np_empty(nh.value, np.int32), _np_empty(nh.value, np.int64)
        off, reqs = _np_empty(nh.value + 1, np.int32), _np_empty(nr.value, np.int64)
        self._f("pool_snapshot", _ptr(ids, C.c_int), _ptr(mapped, i64), _ptr(off, C.c_int),
                _ptr(reqs, i64), nh.value, nr.value, C.byref(nh), C.byref(nr))
        n = nh.value
        idl, mp, of, rq = ids[:n].tolist(), mapped[:n].tolist(), off[:n + 1].tolist(), reqs[:nr.value].tolist()
        inst = ReclaimInstance()
        inst.handles = [ReclaimHandle(idl[i], mp[i], rq[of[i]:of[i + 1]]) for i in range(n)]
        return inst

    def apply_reclaim(self, handle_ids: Sequence[int], t: int) -> ReclaimResult:
        """memory.hpp:69-71"""
        np = _np()
        k = len(handle_ids)
        ids = np.array([int(h) for h in handle_ids], np.int32) if k else _np_empty(0, np.int32)
        cap_pages = self._total * self._hsz
        cap_ev = max(cap_pages, 1)
        hs = _np_empty(max(k, self._total), np.int32)
        ev, off = _np_empty(cap_ev, np.int64), _np_empty(cap_ev + 1, np.int32)
        pg, ph, bl = _np_empty(cap_pages, np.int64), _np_empty(cap_pages, np.int32), _np_empty(cap_pages, np.int32)
        nh, ne, npg = C.c_int(0), C.c_int(0), C.c_int(0)
        self._f("pool_apply_reclaim", _ptr(ids, C.c_int), k, int(t), _ptr(hs, C.c_int),
                C.byref(nh), _ptr(ev, i64), C.byref(ne), _ptr(off, C.c_int), _ptr(pg, i64),
                _ptr(ph, C.c_int), _ptr(bl, C.c_int), cap_ev, cap_pages, C.byref(npg))
        return _result(hs, nh.value, ev, ne.value, off, pg, ph, bl)

    def handle_state(self, handle: int) -> int:
        r = C.c_int(0)
        self._f("pool_handle_state", int(handle), C.byref(r))
        return r.value

    def handle_mapped_at(self, handle: int) -> int:
        r = i64(0)
        self._f("pool_handle_mapped_at", int(handle), C.byref(r))
        return r.value

    def check_invariants(self) -> None:
        self._f("pool_check_invariants")

    def block_table(self, req: int) -> List[int]:
        """Physical page of every block of a live request (B200 addition)."""
        n = C.c_int(0)
        cap = self._total * self._hsz
        out = _arr(C.c_int, cap)
        self._f("pool_block_table", int(req), _ptr(out, C.c_int), cap, C.byref(n))
        return [out[i] for i in range(n.value)]


def _result(hs, nh, ev, ne, off, pg, ph, bl) -> ReclaimResult:
    np = _np()

    def lst(a, n):
        a = a if isinstance(a, np.ndarray) else np.ctypeslib.as_array(a)
        return a[:n].tolist()

    evl, ofl = lst(ev, ne), lst(off, ne + 1)
    npg = ofl[ne] if ne else 0
    pgl, phl, bll = lst(pg, npg), lst(ph, npg), lst(bl, npg)
    res = ReclaimResult(lst(hs, nh), evl, {}, {}, {})
    for i, req in enumerate(evl):
        a, b = ofl[i], ofl[i + 1]
        res.invalidated_pages[req] = pgl[a:b]
        res.physical_pages[req] = phl[a:b]
        res.block_index[req] = bll[a:b]
    return res


# ------------------------------------------------------------------ reservation controller

@dataclass
class ReservationParams:
    """memory.hpp:103-114"""
    alpha: float = 1.5
    beta: float = 2.0
    t_init_us: int = 1_000_000
    delta_us: int = 100_000
    t_min_us: int = 100_000
    t_max_us: int = 60_000_000
    window_us: int = 60_000_000
    target_per_window: float = 1.0
    h_min: int = 1
    pressure_threshold: float = 0.9

    def _c(self):
        return _ResParams(self.alpha, self.beta, self.t_init_us, self.delta_us, self.t_min_us,
                          self.t_max_us, self.window_us, self.target_per_window, self.h_min,
                          self.pressure_threshold)


class ReservationController:
    """memory.hpp:116-146 (host control plane)."""

    def __init__(self, p: Optional[ReservationParams] = None, *, backend: Optional[Backend] = None):
        self._b = backend or valve_backend()
        self._p = p or ReservationParams()
        self._h = C.c_void_p()
        cp = self._p._c()
        self._b.check(self._b.fn("resctl_create")(C.byref(cp), C.byref(self._h)))

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value:
            self._b.fn("resctl_destroy")(h)
            self._h = C.c_void_p()

    def params(self) -> ReservationParams:
        return self._p

    def interval(self) -> int:
        return self._b.fn("resctl_interval")(self._h)

    def pressure_events(self) -> int:
        return self._b.fn("resctl_pressure_events")(self._h)

    def grow_target(self, h: int, cap: int) -> int:
        return self._b.fn("resctl_grow_target")(self._h, h, cap)

    def record_pressure(self, t: int) -> None:
        self._b.fn("resctl_record_pressure")(self._h, t)

    def release_due(self, t: int, h: int) -> bool:
        return bool(self._b.fn("resctl_release_due")(self._h, t, h))

    def note_tick(self, t: int) -> None:
        self._b.fn("resctl_note_tick")(self._h, t)

    def window_tick(self, t: int) -> int:
        return self._b.fn("resctl_window_tick")(self._h, t)

    def pressure_in_window(self, t: int) -> int:
        return self._b.fn("resctl_pressure_in_window")(self._h, t)


# ------------------------------------------------------------------------ channel control

class ChannelLog:
    """channel.hpp:17-24"""
    kDisableIssued, kDisabled, kEnableIssued, kEnabled, kCooldownScheduled, kCooldownCancelled = range(6)


@dataclass
class CooldownPolicy:
    """channel.hpp:12-15: T_cool = 2 G"""
    max_gap_us: int = 0

    def cooldown_us(self) -> int:
        return 2 * self.max_gap_us


@dataclass
class Hooks:
    """channel.hpp:34-40"""
    schedule: Optional[Callable[[int, int, bool], None]] = None
    on_disabled: Optional[Callable[[int], None]] = None
    on_enabled: Optional[Callable[[int], None]] = None
    log: Optional[Callable[[int, int, int, bool], None]] = None


class ChannelController:
    """channel.hpp:30-80.  With `gate=` the disable/enable edges also raise/release the
    device gate (valve_channel_bind_gate)."""

    kEnabled, kDisabling, kDisabled, kEnabling = range(4)

    def __init__(self, toggle_us: int, cooldown_us: int, hooks: Optional[Hooks] = None, *,
                 backend: Optional[Backend] = None, gate=None, gate_stream: Optional[int] = None):
        self._b = backend or valve_backend()
        hk = hooks or Hooks()
        self._cbs = (
            _SCHED((lambda u, w, g, cd: hk.schedule(w, g, bool(cd))) if hk.schedule else (lambda *a: None)),
            _ONT((lambda u, t: hk.on_disabled(t)) if hk.on_disabled else (lambda *a: None)),
            _ONT((lambda u, t: hk.on_enabled(t)) if hk.on_enabled else (lambda *a: None)),
            _LOG((lambda u, t, w, a, m: hk.log(t, w, a, bool(m))) if hk.log else (lambda *a: None)),
        )
        self._hooks = _Hooks(None, *self._cbs)
        self._h = C.c_void_p()
        self._b.check(self._b.fn("channel_create")(int(toggle_us), int(cooldown_us),
                                                   C.byref(self._hooks), C.byref(self._h)))
        self._gate = None
        if gate is not None:
            # gate_stream: the stream the raise/release stores go on -- the online stream, so a
            # wait_quiesced enqueued there afterwards is ordered behind the raise
            self._b.check(self._b.lib.valve_channel_bind_gate_stream(
                self._h, gate.handle, C.c_void_p(gate_stream) if gate_stream else None))
            self._gate = gate

    def _gate_check(self):
        # a failed device-gate store surfaces here (the transitions return void, channel.hpp)
        if self._gate is not None:
            self._b.check(self._b.lib.valve_channel_gate_status(self._h))

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value:
            self._b.fn("channel_destroy")(h)
            self._h = C.c_void_p()

    def state(self) -> int:
        return self._b.fn("channel_state")(self._h)

    def offline_compute_allowed(self) -> bool:
        return bool(self._b.fn("channel_offline_compute_allowed")(self._h))

    def disables_issued(self) -> int:
        return self._b.fn("channel_disables_issued")(self._h)

    def pending_effective(self) -> int:
        return self._b.fn("channel_pending_effective")(self._h)

    def note_busy(self, t: int) -> None:
        self._b.fn("channel_note_busy")(self._h, int(t))
        self._gate_check()

    def note_all_idle(self, t: int) -> None:
        self._b.fn("channel_note_all_idle")(self._h, int(t))

    def ensure_disabled(self, t: int) -> int:
        e = self._b.fn("channel_ensure_disabled")(self._h, int(t))
        self._gate_check()
        return e

    def handle_toggle(self, t: int, gen: int) -> None:
        self._b.fn("channel_handle_toggle")(self._h, int(t), int(gen))
        self._gate_check()

    def handle_cooldown(self, t: int, gen: int) -> None:
        self._b.fn("channel_handle_cooldown")(self._h, int(t), int(gen))
        self._gate_check()


# ----------------------------------------------------------- device-only (B200) surfaces

class PoolConfig(C.Structure):
    _fields_ = [("device", C.c_int), ("total_handles", C.c_int), ("handle_size_pages", C.c_int),
                ("page_size_tokens", C.c_int), ("slot_bytes", i64), ("page_bytes", i64),
                ("max_requests", C.c_int), ("max_pages_per_request", C.c_int)]


class CopyParams(C.Structure):
    _fields_ = [("ctas", C.c_int), ("threads", C.c_int), ("chunk_bytes", i64),
                ("rate_bytes_per_s", dbl), ("burst_bytes", i64), ("use_tma", C.c_int),
                ("trace", C.c_void_p)]


class CopyStats(C.Structure):
    _fields_ = [("bytes", i64), ("pages", i64), ("kernel_ms", dbl), ("t_first_ns", C.c_uint64),
                ("t_last_ns", C.c_uint64)]


class GateState(C.Structure):
    _fields_ = [("gen", u32), ("closed", u32), ("quiesced_gen", u32), ("live_ctas", u32),
                ("t_first_seen_ns", C.c_uint64), ("t_quiesced_ns", C.c_uint64),
                ("tiles_done", C.c_uint64), ("canary_hits", C.c_uint64),
                ("tiles_claimed", C.c_uint64), ("t_raise_ns", C.c_uint64), ("total_tiles", C.c_uint64)]


class OfflineWork(C.Structure):
    _fields_ = [("rows", C.c_void_p), ("npages", C.c_void_p), ("n_requests", C.c_int),
                ("total_tiles", i64), ("out", C.c_void_p), ("ctas", C.c_int), ("threads", C.c_int),
                ("poll", C.c_int), ("tile_bytes", i64)]


class OfflineGemmWork(C.Structure):
    _fields_ = [("a", C.c_void_p), ("b", C.c_void_p), ("c", C.c_void_p), ("m", C.c_int), ("n", C.c_int),
                ("k", C.c_int), ("ctas", C.c_int), ("poll", C.c_int), ("fresh", C.c_int), ("mode", C.c_int)]


class PoolView(C.Structure):
    _fields_ = [("pages", C.c_void_p), ("block_tables", C.c_void_p), ("slot_bytes", i64),
                ("page_bytes", i64), ("max_pages_per_request", C.c_int),
                ("quarantine_page", C.c_int), ("stream", C.c_void_p)]


def _declare_valve_extras(L):
    vp = C.c_void_p
    sig = {
        "valve_kernel_launches": (i64, []),
        "valve_pool_config_default": (None, [P(PoolConfig)]),
        "valve_pool_create_ex": (C.c_int, [P(PoolConfig), P(vp)]),
        "valve_pool_set_costs": (C.c_int, [vp, C.c_int, P(i64), P(i64)]),
        "valve_pool_reclaim": (C.c_int, [vp, C.c_int, C.c_int, i64, P(C.c_int), P(C.c_int), P(C.c_int)]),
        "valve_pool_last_reclaim": (C.c_int, [vp, P(C.c_int), P(i64), P(C.c_int), P(i64), P(C.c_int),
                                              P(C.c_int), C.c_int, C.c_int, C.c_int]),
        "valve_copy_params_default": (None, [P(CopyParams)]),
        "valve_pool_reclaim_copy": (C.c_int, [vp, vp, i64, P(CopyParams), P(CopyStats)]),
        "valve_pool_reclaim_copy_ce": (C.c_int, [vp, vp, i64, P(CopyStats)]),
        "valve_pool_reclaim_copy_start": (C.c_int, [vp, vp, i64, P(CopyParams)]),
        "valve_pool_reclaim_copy_wait": (C.c_int, [vp, P(CopyStats)]),
        "valve_pool_reset": (C.c_int, [vp]),
        "valve_pool_online_handles": (C.c_int, [vp, P(C.c_int), C.c_int, P(C.c_int)]),
        "valve_pool_copy_ticket": (C.c_int, [vp, P(C.c_uint64), P(C.c_int), P(i64)]),
        "valve_pool_wait_landed": (C.c_int, [vp, C.c_uint64, vp]),
        "valve_pool_landed": (C.c_int, [vp, P(C.c_uint64), P(C.c_uint64)]),
        "valve_pool_reclaim_phases": (C.c_int, [vp, P(i64)]),
        "valve_pool_restore": (C.c_int, [vp, i64, vp, C.c_int, P(C.c_int), P(CopyParams), P(CopyStats)]),
        "valve_pool_set_page_bytes": (C.c_int, [vp, C.c_int, P(i64), P(i64)]),
        "valve_pool_last_copy_layout": (C.c_int, [vp, P(i64), C.c_int, P(i64)]),
        "valve_host_alloc": (C.c_int, [i64, P(vp)]),
        "valve_host_free": (None, [vp]),
        "valve_pool_fill_pages": (C.c_int, [vp]),
        "valve_pool_view_get": (C.c_int, [vp, P(PoolView)]),
        "valve_pool_request_row": (C.c_int, [vp, i64, P(C.c_int)]),
        "valve_gate_create": (C.c_int, [C.c_int, P(vp)]),
        "valve_gate_destroy": (None, [vp]),
        "valve_gate_raise": (C.c_int, [vp, u32, vp]),
        "valve_gate_release": (C.c_int, [vp, u32, vp]),
        "valve_gate_raise_stamped": (C.c_int, [vp, u32, vp]),
        "valve_gate_wait_quiesced": (C.c_int, [vp, u32, vp]),
        "valve_gate_wait_closed_quiesced": (C.c_int, [vp, vp]),
        "valve_gate_attach_peers": (C.c_int, [vp, P(vp), C.c_int]),
        "valve_gate_set_fanout": (C.c_int, [vp, C.c_int]),
        "valve_gate_export": (C.c_int, [vp, C.c_char_p]),
        "valve_gate_open_remote": (C.c_int, [C.c_int, C.c_char_p, P(vp)]),
        "valve_gate_read": (C.c_int, [vp, P(GateState)]),
        "valve_gate_stream": (vp, [vp]),
        "valve_offline_launch": (C.c_int, [vp, vp, P(OfflineWork), vp]),
        "valve_offline_reset": (C.c_int, [vp]),
        "valve_offline_cancel": (C.c_int, [vp]),
        "valve_offline_gemm": (C.c_int, [vp, P(OfflineGemmWork), vp]),
        "valve_channel_bind_gate": (C.c_int, [vp, vp]),
        "valve_channel_bind_gate_stream": (C.c_int, [vp, vp, vp]),
        "valve_channel_gate_status": (C.c_int, [vp]),
    }
    for name, (res, args) in sig.items():
        f = getattr(L, name)
        f.restype = res
        f.argtypes = args


def kernel_launches() -> int:
    """CUDA kernels launched by libvalve in this process."""
    return valve_backend().lib.valve_kernel_launches()


class DevicePool(MemoryPool):
    """MemoryPool with a physical page store and the fused device reclaim + copy path."""

    def __init__(self, total_handles: int, handle_size_pages: int, page_size_tokens: int, *,
                 device: int = 0, slot_bytes: int = 0, page_bytes: int = 0,
                 max_requests: int = 4096, max_pages_per_request: int = 4096):
        super().__init__(total_handles, handle_size_pages, page_size_tokens,
                         config=dict(device=device, slot_bytes=slot_bytes, page_bytes=page_bytes,
                                     max_requests=max_requests,
                                     max_pages_per_request=max_pages_per_request))
        self.device = device
        self.slot_bytes = slot_bytes
        self.page_bytes = page_bytes

    def set_costs(self, costs: Dict[int, int]) -> None:
        n = len(costs)
        rq, cv = _arr(i64, n), _arr(i64, n)
        for i, (r, c) in enumerate(costs.items()):
            rq[i], cv[i] = int(r), int(c)
        self._b.check(self._b.lib.valve_pool_set_costs(self._h, n, _ptr(rq, i64), _ptr(cv, i64)))

    def apply_reclaim(self, handle_ids: Sequence[int], t: int) -> ReclaimResult:
        res = super().apply_reclaim(handle_ids, t)
        self._last = (len(res.handles), len(res.evicted_requests),
                      sum(len(v) for v in res.invalidated_pages.values()))
        return res

    def set_page_bytes(self, sizes: Dict[int, int]) -> None:
        """Per-request page size (0 = the pool's page_bytes), e.g. whole-slot weight pages (C3)."""
        n = len(sizes)
        rq, bv = _arr(i64, n), _arr(i64, n)
        for i, (r, b) in enumerate(sizes.items()):
            rq[i], bv[i] = int(r), int(b)
        self._b.check(self._b.lib.valve_pool_set_page_bytes(self._h, n, _ptr(rq, i64), _ptr(bv, i64)))

    def last_copy_layout(self):
        """(total destination bytes, page size of each evicted request in report order) of the
        last apply_reclaim / reclaim: the copy writes request e's pages after those of e' < e."""
        ne = self._last[1] if getattr(self, "_last", None) else 0
        pb, tot = _arr(i64, max(ne, 1)), C.c_int64(0)
        self._b.check(self._b.lib.valve_pool_last_copy_layout(self._h, _ptr(pb, i64), ne, C.byref(tot)))
        return tot.value, [pb[i] for i in range(ne)]

    def reclaim(self, k: int, t: int, mode: int = 0):
        """Fused snapshot -> select -> apply on the device; returns (n_handles, n_evicted, n_pages)."""
        a, b, c = C.c_int(0), C.c_int(0), C.c_int(0)
        self._b.check(self._b.lib.valve_pool_reclaim(self._h, int(k), int(mode), int(t),
                                                     C.byref(a), C.byref(b), C.byref(c)))
        self._last = (a.value, b.value, c.value)
        return self._last

    def last_reclaim(self) -> ReclaimResult:
        """Full result of the last reclaim() (device -> host)."""
        nh, ne, npg = self._last
        hs, ev, off = _arr(C.c_int, nh), _arr(i64, ne), _arr(C.c_int, ne + 1)
        pg, ph, bl = _arr(i64, npg), _arr(C.c_int, npg), _arr(C.c_int, npg)
        self._b.check(self._b.lib.valve_pool_last_reclaim(
            self._h, _ptr(hs, C.c_int), _ptr(ev, i64), _ptr(off, C.c_int), _ptr(pg, i64),
            _ptr(ph, C.c_int), _ptr(bl, C.c_int), nh, ne, npg))
        return _result(hs, nh, ev, ne, off, pg, ph, bl)

    def fill_pages(self) -> None:
        self._b.check(self._b.lib.valve_pool_fill_pages(self._h))

    def reclaim_copy(self, host_ptr: int, nbytes: int, params: Optional[CopyParams] = None,
                     engine: str = "sm") -> CopyStats:
        st = CopyStats()
        if engine == "ce":
            self._b.check(self._b.lib.valve_pool_reclaim_copy_ce(self._h, C.c_void_p(host_ptr),
                                                                 int(nbytes), C.byref(st)))
        else:
            self._b.check(self._b.lib.valve_pool_reclaim_copy(
                self._h, C.c_void_p(host_ptr), int(nbytes),
                C.byref(params) if params is not None else None, C.byref(st)))
        return st

    def reclaim_copy_start(self, host_ptr: int, nbytes: int, params: Optional[CopyParams] = None):
        """Start the gather copy of the last reclaim's report asynchronously.  The copy works from
        its own snapshot of the report, so bookkeeping calls and the next reclaim / apply_reclaim
        overlap it; up to two copies may be in flight (valve_pool_reclaim_copy_start)."""
        self._b.check(self._b.lib.valve_pool_reclaim_copy_start(
            self._h, C.c_void_p(host_ptr), int(nbytes), C.byref(params) if params is not None else None))

    def reclaim_copy_wait(self) -> CopyStats:
        """Complete the oldest copy in flight (FIFO) and return its stats."""
        st = CopyStats()
        self._b.check(self._b.lib.valve_pool_reclaim_copy_wait(self._h, C.byref(st)))
        return st

    def reset(self) -> None:
        """Back to the freshly created state, keeping the allocation (valve_pool_reset)."""
        self._b.check(self._b.lib.valve_pool_reset(self._h))
        self._last = (0, 0, 0)

    def online_handle_ids(self) -> List[int]:
        """Online-reserved handle ids, ascending (valve_pool_online_handles)."""
        out, n = _arr(C.c_int, self._total), C.c_int(0)
        self._b.check(self._b.lib.valve_pool_online_handles(self._h, _ptr(out, C.c_int), self._total, C.byref(n)))
        return [out[i] for i in range(n.value)]

    def copy_ticket(self):
        """(wave_base, n_waves, wave_bytes) of the last started copy: wave w of it covers slot
        bytes [w*wave_bytes, (w+1)*wave_bytes) of every reclaimed page and is out once
        landed() >= wave_base + w + 1 (valve_pool_copy_ticket)."""
        b, n, wb = C.c_uint64(0), C.c_int(0), C.c_int64(0)
        self._b.check(self._b.lib.valve_pool_copy_ticket(self._h, C.byref(b), C.byref(n), C.byref(wb)))
        return b.value, n.value, wb.value

    def wait_landed(self, ticket: int, stream: Optional[int] = None):
        """Stream-ordered wait (cuStreamWaitValue64 >=) for `ticket` published copy waves."""
        self._b.check(self._b.lib.valve_pool_wait_landed(self._h, int(ticket),
                                                         C.c_void_p(stream) if stream else None))

    def landed(self):
        """(published waves, issued waves)."""
        a, b = C.c_uint64(0), C.c_uint64(0)
        self._b.check(self._b.lib.valve_pool_landed(self._h, C.byref(a), C.byref(b)))
        return a.value, b.value

    def restore(self, req: int, host_ptr: int, blocks: Sequence[int],
                params: Optional[CopyParams] = None) -> CopyStats:
        """Scatter host pages back into `req`'s slots: host page i -> block blocks[i]
        (the inverse of reclaim_copy for a request re-reserved after eviction)."""
        n = len(blocks)
        b = _arr(C.c_int, n)
        for i, x in enumerate(blocks):
            b[i] = int(x)
        st = CopyStats()
        self._b.check(self._b.lib.valve_pool_restore(
            self._h, int(req), C.c_void_p(host_ptr), n, _ptr(b, C.c_int),
            C.byref(params) if params is not None else None, C.byref(st)))
        return st

    def reclaim_phases_us(self):
        """(instance, select, apply) device microseconds of the last reclaim()."""
        out = _arr(i64, 16)
        self._b.check(self._b.lib.valve_pool_reclaim_phases(self._h, _ptr(out, i64)))
        return out[0] / 1e3, out[1] / 1e3, out[2] / 1e3

    def view(self) -> PoolView:
        v = PoolView()
        self._b.check(self._b.lib.valve_pool_view_get(self._h, C.byref(v)))
        return v

    def request_row(self, req: int) -> int:
        r = C.c_int(0)
        self._b.check(self._b.lib.valve_pool_request_row(self._h, int(req), C.byref(r)))
        return r.value


class HostBuffer:
    """Pinned, device-mapped host memory (valve_host_alloc) -- the reclaim destination."""

    def __init__(self, nbytes: int):
        self._b = valve_backend()
        self.nbytes = int(nbytes)
        self._p = C.c_void_p()
        self._b.check(self._b.lib.valve_host_alloc(self.nbytes, C.byref(self._p)))

    @property
    def ptr(self) -> int:
        return self._p.value

    def view(self):
        """numpy uint8 view (no copy)."""
        import numpy as np

        return np.ctypeslib.as_array((C.c_uint8 * self.nbytes).from_address(self.ptr))

    def __del__(self):
        p = getattr(self, "_p", None)
        if p is not None and p.value:
            self._b.lib.valve_host_free(p)
            self._p = C.c_void_p()


def copy_params(**kw) -> CopyParams:
    c = CopyParams()
    valve_backend().lib.valve_copy_params_default(C.byref(c))
    for k, v in kw.items():
        setattr(c, k, v)
    return c


class Gate:
    """Device preemption gate (valve_gate_*)."""

    HANDLE_BYTES = 64

    def __init__(self, device: int = 0, _remote_handle: Optional[bytes] = None):
        self._b = valve_backend()
        self._h = C.c_void_p()
        self.device = device
        self._peers = []
        if _remote_handle is not None:
            self._b.check(self._b.lib.valve_gate_open_remote(device, _remote_handle, C.byref(self._h)))
        else:
            self._b.check(self._b.lib.valve_gate_create(device, C.byref(self._h)))

    @classmethod
    def open_remote(cls, handle: bytes, device: int = 0) -> "Gate":
        """A TP member's gate words exported by another process (CUDA IPC)."""
        return cls(device, _remote_handle=bytes(handle))

    def export(self) -> bytes:
        buf = C.create_string_buffer(self.HANDLE_BYTES)
        self._b.check(self._b.lib.valve_gate_export(self._h, buf))
        return buf.raw

    FANOUT_BATCHED, FANOUT_STREAMS = 0, 1

    def set_fanout(self, mode: int):
        """Leader's ack wait: FANOUT_BATCHED (one memop submission, default) or FANOUT_STREAMS."""
        self._b.check(self._b.lib.valve_gate_set_fanout(self._h, int(mode)))

    def attach_peers(self, members: Sequence["Gate"]):
        """TP fan-out: raise/release/wait on this (leader) gate also drive the members' words."""
        arr = (C.c_void_p * max(1, len(members)))(*[m.handle.value for m in members])
        self._b.check(self._b.lib.valve_gate_attach_peers(self._h, arr, len(members)))
        self._peers.extend(members)  # keep the member objects alive

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value:
            self._b.lib.valve_gate_destroy(h)
            self._h = C.c_void_p()

    @property
    def handle(self):
        return self._h

    @property
    def stream(self) -> int:
        return self._b.lib.valve_gate_stream(self._h)

    def raise_(self, gen: int, stream: Optional[int] = None):
        self._b.check(self._b.lib.valve_gate_raise(self._h, gen, C.c_void_p(stream) if stream else None))

    def raise_stamped(self, gen: int, stream: Optional[int] = None):
        self._b.check(self._b.lib.valve_gate_raise_stamped(self._h, gen,
                                                           C.c_void_p(stream) if stream else None))

    def release(self, gen: int, stream: Optional[int] = None):
        self._b.check(self._b.lib.valve_gate_release(self._h, gen, C.c_void_p(stream) if stream else None))

    def wait_quiesced(self, gen: int, stream: Optional[int] = None):
        self._b.check(self._b.lib.valve_gate_wait_quiesced(self._h, gen,
                                                           C.c_void_p(stream) if stream else None))

    def wait_closed_quiesced(self, stream: Optional[int] = None):
        """TP member: `stream` waits for the leader's raise to land here and this GPU's gated
        CTAs to retire (valve_gate_wait_closed_quiesced)."""
        self._b.check(self._b.lib.valve_gate_wait_closed_quiesced(self._h, C.c_void_p(stream) if stream else None))

    def read(self) -> GateState:
        s = GateState()
        self._b.check(self._b.lib.valve_gate_read(self._h, C.byref(s)))
        return s

    def reset_work(self):
        self._b.check(self._b.lib.valve_offline_reset(self._h))

    def cancel_work(self):
        """Drop the rest of the work list: queued / resumed launches retire at once."""
        self._b.check(self._b.lib.valve_offline_cancel(self._h))

    def launch_gemm(self, a_ptr: int, b_ptr: int, c_ptr: int, m: int, n: int, k: int, *, ctas: int = 0,
                    poll: bool = True, stream: Optional[int] = None, fresh: bool = False, mode: int = 0):
        """Gated tcgen05 GEMM C[m,n] = A[m,k] B[n,k]^T (bf16, device pointers), preemptible at
        128x256-tile granularity (valve_offline_gemm).  fresh=True starts a new work list
        (stream-ordered cursor reset); otherwise the launch resumes from the gate's cursors.
        mode: 0 auto (CTA pairs when m % 256 == 0), 1 single-CTA 128x256 tiles, 2 CTA pairs
        (tcgen05 cta_group::2 on 256x256 tiles)."""
        w = OfflineGemmWork(a_ptr, b_ptr, c_ptr, m, n, k, ctas, 1 if poll else 0, 1 if fresh else 0, mode)
        self._b.check(self._b.lib.valve_offline_gemm(self._h, C.byref(w),
                                                     C.c_void_p(stream) if stream else None))

    def launch_offline(self, pool: DevicePool, rows_ptr: Optional[int], npages_ptr: Optional[int],
                       n_requests: int, total_tiles: int, out_ptr: Optional[int], *, ctas: int = 0,
                       threads: int = 0, poll: bool = True, stream: Optional[int] = None,
                       tile_bytes: int = 0):
        """rows_ptr=None decodes every request row of the pool; out_ptr=None drops results."""
        w = OfflineWork(rows_ptr, npages_ptr, n_requests, total_tiles, out_ptr, ctas, threads,
                        1 if poll else 0, tile_bytes)
        self._b.check(self._b.lib.valve_offline_launch(self._h, pool.handle, C.byref(w),
                                                       C.c_void_p(stream) if stream else None))
