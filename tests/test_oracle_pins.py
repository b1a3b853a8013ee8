"""Pins the CPU checkers before anything is checked against them (CPU only).

* The Python port of the reference RNG draws the same numbers as the compiled reference.
* The C restatement (oracle/valve_oracle.c) agrees with the reference compiled from
  /root/reference (oracle/_ref) on randomized call sequences: pool ops incl. error paths,
  selection (greedy / fifo / exhaustive), evicted_cost, the MIAD controller and the channel
  state machine.
"""
import ctypes as C
import random

import pytest

import fuzz
from paper_2604_07874_b200 import api as A
from refrng import Rng


def test_rng_port_matches_reference(ref):
    f = ref.lib.vr_rng_draws
    f.restype = None
    f.argtypes = [C.c_uint64, C.c_char_p, C.c_int, C.POINTER(C.c_uint64)]
    for seed, label in [(2024, "reclaim-step-invariant"), (20_240_817, None), (7, "x")]:
        out = (C.c_uint64 * 700)()
        f(seed, label.encode() if label else None, 700, out)
        rng = Rng.substream(seed, label) if label else Rng(seed)
        assert [rng.uniform_int(0, (1 << 63) - 2) for _ in range(700)] == list(out)


@pytest.mark.parametrize("seed", range(24))
def test_pool_ops_oracle_vs_reference(ref, oracle_c, seed):
    rng = random.Random(seed)
    H, S = rng.choice([(4, 4), (8, 4), (16, 4), (6, 3), (32, 8), (12, 64), (64, 16), (128, 64)])
    pair = fuzz.PoolPair(H, S, 16, ref, oracle_c)
    fuzz.random_pool_ops(pair, rng, 400)


@pytest.mark.parametrize("mode", [0, 1, 2])
def test_selection_oracle_vs_reference(ref, oracle_c, mode):
    rng = random.Random(100 + mode)
    for _ in range(300):
        inst = fuzz.random_instance(rng, n_max=12 if mode != 2 else 9, allow_dupes=True)
        if rng.random() < 0.05 and inst.cost:
            inst.cost.pop(next(iter(inst.cost)))
        for k in [0, 1, rng.randint(0, len(inst.handles) + 2)]:
            ra = fuzz.outcome(A._select, inst, k, mode, ref, 0)
            rb = fuzz.outcome(A._select, inst, k, mode, oracle_c, 0)
            assert ra == rb, (inst, k, mode)


def test_evicted_cost_oracle_vs_reference(ref, oracle_c):
    rng = random.Random(7)
    for _ in range(300):
        inst = fuzz.random_instance(rng, allow_dupes=True)
        if rng.random() < 0.1 and inst.cost:
            inst.cost.pop(next(iter(inst.cost)))
        ids = [h.id for h in inst.handles]
        pick = rng.sample(ids, rng.randint(0, len(ids)))
        if rng.random() < 0.1:
            pick.insert(rng.randint(0, len(pick)), 10_000)
        assert fuzz.outcome(lambda: A.evicted_cost(inst, pick, backend=ref)) == \
            fuzz.outcome(lambda: A.evicted_cost(inst, pick, backend=oracle_c))


def _resctl_trace(b, rng):
    p = A.ReservationParams(alpha=rng.choice([1.5, 1.1, 2.7]), beta=rng.choice([2.0, 1.3]),
                            t_init_us=rng.randint(1, 10**6), delta_us=rng.randint(0, 10**5),
                            t_min_us=rng.randint(1, 10**5), t_max_us=10**7,
                            window_us=rng.randint(1, 10**7), target_per_window=rng.choice([1.0, 0.5, 3.0]),
                            h_min=rng.randint(0, 3))
    ctl = A.ReservationController(p, backend=b)
    out, t = [], 0
    r2 = random.Random(rng.random())
    for _ in range(300):
        t += r2.randint(0, 10**6)
        op = r2.random()
        if op < 0.3:
            ctl.record_pressure(t)
        elif op < 0.5:
            out.append(ctl.grow_target(r2.randint(0, 200), r2.randint(0, 300)))
        elif op < 0.7:
            out.append(ctl.release_due(t, r2.randint(0, 5)))
            ctl.note_tick(t)
        elif op < 0.9:
            out.append(ctl.window_tick(t))
        else:
            out.append(ctl.pressure_in_window(t))
    out.append((ctl.interval(), ctl.pressure_events()))
    return out


def test_resctl_oracle_vs_reference(ref, oracle_c):
    for s in range(20):
        assert _resctl_trace(ref, random.Random(s)) == _resctl_trace(oracle_c, random.Random(s))


def _channel_trace(b, seed):
    rng = random.Random(seed)
    events = []
    rec = []
    hooks = A.Hooks(schedule=lambda w, g, cd: (events.append((w, g, cd)), rec.append(("s", w, g, cd))),
                    on_disabled=lambda t: rec.append(("d", t)),
                    on_enabled=lambda t: rec.append(("e", t)),
                    log=lambda t, w, a, m: rec.append(("l", t, w, a, m)))
    ctl = A.ChannelController(rng.choice([0, 50, 1000]), rng.choice([0, 100, 600]), hooks, backend=b)
    t = 0
    for _ in range(200):
        t += rng.randint(0, 700)
        events.sort()
        while events and events[0][0] <= t:
            w, g, cd = events.pop(0)
            (ctl.handle_cooldown if cd else ctl.handle_toggle)(w, g)
        op = rng.random()
        if op < 0.35:
            ctl.note_busy(t)
        elif op < 0.7:
            ctl.note_all_idle(t)
        elif op < 0.85:
            rec.append(("ensure", ctl.ensure_disabled(t)))
        else:
            (ctl.handle_toggle if rng.random() < 0.5 else ctl.handle_cooldown)(t, rng.randint(0, 5))
        rec.append((ctl.state(), ctl.offline_compute_allowed(), ctl.disables_issued(),
                    ctl.pending_effective()))
    return rec


def test_channel_oracle_vs_reference(ref, oracle_c):
    for s in range(30):
        assert _channel_trace(ref, s) == _channel_trace(oracle_c, s)
