"""Differential drivers: the same call sequence against two implementations of the reference
API (device vs C restatement vs the reference itself), compared call by call.

Every call's outcome is (exception class name | return value); pool state is compared through
the public API only.  `extended=True` also compares what only the device and the C
restatement model: physical pages and block indices of invalidated pages, block tables.
"""
import random

from paper_2604_07874_b200 import api as A


def outcome(fn, *args):
    try:
        return ("ok", fn(*args))
    except A.LogicError as e:  # includes InvalidArgument / OutOfRange
        return (type(e).__name__, None)
    except A.ValveRuntimeError as e:
        return ("RuntimeError", str(e))


def result_tuple(res, extended):
    if not isinstance(res, A.ReclaimResult):
        return res
    base = (res.handles, res.evicted_requests, sorted(res.invalidated_pages.items()))
    if extended:
        base += (sorted(res.physical_pages.items()), sorted(res.block_index.items()))
    return base


class PoolPair:
    """Two pools driven in lockstep."""

    def __init__(self, H, S, T, backend_a, backend_b, extended=False):
        self.a = A.MemoryPool(H, S, T, backend=backend_a)
        self.b = A.MemoryPool(H, S, T, backend=backend_b)
        self.H, self.S = H, S
        self.extended = extended
        self.log = []

    def call(self, name, *args):
        ra = outcome(getattr(self.a, name), *args)
        rb = outcome(getattr(self.b, name), *args)
        ra = (ra[0], result_tuple(ra[1], self.extended))
        rb = (rb[0], result_tuple(rb[1], self.extended))
        self.log.append((name, args))
        assert ra == rb, f"{name}{args}: {ra} != {rb}\nafter {self.log[-20:]}"
        return ra

    def state(self):
        for fn in ("free_handles", "online_handles", "offline_handles", "online_used_pages",
                   "online_capacity_pages"):
            self.call(fn)
        self.call("snapshot_tuple")


def _snap(pool):
    inst = pool.snapshot()
    return [(h.id, h.mapped_at, list(h.requests)) for h in inst.handles]


A.MemoryPool.snapshot_tuple = _snap  # comparison helper (not part of the API)


def random_pool_ops(pair: PoolPair, rng: random.Random, n_ops: int, live_cap: int = 64):
    H, S = pair.H, pair.S
    live = []
    next_req = 0
    t = 0
    for _ in range(n_ops):
        t += rng.randint(0, 50)
        r = rng.random()
        if r < 0.30:
            if live and rng.random() < 0.1:
                req = rng.choice(live)  # second reservation of a live request
            else:
                req = next_req + rng.choice([0, 0, 0, 1000, -7])
                next_req += 1
            pages = rng.choice([0, 1, 2, S - 1, S, S + 1, 2 * S + 3, rng.randint(1, 3 * S)])
            cap = rng.choice([-1, -1, -1, rng.randint(0, H)])
            ok = pair.call("offline_reserve", req, pages, t, cap)
            if ok == ("ok", True) and pages > 0 and req not in live and len(live) < live_cap:
                live.append(req)
        elif r < 0.45:
            if live:
                req = live.pop(rng.randrange(len(live)))
            else:
                req = rng.randint(0, 50)
            pair.call("offline_release", req)
        elif r < 0.52:
            pair.call("online_grow", rng.choice([0, 1, 2, rng.randint(-1, H)]), t)
        elif r < 0.58:
            pair.call("online_release", rng.choice([0, 1, 2, rng.randint(-1, H)]))
        elif r < 0.64:
            pair.call("online_use_pages", rng.choice([0, 1, S, rng.randint(-1, 2 * S)]))
        elif r < 0.68:
            pair.call("online_free_pages", rng.choice([0, 1, S, rng.randint(-1, 2 * S)]))
        elif r < 0.80:
            snap = pair.a.snapshot()
            ids = [h.id for h in snap.handles]
            k = rng.randint(0, min(len(ids), 4))
            pick = rng.sample(ids, k) if ids else []
            if rng.random() < 0.1:
                pick.append(rng.choice([-1, H, rng.randrange(H)] + pick))
            res = pair.call("apply_reclaim", pick, t)
            if res[0] == "ok":
                for req in res[1][1]:
                    if req in live:
                        live.remove(req)
        elif r < 0.84:
            pair.call("requests_on_handle", rng.randint(-1, H))
        elif r < 0.88:
            pair.call("handles_of_request", rng.choice(live) if live else rng.randint(0, 9))
        elif r < 0.91:
            pair.call("offline_pages_of", rng.choice(live) if live else rng.randint(0, 9))
        elif r < 0.94:
            h = rng.randint(-1, H)
            pair.call("handle_state", h)
            pair.call("handle_mapped_at", h)
        elif r < 0.97:
            pair.call("check_invariants")
        else:
            pair.state()
        if pair.extended and live and rng.random() < 0.1:
            pair.call("block_table", rng.choice(live))
    pair.state()
    pair.call("check_invariants")


# ------------------------------------------------------------------ selection instances

def random_instance(rng, n_max=12, req_max=8, cost_max=50, allow_dupes=False, ids_shuffled=True):
    n = rng.randint(1, n_max)
    n_req = rng.randint(1, req_max)
    cost = {r: rng.randint(0, cost_max) for r in range(n_req)}
    ids = list(range(n))
    if ids_shuffled:
        ids = rng.sample(range(3 * n + 5), n)
    handles = []
    for h in ids:
        members = sorted(set(rng.randrange(n_req) for _ in range(rng.randint(1, min(n_req, 4)))))
        if allow_dupes and members and rng.random() < 0.2:
            members.append(members[0])
        handles.append(A.ReclaimHandle(h, rng.randint(0, 1000), members))
    return A.ReclaimInstance(handles, cost)
