"""Device parity (sm_100a kernels via the C ABI) against the pinned checkers.

* pool bookkeeping: randomized call sequences, device vs C restatement, including physical
  pages, block indices and block tables (extended comparison), at reference geometries;
* selection: device vs the reference itself on random instances and on the reference's own
  property tests (test_reclaim.cpp:187-256, acceptance.cpp:313-398 generators, same seeds);
* fused device reclaim (snapshot -> select -> apply in one launch) vs oracle
  snapshot + selective_reclaim + apply_reclaim.
"""
import random

import pytest

import fuzz
from conftest import backend_by_name
from paper_2604_07874_b200 import api as A
from refrng import Rng

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("seed,geom,n_ops", [
    (0, (4, 4), 300), (1, (8, 4), 300), (2, (16, 4), 400), (3, (6, 3), 300),
    (4, (32, 8), 400), (5, (12, 64), 400), (6, (128, 64), 300), (7, (64, 16), 400),
])
def test_pool_ops_device_vs_oracle(oracle_c, seed, geom, n_ops):
    rng = random.Random(1000 + seed)
    H, S = geom
    pair = fuzz.PoolPair(H, S, 16, None, oracle_c, extended=True)
    fuzz.random_pool_ops(pair, rng, n_ops)


def test_pool_ops_device_vs_reference(ref):
    rng = random.Random(77)
    pair = fuzz.PoolPair(16, 4, 16, None, ref)
    fuzz.random_pool_ops(pair, rng, 500)


@pytest.mark.parametrize("mode", [0, 1, 2])
def test_selection_device_vs_reference(ref, mode):
    rng = random.Random(300 + mode)
    for _ in range(200):
        inst = fuzz.random_instance(rng, n_max=14 if mode != 2 else 10, allow_dupes=True,
                                    cost_max=rng.choice([3, 50, 10**12]))
        if rng.random() < 0.05 and inst.cost:
            inst.cost.pop(next(iter(inst.cost)))
        for k in [0, 1, rng.randint(0, len(inst.handles) + 2)]:
            ra = fuzz.outcome(A._select, inst, k, mode, ref, 0)
            rb = fuzz.outcome(A._select, inst, k, mode, None, 0)
            assert ra == rb, (inst, k, mode)


def test_selection_large_instances_device_vs_oracle(oracle_c):
    """B200-scale instances (C2: ~950 handles, ~1500 refs, ~310 requests)."""
    rng = random.Random(5)
    for n, n_req in [(114, 40), (920, 310), (1024, 600), (4096, 2500), (6000, 300)]:
        cost = {r: rng.randint(2000, 4400) for r in range(n_req)}
        handles = [A.ReclaimHandle(h, rng.randint(0, 10**6),
                                   sorted(set(rng.randrange(n_req) for _ in range(rng.randint(1, 3)))))
                   for h in range(n)]
        inst = A.ReclaimInstance(handles, cost)
        for k in (1, 15, 64):
            assert A.selective_reclaim(inst, k) == A.selective_reclaim(inst, k, backend=oracle_c)
            assert A.fifo_reclaim(inst, k) == A.fifo_reclaim(inst, k, backend=oracle_c)


def test_selection_packed_key_boundaries_vs_oracle(oracle_c):
    """The device's packed-key rounds (u32 (marginal << idbits) | index, taken when ids ascend,
    costs >= 0 and marginals fit) against the oracle at their edges: marginals just below and just
    above 2^(32 - idbits), all-equal marginals (pure id tie-breaks), zero costs, and shuffled
    handle order (ids not ascending -> the general path)."""
    rng = random.Random(77)
    for n in (1, 2, 3, 513, 1024, 2048):
        idbits = max(1, (n - 1).bit_length())
        lim = 1 << (32 - idbits)
        for case in ("below", "above", "ties", "zeros", "shuffled"):
            n_req = max(1, n // 2)
            if case == "below":
                cost = {r: rng.randint(lim // 8, lim // 4 - 1) for r in range(n_req)}
            elif case == "above":
                cost = {r: rng.randint(lim // 2, lim) for r in range(n_req)}
            elif case == "ties":
                cost = {r: 7 for r in range(n_req)}
            else:
                cost = {r: (0 if case == "zeros" else rng.randint(0, 5000)) for r in range(n_req)}
            handles = []
            for h in range(n):
                if case == "ties":
                    reqs = [h % n_req]
                else:
                    reqs = sorted(set(rng.randrange(n_req) for _ in range(rng.randint(1, 3))))
                handles.append(A.ReclaimHandle(h * 3 + 1, rng.randint(0, 10**6), reqs))
            if case == "shuffled":
                rng.shuffle(handles)
            inst = A.ReclaimInstance(handles, cost)
            for k in sorted({1, min(n, 7), min(n, 64)}):
                want = A.selective_reclaim(inst, k, backend=oracle_c)
                assert A.selective_reclaim(inst, k) == want, (n, case, k)


# ---------------------------------------------- the reference's property tests, same seeds

def ref_random_instance(rng):
    """test_reclaim.cpp:24-40"""
    n = rng.uniform_int(1, 12)
    n_req = rng.uniform_int(1, 8)
    cost = {r: rng.uniform_int(0, 50) for r in range(n_req)}
    hs = []
    for h in range(n):
        mapped = rng.uniform_int(0, 1000)
        members = rng.uniform_int(1, min(n_req, 4))
        used = set(rng.uniform_int(0, n_req - 1) for _ in range(members))
        hs.append(A.ReclaimHandle(h, mapped, sorted(used)))
    return A.ReclaimInstance(hs, cost)


def ref_disjoint_instance(rng):
    """test_reclaim.cpp:43-59"""
    n = rng.uniform_int(1, 9)
    cost, hs, nxt = {}, [], 0
    for h in range(n):
        mapped = rng.uniform_int(0, 1000)
        members = rng.uniform_int(1, 3)
        reqs = []
        for _ in range(members):
            cost[nxt] = rng.uniform_int(0, 40)
            reqs.append(nxt)
            nxt += 1
        hs.append(A.ReclaimHandle(h, mapped, reqs))
    return A.ReclaimInstance(hs, cost)


def ref_adversarial_instance(rng):
    """test_reclaim.cpp:63-94"""
    n = rng.uniform_int(8, 16)
    n_hot = rng.uniform_int(2, 4)
    cost, hot, nxt = {}, [], 0
    for _ in range(n_hot):
        cost[nxt] = rng.uniform_int(200, 400)
        hot.append(nxt)
        nxt += 1
    oldest = max(1, n // 3)
    hs = []
    for h in range(n):
        if h < oldest:
            picks = rng.uniform_int(2, n_hot)
            used = set(hot[rng.uniform_int(0, n_hot - 1)] for _ in range(picks))
            reqs = sorted(used)
        else:
            cost[nxt] = rng.uniform_int(1, 20)
            reqs = [nxt]
            nxt += 1
            if rng.uniform() < 0.2:
                reqs.insert(0, hot[rng.uniform_int(0, n_hot - 1)])
        hs.append(A.ReclaimHandle(h, h, reqs))
    return A.ReclaimInstance(hs, cost)


def marginal_of(inst, h, evicted):
    return sum(inst.cost[r] for r in h.requests if r not in evicted)


def test_greedy_step_invariant_1000_cases():
    """test_reclaim.cpp:187-220 (Rng::substream(2024, "reclaim-step-invariant"))"""
    rng = Rng.substream(2024, "reclaim-step-invariant")
    for case in range(1000):
        inst = ref_random_instance(rng)
        k = rng.uniform_int(0, len(inst.handles))
        picked = A.selective_reclaim(inst, k)
        assert len(picked) == k
        evicted, taken = set(), set()
        for pick in picked:
            best = None
            for h in inst.handles:
                if h.id in taken:
                    continue
                m = marginal_of(inst, h, evicted)
                if best is None or m < best[0] or (m == best[0] and h.id < best[1]):
                    best = (m, h.id, h)
            assert pick == best[1], case
            taken.add(pick)
            evicted.update(best[2].requests)


def test_greedy_equals_oracle_on_disjoint():
    """test_reclaim.cpp:222-233"""
    rng = Rng.substream(2024, "reclaim-disjoint")
    for case in range(200):
        inst = ref_disjoint_instance(rng)
        for k in range(len(inst.handles) + 1):
            assert A.evicted_cost(inst, A.selective_reclaim(inst, k)) == \
                A.evicted_cost(inst, A.oracle_reclaim(inst, k)), (case, k)


def test_greedy_beats_fifo_adversarial():
    """test_reclaim.cpp:235-256"""
    rng = Rng.substream(2024, "reclaim-adversarial")
    fifo_total = greedy_total = 0
    never_worse = 0
    for _ in range(300):
        inst = ref_adversarial_instance(rng)
        k = rng.uniform_int(1, max(1, len(inst.handles) // 3))
        g = A.evicted_cost(inst, A.selective_reclaim(inst, k))
        f = A.evicted_cost(inst, A.fifo_reclaim(inst, k))
        greedy_total += g
        fifo_total += f
        never_worse += g <= f
    assert fifo_total > 0
    assert (fifo_total - greedy_total) / fifo_total >= 0.20
    assert never_worse == 300


# -------------------------------------------------------------------- fused device reclaim

def _populate(pool_d, pool_o, rng, H, S, n_req):
    live = []
    pool_d.online_grow(max(1, H // 10), 0)
    pool_o.online_grow(max(1, H // 10), 0)
    t = 0
    for r in range(n_req):
        t += rng.randint(1, 100)
        pages = rng.randint(1, 3 * S)
        a = pool_d.offline_reserve(r, pages, t)
        b = pool_o.offline_reserve(r, pages, t)
        assert a == b
        if a:
            live.append(r)
        if live and rng.random() < 0.2:
            x = live.pop(rng.randrange(len(live)))
            pool_d.offline_release(x)
            pool_o.offline_release(x)
    return live, t


@pytest.mark.parametrize("seed,H,S,mode", [(0, 16, 4, 0), (1, 128, 64, 0), (2, 128, 64, 1),
                                           (3, 1024, 64, 0), (4, 300, 16, 0),
                                           # beyond the shared-memory fast paths: > 2048 handles,
                                           # > 4096 listings, 128/256-slot handles (4/8 chunks)
                                           (5, 3000, 8, 0), (6, 2500, 16, 1), (7, 96, 128, 0),
                                           (8, 48, 256, 0)])
def test_fused_reclaim_vs_oracle(oracle_c, seed, H, S, mode):
    rng = random.Random(seed)
    pool_d = A.DevicePool(H, S, 16)
    pool_o = A.MemoryPool(H, S, 16, backend=oracle_c)
    live, t = _populate(pool_d, pool_o, rng, H, S, n_req=H * S // 40 + 5)
    for _ in range(4):
        costs = {r: rng.randint(1, 5000) for r in live}
        pool_d.set_costs(costs)
        inst = pool_o.snapshot()
        inst.cost = {r: costs[r] for h in inst.handles for r in h.requests}
        k = rng.randint(0, max(1, len(inst.handles) // 4))
        pick = (A.selective_reclaim if mode == 0 else A.fifo_reclaim)(inst, k, backend=oracle_c)
        t += 10
        pool_d.reclaim(k, t, mode)
        got = pool_d.last_reclaim()
        want = pool_o.apply_reclaim(pick, t)
        assert fuzz.result_tuple(got, True) == fuzz.result_tuple(want, True)
        for r in got.evicted_requests:
            live.remove(r)
        pool_d.check_invariants()
        assert fuzz._snap(pool_d) == fuzz._snap(pool_o)
        # keep the population moving between ops
        for r in range(10_000 + 100 * _, 10_000 + 100 * _ + rng.randint(0, 5)):
            pages = rng.randint(1, 2 * S)
            assert pool_d.offline_reserve(r, pages, t) == pool_o.offline_reserve(r, pages, t)
            if pool_o.offline_pages_of(r):
                live.append(r)


def test_device_errors_match_reference(ref):
    """Error paths cross the C ABI as the reference's exception types."""
    d = A.MemoryPool(4, 4, 16)
    r = A.MemoryPool(4, 4, 16, backend=ref)
    for pool in (d, r):
        with pytest.raises(A.InvalidArgument):
            pool.online_grow(-1, 0)
        with pytest.raises(A.OutOfRange):
            pool.handle_state(4)
        with pytest.raises(A.OutOfRange):
            pool.requests_on_handle(-1)
        assert pool.offline_reserve(1, 3, 0)
        with pytest.raises(A.LogicError):
            pool.apply_reclaim([0, 0], 5)  # second entry is online by then
        assert pool.online_handles() == 1  # first conversion stuck (memory.cpp mutates in order)
    with pytest.raises(A.InvalidArgument):
        A.MemoryPool(0, 4, 16)


# ------------------------------------------------------------- round-2 boundary regressions

def test_evicted_cost_long_pick_lists_device_vs_reference(ref):
    """Pick lists longer than the instance -- duplicates and unknown ids, which the reference
    accepts (reclaim.cpp:19-31) -- once made the device path grow its buffers after the instance
    upload (use-after-free).  Device vs the reference itself, sized past every buffer's capacity."""
    rng = random.Random(4242)
    for _ in range(120):
        inst = fuzz.random_instance(rng, n_max=rng.choice([1, 3, 12]), cost_max=rng.choice([5, 10**9]))
        ids = [h.id for h in inst.handles]
        n_pick = rng.choice([len(ids) + 1, 2 * len(ids) + 3, 64, 257])
        pick = [rng.choice(ids) for _ in range(n_pick)]
        if rng.random() < 0.3:
            pick[rng.randrange(n_pick)] = max(ids) + 1000  # unknown id -> invalid_argument
        a = fuzz.outcome(lambda: A.evicted_cost(inst, pick, backend=ref))
        b = fuzz.outcome(lambda: A.evicted_cost(inst, pick))
        assert a == b, (inst, pick)


@pytest.mark.parametrize("seed,geom,rows,blocks", [
    (0, (16, 4), 1, 1), (1, (32, 8), 2, 4), (2, (64, 16), 3, 8), (3, (12, 64), 1, 16),
])
def test_request_table_grows_like_the_reference(oracle_c, seed, geom, rows, blocks):
    """The device request table starts at `rows` x `blocks` and must grow on demand: the
    reference MemoryPool has no limit on live requests or pages per request.  The
    randomized sequence (with block tables and physical pages compared) forces several growths
    of both dimensions mid-run, interleaved with reclaims."""
    rng = random.Random(9000 + seed)
    H, S = geom
    pair = fuzz.PoolPair(H, S, 16, None, oracle_c, extended=True)
    pair.a = A.MemoryPool(H, S, 16, config=dict(max_requests=rows, max_pages_per_request=blocks))
    fuzz.random_pool_ops(pair, rng, 400)
    # one request spanning the whole pool
    pair.call("online_release", H)
    big = 10**6
    pair.call("offline_reserve", big, pair.a.free_handles() * S, 5000, -1)
    pair.call("block_table", big)
    pair.call("check_invariants")
