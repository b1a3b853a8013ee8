"""The reference's own known-answer tests, restated against the reference API.

Each test runs three times: against the reference compiled from /root/reference (`ref`, the
pin), the C restatement (`oracle`) and the sm_100a device path (`device`, marked gpu).
Sources: /root/reference/proj/tests/test_memory.cpp, test_reclaim.cpp, test_channel.cpp
(line numbers per test).
"""
import heapq

import pytest

from conftest import BACKENDS, backend_by_name
from paper_2604_07874_b200 import api as A

US_PER_MS, US_PER_S = 1000, 1_000_000


# ------------------------------------------------------------------- test_memory.cpp

@pytest.mark.parametrize("be", BACKENDS)
def test_online_reservation(be):
    """test_memory.cpp:10-28"""
    b = backend_by_name(be)
    pool = A.MemoryPool(8, 4, 16, backend=b)
    assert pool.free_handles() == 8
    pool.online_grow(3, 0)
    assert pool.online_handles() == 3
    assert pool.online_capacity_pages() == 12
    pool.online_use_pages(9)
    assert pool.online_used_pages() == 9
    with pytest.raises(A.LogicError):
        pool.online_use_pages(4)
    assert pool.online_release(2) == 0
    pool.online_free_pages(5)
    assert pool.online_release(3) == 2
    assert pool.online_handles() == 1
    assert pool.free_handles() == 7
    pool.check_invariants()
    with pytest.raises(A.LogicError):
        pool.online_grow(8, 0)


def _packed_pool(b):
    pool = A.MemoryPool(4, 4, 16, backend=b)
    assert pool.offline_reserve(100, 3, 5)
    assert pool.offline_handles() == 1
    assert pool.offline_pages_of(100) == 3
    assert pool.offline_reserve(101, 2, 6)
    assert pool.offline_handles() == 2
    assert pool.requests_on_handle(0) == [100, 101]
    assert pool.handles_of_request(101) == [0, 1]
    assert not pool.offline_reserve(102, 12, 7)
    assert pool.offline_pages_of(102) == 0
    pool.check_invariants()
    return pool


@pytest.mark.parametrize("be", BACKENDS)
def test_offline_release_subcase(be):
    """test_memory.cpp:30-44 + SUBCASE 45-52"""
    pool = _packed_pool(backend_by_name(be))
    pool.offline_release(101)
    assert pool.offline_handles() == 1
    pool.offline_release(100)
    assert pool.offline_handles() == 0
    assert pool.free_handles() == 4
    pool.check_invariants()


@pytest.mark.parametrize("be", BACKENDS)
def test_offline_cap_subcase(be):
    """test_memory.cpp:30-44 + SUBCASE 54-60"""
    pool = _packed_pool(backend_by_name(be))
    assert not pool.offline_reserve(103, 6, 8, 2)
    assert pool.offline_reserve(104, 3, 9, 2)
    assert pool.offline_handles() == 2


@pytest.mark.parametrize("be", BACKENDS)
def test_apply_reclaim_evicts_residents(be):
    """test_memory.cpp:63-90"""
    pool = A.MemoryPool(4, 4, 16, backend=backend_by_name(be))
    assert pool.offline_reserve(7, 3, 1)
    assert pool.offline_reserve(8, 2, 2)
    assert pool.offline_reserve(9, 4, 3)
    pool.check_invariants()
    before_free = pool.free_handles()
    res = pool.apply_reclaim([1], 10)
    assert res.handles == [1]
    assert res.evicted_requests == [8, 9]
    assert len(res.invalidated_pages[8]) == 1
    assert len(res.invalidated_pages[9]) == 3
    assert pool.online_handles() == 1
    assert pool.offline_pages_of(8) == 0
    assert pool.offline_pages_of(9) == 0
    assert pool.offline_pages_of(7) == 3
    assert pool.free_handles() == before_free + 1
    pool.check_invariants()
    for pages in res.invalidated_pages.values():
        for p in pages:
            assert 0 <= p < pool.quarantine_page_id()


@pytest.mark.parametrize("be", BACKENDS)
def test_snapshot(be):
    """test_memory.cpp:92-103"""
    pool = A.MemoryPool(4, 4, 16, backend=backend_by_name(be))
    assert pool.offline_reserve(1, 4, 100)
    assert pool.offline_reserve(2, 2, 200)
    inst = pool.snapshot()
    assert len(inst.handles) == 2
    assert inst.handles[0].id == 0 and inst.handles[0].mapped_at == 100
    assert inst.handles[0].requests == [1]
    assert inst.handles[1].mapped_at == 200 and inst.handles[1].requests == [2]


@pytest.mark.parametrize("be", BACKENDS)
def test_reservation_miad(be):
    """test_memory.cpp:105-121"""
    b = backend_by_name(be)
    p = A.ReservationParams()
    ctl = A.ReservationController(p, backend=b)
    assert ctl.grow_target(10, 100) == 15
    assert ctl.grow_target(10, 12) == 12
    assert ctl.grow_target(1, 100) == 2
    assert ctl.grow_target(0, 100) == 1
    ctl.note_tick(0)
    assert ctl.release_due(p.t_init_us, 5)
    assert not ctl.release_due(p.t_init_us, p.h_min)
    ctl.record_pressure(p.t_init_us // 2)
    assert not ctl.release_due(p.t_init_us, 5)


@pytest.mark.parametrize("be", BACKENDS)
def test_reservation_interval(be):
    """test_memory.cpp:123-145"""
    b = backend_by_name(be)
    p = A.ReservationParams()
    ctl = A.ReservationController(p, backend=b)
    assert ctl.interval() == US_PER_S
    ctl.record_pressure(10 * US_PER_S)
    ctl.record_pressure(20 * US_PER_S)
    assert ctl.window_tick(60 * US_PER_S) == 2 * US_PER_S
    assert ctl.window_tick(120 * US_PER_S) == 2 * US_PER_S - 100 * US_PER_MS
    low = A.ReservationController(p, backend=b)
    for i in range(1000):
        low.window_tick((i + 1) * p.window_us)
    assert low.interval() == p.t_min_us
    high = A.ReservationController(p, backend=b)
    for i in range(20):
        high.record_pressure(i * p.window_us + 1)
        high.record_pressure(i * p.window_us + 2)
        high.window_tick((i + 1) * p.window_us)
    assert high.interval() == p.t_max_us


@pytest.mark.parametrize("be", BACKENDS)
def test_pressure_window(be):
    """test_memory.cpp:147-156"""
    ctl = A.ReservationController(A.ReservationParams(), backend=backend_by_name(be))
    ctl.record_pressure(1)
    ctl.record_pressure(30 * US_PER_S)
    ctl.record_pressure(61 * US_PER_S)
    assert ctl.pressure_in_window(60 * US_PER_S) == 2
    assert ctl.pressure_in_window(120 * US_PER_S) == 1
    assert ctl.pressure_events() == 3


@pytest.mark.parametrize("be", BACKENDS)
def test_reservation_params_validation(be):
    """memory.cpp:213-218"""
    b = backend_by_name(be)
    for bad in (dict(alpha=1.0), dict(beta=0.5), dict(t_init_us=0), dict(t_min_us=0),
                dict(t_max_us=10, t_min_us=20), dict(window_us=0), dict(h_min=-1)):
        with pytest.raises(A.InvalidArgument):
            A.ReservationController(A.ReservationParams(**bad), backend=b)


# ------------------------------------------------------------------- test_reclaim.cpp

def tiny_instance():
    # test_reclaim.cpp:15-21: h1={r1}, h2={r2}, h3={r1,r2}; cost r1=10, r2=4
    return A.ReclaimInstance([A.ReclaimHandle(1, 100, [1]), A.ReclaimHandle(2, 200, [2]),
                              A.ReclaimHandle(3, 300, [1, 2])], {1: 10, 2: 4})


@pytest.mark.parametrize("be", BACKENDS)
def test_cheapest_single_handle(be):
    """test_reclaim.cpp:107-112"""
    b = backend_by_name(be)
    inst = tiny_instance()
    assert A.selective_reclaim(inst, 1, backend=b) == [2]
    assert A.evicted_cost(inst, [2], backend=b) == 4
    assert A.oracle_reclaim(inst, 1, backend=b) == [2]


@pytest.mark.parametrize("be", BACKENDS)
def test_shared_requests_marginal(be):
    """test_reclaim.cpp:114-124"""
    b = backend_by_name(be)
    inst = A.ReclaimInstance([A.ReclaimHandle(1, 10, [1, 4]), A.ReclaimHandle(2, 20, [2, 5]),
                              A.ReclaimHandle(3, 30, [1, 2])], {1: 10, 2: 4, 4: 100, 5: 106})
    assert A.selective_reclaim(inst, 2, backend=b) == [3, 1]
    assert A.evicted_cost(inst, [3, 1], backend=b) == 114


@pytest.mark.parametrize("be", BACKENDS)
def test_tie_smallest_id(be):
    """test_reclaim.cpp:126-132"""
    b = backend_by_name(be)
    inst = A.ReclaimInstance([A.ReclaimHandle(7, 10, [1]), A.ReclaimHandle(3, 20, [2]),
                              A.ReclaimHandle(5, 30, [3])], {1: 9, 2: 9, 3: 9})
    assert A.selective_reclaim(inst, 1, backend=b) == [3]
    assert A.selective_reclaim(inst, 2, backend=b) == [3, 5]


@pytest.mark.parametrize("be", BACKENDS)
def test_full_pool_and_clamp(be):
    """test_reclaim.cpp:134-145"""
    b = backend_by_name(be)
    inst = tiny_instance()
    assert sorted(A.selective_reclaim(inst, 3, backend=b)) == [1, 2, 3]
    assert sorted(A.selective_reclaim(inst, 99, backend=b)) == [1, 2, 3]
    assert A.selective_reclaim(inst, 0, backend=b) == []
    with pytest.raises(A.InvalidArgument):
        A.selective_reclaim(inst, -1, backend=b)


@pytest.mark.parametrize("be", BACKENDS)
def test_straddling_charged_once(be):
    """test_reclaim.cpp:147-156"""
    b = backend_by_name(be)
    inst = tiny_instance()
    assert A.evicted_cost(inst, [1, 2, 3], backend=b) == 14
    assert A.evicted_cost(inst, [3], backend=b) == 14
    assert A.evicted_cost(inst, [], backend=b) == 0
    with pytest.raises(A.InvalidArgument):
        A.evicted_cost(inst, [9], backend=b)
    missing = tiny_instance()
    del missing.cost[2]
    with pytest.raises(A.InvalidArgument):
        A.evicted_cost(missing, [2], backend=b)


@pytest.mark.parametrize("be", BACKENDS)
def test_fifo(be):
    """test_reclaim.cpp:158-169"""
    b = backend_by_name(be)
    inst = A.ReclaimInstance([A.ReclaimHandle(1, 5, [1]), A.ReclaimHandle(2, 3, [2])], {1: 1, 2: 1})
    assert A.fifo_reclaim(inst, 1, backend=b) == [2]
    assert A.fifo_reclaim(inst, 2, backend=b) == [2, 1]
    tied = A.ReclaimInstance([A.ReclaimHandle(4, 7, [1]), A.ReclaimHandle(2, 7, [1]),
                              A.ReclaimHandle(3, 6, [1])], {1: 1})
    assert A.fifo_reclaim(tied, 3, backend=b) == [3, 2, 4]


@pytest.mark.parametrize("be", BACKENDS)
def test_oracle_two_subsets(be):
    """test_reclaim.cpp:171-179"""
    b = backend_by_name(be)
    inst = tiny_instance()
    for pick in ([1, 2], [1, 3], [2, 3]):
        assert A.evicted_cost(inst, pick, backend=b) == 14
    assert A.oracle_reclaim(inst, 2, backend=b) == [1, 2]
    assert A.evicted_cost(inst, A.selective_reclaim(inst, 2, backend=b), backend=b) == 14


@pytest.mark.parametrize("be", BACKENDS)
def test_oracle_size_limit(be):
    """test_reclaim.cpp:181-185"""
    big = A.ReclaimInstance([A.ReclaimHandle(h, 0, []) for h in range(21)], {})
    with pytest.raises(A.InvalidArgument):
        A.oracle_reclaim(big, 2, backend=backend_by_name(be))


@pytest.mark.parametrize("be", BACKENDS)
def test_missing_cost_throws_only_when_evaluated(be):
    """reclaim.cpp:12-16,33-46: cost_of throws on the first evaluation (k > 0 only)."""
    b = backend_by_name(be)
    inst = tiny_instance()
    del inst.cost[1]
    assert A.selective_reclaim(inst, 0, backend=b) == []
    with pytest.raises(A.InvalidArgument):
        A.selective_reclaim(inst, 1, backend=b)
    assert A.fifo_reclaim(inst, 2, backend=b) == [1, 2]  # fifo never looks at costs


# ------------------------------------------------------------------- test_channel.cpp

class Harness:
    """test_channel.cpp:15-43: private event queue + recording hooks."""

    def __init__(self, toggle, cooldown, b):
        self.q = []
        self.seq = 0
        self.logs = []
        self.stops = []
        self.now = 0
        hooks = A.Hooks(schedule=self._schedule, on_disabled=lambda t: self.stops.append((t, True)),
                        on_enabled=lambda t: self.stops.append((t, False)),
                        log=lambda t, w, aux, mem: self.logs.append((t, w, aux)))
        self.ctl = A.ChannelController(toggle, cooldown, hooks, backend=b)

    def _schedule(self, when, gen, cooldown):
        assert when >= self.now  # engine.cpp:10-13
        heapq.heappush(self.q, (when, self.seq, cooldown, gen))
        self.seq += 1

    def run(self, until):
        while self.q and self.q[0][0] <= until:
            when, _, cd, gen = heapq.heappop(self.q)
            self.now = when
            if cd:
                self.ctl.handle_cooldown(when, gen)
            else:
                self.ctl.handle_toggle(when, gen)
        self.now = max(self.now, until)

    def logged(self, what):
        return any(w == what for _, w, _ in self.logs)


@pytest.mark.parametrize("be", BACKENDS)
def test_disable_latency(be):
    """test_channel.cpp:47-58"""
    h = Harness(1000, 600, backend_by_name(be))
    assert h.ctl.offline_compute_allowed()
    h.ctl.note_busy(10)
    assert h.ctl.state() == A.ChannelController.kDisabling
    assert not h.ctl.offline_compute_allowed()
    assert h.ctl.pending_effective() == 1010
    h.run(1010)
    assert h.ctl.state() == A.ChannelController.kDisabled
    assert h.stops == [(1010, True)]
    assert h.ctl.disables_issued() == 1


@pytest.mark.parametrize("be", BACKENDS)
def test_multi_gpu_latency(be):
    """test_channel.cpp:60-66"""
    h = Harness(8 * 1000, 0, backend_by_name(be))
    h.ctl.note_busy(0)
    assert h.ctl.pending_effective() == 8000
    h.run(8000)
    assert h.ctl.state() == A.ChannelController.kDisabled


@pytest.mark.parametrize("be", BACKENDS)
def test_cooldown_2g(be):
    """test_channel.cpp:68-81"""
    assert A.CooldownPolicy(12 * US_PER_MS).cooldown_us() == 24 * US_PER_MS
    assert A.CooldownPolicy(0).cooldown_us() == 0
    h = Harness(1000, 24 * US_PER_MS, backend_by_name(be))
    h.ctl.note_busy(0)
    h.run(1000)
    h.ctl.note_all_idle(5000)
    h.run(5000 + 24 * US_PER_MS)
    assert h.ctl.state() == A.ChannelController.kEnabling
    h.run(5000 + 24 * US_PER_MS + 1000)
    assert h.ctl.state() == A.ChannelController.kEnabled
    assert h.stops[-1] == (5000 + 24 * US_PER_MS + 1000, False)


@pytest.mark.parametrize("be", BACKENDS)
def test_zero_cooldown(be):
    """test_channel.cpp:83-94"""
    h = Harness(50, 0, backend_by_name(be))
    h.ctl.note_busy(0)
    h.run(50)
    h.ctl.note_all_idle(100)
    h.run(200)
    assert h.ctl.state() == A.ChannelController.kEnabled
    h.ctl.note_busy(300)
    h.run(400)
    assert h.ctl.disables_issued() == 2


@pytest.mark.parametrize("be", BACKENDS)
def test_cancel_in_window(be):
    """test_channel.cpp:96-107"""
    h = Harness(1000, 600, backend_by_name(be))
    h.ctl.note_busy(0)
    h.run(1000)
    h.ctl.note_all_idle(2000)
    h.ctl.note_busy(2400)
    assert h.logged(A.ChannelLog.kCooldownCancelled)
    assert h.ctl.disables_issued() == 1
    h.run(3000)
    assert h.ctl.state() == A.ChannelController.kDisabled
    assert not h.logged(A.ChannelLog.kEnableIssued)


@pytest.mark.parametrize("be", BACKENDS)
def test_rearmed_cooldown(be):
    """test_channel.cpp:109-120"""
    h = Harness(100, 500, backend_by_name(be))
    h.ctl.note_busy(0)
    h.run(100)
    h.ctl.note_all_idle(200)
    h.ctl.note_busy(600)
    h.ctl.note_all_idle(1000)
    h.run(1400)
    assert h.ctl.state() == A.ChannelController.kDisabled
    h.run(1600)
    assert h.ctl.state() == A.ChannelController.kEnabled


@pytest.mark.parametrize("be", BACKENDS)
def test_ensure_disabled(be):
    """test_channel.cpp:122-134"""
    h = Harness(1000, 0, backend_by_name(be))
    assert h.ctl.ensure_disabled(100) == 1100
    assert h.ctl.state() == A.ChannelController.kDisabling
    assert h.ctl.ensure_disabled(300) == 1100
    assert h.ctl.disables_issued() == 1
    h.run(1100)
    assert h.ctl.ensure_disabled(2000) == 2000
    assert h.ctl.disables_issued() == 1


@pytest.mark.parametrize("be", BACKENDS)
def test_deferred_enable(be):
    """test_channel.cpp:136-144"""
    h = Harness(1000, 100, backend_by_name(be))
    h.ctl.note_busy(0)
    h.ctl.note_all_idle(500)
    h.run(2100)
    assert h.stops == [(1000, True), (2000, False)]


@pytest.mark.parametrize("be", BACKENDS)
def test_busy_during_drain_squash(be):
    """test_channel.cpp:146-155"""
    h = Harness(1000, 100, backend_by_name(be))
    h.ctl.note_busy(0)
    h.ctl.note_all_idle(500)
    h.run(700)
    h.ctl.note_busy(800)
    h.run(3000)
    assert h.ctl.state() == A.ChannelController.kDisabled
    assert h.ctl.disables_issued() == 1


@pytest.mark.parametrize("be", BACKENDS)
def test_channel_negative_latency(be):
    """channel.cpp:9-10"""
    with pytest.raises(A.InvalidArgument):
        A.ChannelController(-1, 0, backend=backend_by_name(be))
