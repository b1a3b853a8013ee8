"""Host-side pieces of the real-time harness (CPU): the online slot allocator (clean / pending
slots, landed tickets, lazy heap deletion) and the pinned copy arena's FIFO byte ring."""
import random

import pytest

from paper_2604_07874_b200 import realtime as RT


class FakePool:
    def __init__(self, S=4):
        self.S, self.ids, self.l = S, [], 0

    def handle_size_pages(self):
        return self.S

    def online_handle_ids(self):
        return list(self.ids)

    def landed(self):
        return (self.l, self.l)


def test_online_pages_clean_first_highest_first_then_by_ticket():
    fp = FakePool()
    op = RT.OnlinePages(fp)
    fp.ids = [0, 1, 2]
    op.sync_handles()
    assert op.alloc(3, 7) == [11, 10, 9]
    op.set_tickets([4, 5], (0, 2, 100))  # free slots 4, 5: a copy has not read them out yet
    assert op.alloc(2, 8) == [8, 7]      # clean ones first
    fp.ids = [0, 1, 2, 3]
    op.set_tickets([12, 13, 14, 15], (2, 3, 100))
    op.sync_handles()
    assert sorted(op.pending) == [4, 5, 12, 13, 14, 15]
    fp.l = 2  # the first copy is out: 4, 5 become clean
    assert op.alloc(4, 9) == [6, 5, 4, 3]
    assert op.clean_count_outside({0}) == len(op.free) - len(op.pending) - sum(
        1 for s in range(0, 4) if s in op.free and s not in op.pending)
    with pytest.raises(RuntimeError):
        op.alloc(len(op.free) + 1, 10)


def test_online_pages_randomized_invariants():
    rng = random.Random(1)
    fp = FakePool()
    op = RT.OnlinePages(fp)
    fp.ids = list(range(8))
    op.sync_handles()
    base = 0
    for it in range(4000):
        x = rng.random()
        if x < 0.4 and len(op.free) > 4:
            got = op.alloc(rng.randint(1, 4), it)
            assert len(set(got)) == len(got) and not any(g in op.free for g in got)
        elif x < 0.7 and op.used:
            op.release(rng.sample(sorted(op.used), min(len(op.used), rng.randint(1, 3))))
        elif x < 0.8:
            free = sorted(op.free)
            op.set_tickets(rng.sample(free, min(3, len(free))), (base, 2, 100))
            base += 2
        else:
            fp.l = base
        assert set(op.used).isdisjoint(op.free)
        assert op.pending <= op.free and all(s in op.ticket for s in op.pending)
        assert len(op.used) + len(op.free) == 32


class _Arena:
    def __init__(self, n):
        self.nbytes, self.ptr = n, 0


class _Ring(RT.Colocation):
    """Only the copy-arena methods of Colocation, over a fake pool that completes copies FIFO."""

    def __init__(self, size):
        self.arena = _Arena(size)
        self._copies = []
        self.completed = []
        self.res = type("R", (), {"copy_gbs": []})()

        class _P:
            def reclaim_copy_wait(p):
                class St:
                    kernel_ms, bytes = 0.0, 0
                return St()
        self.pool = _P()

    def _complete_copy(self):
        self.completed.append(self._copies[0])
        super()._complete_copy()


def test_copy_arena_ring_never_overlaps_in_flight_bytes():
    rng = random.Random(3)
    ring = _Ring(100)
    for op in range(2000):
        n = rng.randint(1, 60)
        off = ring._arena_alloc(n)
        assert 0 <= off and off + n <= 100
        for _, o, m in ring._copies:  # no overlap with any copy still in flight
            assert off + n <= o or o + m <= off
        assert len(ring._copies) < RT.A.COPY_RING
        ring._copies.append((op, off, n))
        if rng.random() < 0.3 and ring._copies:
            ring._complete_copy()
