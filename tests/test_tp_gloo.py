"""Multi-process host logic (world size 2 and 4, gloo, CPU): TP group formation, gate-handle
exchange, and that only group leaders attach members and may drive the group gate.  The device
side of the same wiring runs in tests/test_gpu_tp.py (two processes sharing one GPU via IPC)."""
import os
import socket

import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2604_07874_b200 import tp as TP


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


class FakeGate:
    """Stands in for api.Gate: export() returns rank-tagged bytes; records attachments/raises."""

    def __init__(self, rank):
        self.rank = rank
        self.attached = []
        self.raised = []

    def export(self):
        return f"gate-of-rank-{self.rank}".encode()

    def attach_peers(self, members):
        self.attached.extend(members)

    def raise_(self, gen, stream=None):
        self.raised.append(gen)


def _worker(rank, world, tp, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    g = FakeGate(rank)
    t = TP.TPGate(g, rank, world, tp, dist, opener=lambda h: h.decode())
    ok_drive = True
    try:
        t.raise_(7)
    except RuntimeError:
        ok_drive = False
    q.put((rank, t.is_leader, t.group, sorted(g.attached), g.raised, ok_drive))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world,tp", [(2, 2), (4, 2), (4, 4)])
def test_tp_gate_wiring_gloo(world, tp):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, tp, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(60)
        assert p.exitcode == 0
    for rank, leader, group, attached, raised, drove in res:
        assert group == [g for g in TP.tp_groups(world, tp) if rank in g][0]
        assert leader == (rank == group[0])
        if leader:
            assert attached == sorted(f"gate-of-rank-{r}" for r in group if r != rank)
            assert raised == [7] and drove
        else:
            assert attached == [] and raised == [] and not drove


def test_tp_groups():
    assert TP.tp_groups(8, 4) == [[0, 1, 2, 3], [4, 5, 6, 7]]
    assert TP.tp_groups(2, 1) == [[0], [1]]
    with pytest.raises(ValueError):
        TP.tp_groups(6, 4)


def test_rank_device_one_process_per_gpu():
    assert [TP.rank_device(r, 8, 8) for r in range(8)] == [(r, False) for r in range(8)]
    assert TP.rank_device(3, 4, 4) == (3, False)
    # fewer GPUs than ranks: round-robin, flagged shared (functional runs only)
    assert TP.rank_device(3, 4, 1) == (0, True)
    assert TP.rank_device(3, 4, 2) == (1, True)
    with pytest.raises(RuntimeError):
        TP.rank_device(0, 1, 0)


class DeviceGate(FakeGate):
    """CPU mock of a gate living in HBM of `device`: honest about what it checks -- which device
    each rank's words live on and on which device the leader maps them -- and nothing about the
    NVLink path itself (that needs a multi-GPU box: bench.py --gpus N, tp_fanout_across_ranks)."""

    def __init__(self, rank, device):
        super().__init__(rank)
        self.device = device

    def export(self):
        return f"gate-of-rank-{self.rank}@cuda:{self.device}".encode()


def _distinct_worker(rank, world, tp, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    dev, shared = TP.rank_device(rank, world, world)  # a node with one GPU per rank
    g = DeviceGate(rank, dev)
    opened = []

    def opener(handle):  # the leader maps a member's words on ITS OWN device (IPC + peer access)
        opened.append((handle.decode(), dev))
        return handle.decode()

    t = TP.TPGate(g, rank, world, tp, dist, opener=opener)
    q.put((rank, dev, shared, t.is_leader, opened))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world,tp", [(2, 2), (4, 4)])
def test_tp_group_spans_distinct_devices_gloo(world, tp):
    """world-size-N wiring as bench.py --gpus N runs it: rank r's gate on cuda:r, the leader
    opens every member's words on its own device, so each member is a different GPU than the
    leader (the peer-memory path), never a same-device alias."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_distinct_worker, args=(r, world, tp, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(60)
        assert p.exitcode == 0
    assert [r[1] for r in res] == list(range(world)) and not any(r[2] for r in res)
    leader = [r for r in res if r[3]]
    assert len(leader) == 1 and leader[0][0] == 0
    assert leader[0][4] == [(f"gate-of-rank-{m}@cuda:{m}", 0) for m in range(1, world)]
