"""Tensor-parallel online groups: one device gate per TP group, driven by the group leader.

The reference has one node-wide channel gate: a busy edge on any online lane stops offline on
every GPU (sim.cpp:362-380, 860-873), at a cost linear in GPUs with the unpatched driver
(scenario.hpp:56-58).  Here every GPU runs its own colocation instance (one process per GPU,
replicas for pool/selection/copy -- no NCCL), and only a TP online group shares a gate:

  * each rank creates its gate (HBM words on its GPU) and exports a CUDA IPC handle;
  * handles are exchanged with torch.distributed (plumbing only: all_gather_object);
  * the group leader opens the members' words and attaches them, so its raise / release / wait
    issue stream memory operations on every member's words over NVLink peer memory (a flat
    fan-out: no extra kernel, no collective);
  * members keep polling their own gate from their offline kernels; their quiesce ack
    (live_ctas) is what the leader's online stream waits on.
"""
from __future__ import annotations

import time
from typing import List, Sequence, Tuple


def tp_groups(world: int, tp: int) -> List[List[int]]:
    """Consecutive ranks form a TP group (rank // tp); the first rank of a group leads it."""
    if tp <= 0 or world % tp:
        raise ValueError(f"world size {world} is not a multiple of tp {tp}")
    return [list(range(g * tp, (g + 1) * tp)) for g in range(world // tp)]


def rank_device(local_rank: int, local_world: int, n_devices: int) -> Tuple[int, bool]:
    """(device, shared) for a rank: one process per GPU -- rank r on cuda:r -- whenever the node
    has a GPU per local rank; a box with fewer GPUs maps ranks round-robin and reports
    shared=True (functional runs only: the contexts time-slice one GPU and there is no NVLink
    hop, so no latency taken there is a TP number)."""
    if n_devices <= 0:
        raise RuntimeError("no CUDA device: every rank's gate lives in HBM")
    return local_rank % n_devices, n_devices < local_world


def group_of(rank: int, groups: Sequence[Sequence[int]]) -> List[int]:
    for g in groups:
        if rank in g:
            return list(g)
    raise ValueError(f"rank {rank} in no group")


class TPGate:
    """Wires the gates of one TP group across processes.

    gate      this rank's device gate (api.Gate, or any object with export()/attach_peers())
    opener    callable(handle_bytes) -> gate view of a member's words in this process
    """

    def __init__(self, gate, rank: int, world: int, tp: int, dist, opener, device: int = 0):
        self.gate = gate
        self.rank = rank
        self.group = group_of(rank, tp_groups(world, tp))
        self.leader = self.group[0]
        self.is_leader = rank == self.leader
        handles = [None] * world
        dist.all_gather_object(handles, gate.export())
        self.members = []
        self.error = None
        if self.is_leader:
            try:
                self.members = [opener(handles[r]) for r in self.group if r != rank]
                if self.members:
                    gate.attach_peers(self.members)
            except Exception as e:  # noqa: BLE001 -- recorded; every rank still reaches the barrier
                self.error = repr(e)[:200]
                self.members = []
        dist.barrier()

    # leader-side controls (members never drive the group gate)
    def raise_(self, gen: int, stream=None):
        self._leader_only()
        self.gate.raise_(gen, stream)

    def release(self, gen: int, stream=None):
        self._leader_only()
        self.gate.release(gen, stream)

    def wait_quiesced(self, gen: int, stream=None):
        self._leader_only()
        self.gate.wait_quiesced(gen, stream)

    def _leader_only(self):
        if not self.is_leader:
            raise RuntimeError(f"rank {self.rank} is not the leader of TP group {self.group}")


def open_member(device: int):
    """Opener for TPGate: a member's exported gate words, mapped into this process on the
    leader's device (CUDA IPC with lazy peer access: the words stay in the member's HBM and the
    leader's stream memory operations reach them over NVLink)."""
    from . import api as A

    return lambda handle: A.Gate.open_remote(handle, device)


def measure_group_fanout(torch, gate, group: "TPGate", pool, dist, device: int, iters: int = 200,
                         ctas: int = 0, seed: int = 0):
    """Preempt-to-quiesce of one TP group, one process (and GPU) per member: every member runs
    its gated offline decode pass over its own pool; the leader raises the group gate (stream
    memory operations on every member's words over peer memory) and its stream waits until every
    member's CTAs retired.  Latency = CUDA events around raise + wait on the leader's gate
    stream.  Iterations are host-synchronised with dist.barrier() so every member is running
    when the leader raises.  The reference's unpatched toggle is linear in the GPUs
    (scenario.hpp:56-58).

    Every rank runs the same barrier schedule whatever happens on its device (a failing call is
    recorded, not raised), so one rank's error cannot leave the others inside a collective.
    Returns (leader's samples in us, errors, members seen not quiesced after the wait)."""
    import random

    rng = random.Random(seed)
    off = torch.cuda.Stream(device=device)
    gs = torch.cuda.ExternalStream(gate.stream, device=device)
    lat, errors, violations = [], [], 0

    def attempt(fn):
        if len(errors) > 3:  # a broken path: stop touching the device, keep the schedule
            return False
        try:
            fn()
            return True
        except Exception as e:  # noqa: BLE001
            errors.append(repr(e)[:200])
            return False

    for it in range(iters + 10):
        def start():
            gate.reset_work()
            gate.launch_offline(pool, None, None, 0, 0, None, ctas=ctas, stream=off.cuda_stream)
        attempt(start)
        time.sleep(0.001)  # the pass is running (it lasts far longer than a sample)
        dist.barrier()
        if group.is_leader:
            def sample():
                deadline = time.perf_counter() + rng.uniform(100e-6, 400e-6)
                while time.perf_counter() < deadline:
                    pass
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(gs)
                group.raise_(it + 1)
                group.wait_quiesced(it + 1)
                e1.record(gs)
                e1.synchronize()
                if it >= 10:
                    lat.append(e0.elapsed_time(e1) * 1e3)
            attempt(sample)
        dist.barrier()

        def check():
            nonlocal violations
            st = gate.read()
            violations += int(not (st.closed == 1 and st.live_ctas == 0))
        attempt(check)
        dist.barrier()
        if group.is_leader:
            attempt(lambda: (group.release(it + 1), gs.synchronize()))
        dist.barrier()
        attempt(lambda: (gate.cancel_work(), off.synchronize()))  # next sample: a fresh pass
    return lat, errors, violations
