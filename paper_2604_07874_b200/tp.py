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

from typing import List, Sequence


def tp_groups(world: int, tp: int) -> List[List[int]]:
    """Consecutive ranks form a TP group (rank // tp); the first rank of a group leads it."""
    if tp <= 0 or world % tp:
        raise ValueError(f"world size {world} is not a multiple of tp {tp}")
    return [list(range(g * tp, (g + 1) * tp)) for g in range(world // tp)]


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
        if self.is_leader:
            self.members = [opener(handles[r]) for r in self.group if r != rank]
            if self.members:
                gate.attach_peers(self.members)
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
