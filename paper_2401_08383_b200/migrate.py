"""Online placement change: move expert weights to the GPUs of a new
placement (histogram rebuild -> solve_staged ->
expert migration).

The affinity histogram comes from the fused per-layer counters
(`MoeModel.affinity_counts`, summed over ranks), the solver is the host
`placement.solve_staged` (proj/src/placement.cpp:720-821); this module moves
the 16*d^2-byte expert weights (W1, b1, W2, b2) into the slots of the new
table and installs it. A rank's slot k of a layer holds its k-th expert in
expert order (the same rule as exf_model_create), so experts that stay on a
GPU can still change slot.

Two transports: `migrate_local` for G virtual ranks in one process (device
copies), `migrate_nccl` for one process per GPU (torch.distributed
batch_isend_irecv on an NCCL group; the old owner sends, the new owner
receives). Both work layer by layer through staging buffers, so old and new
slots never alias.
"""
from __future__ import annotations

from typing import Dict, List, Sequence, Tuple

import numpy as np


def slot_table(assign: np.ndarray, G: int) -> np.ndarray:
    """[L][E] local slot of every expert on its GPU (expert order)."""
    assign = np.asarray(assign)
    slots = np.zeros_like(assign)
    for j in range(assign.shape[0]):
        load = [0] * G
        for e in range(assign.shape[1]):
            g = int(assign[j, e])
            slots[j, e] = load[g]
            load[g] += 1
    return slots


def plan(old: np.ndarray, new: np.ndarray, G: int) -> List[Tuple[int, int, int, int, int, int]]:
    """Every (layer, expert, src rank, src slot, dst rank, dst slot) whose
    storage changes, in a deterministic global order (layer, expert)."""
    so, sn = slot_table(old, G), slot_table(new, G)
    out = []
    for j in range(old.shape[0]):
        for e in range(old.shape[1]):
            src, dst = int(old[j, e]), int(new[j, e])
            if (src, int(so[j, e])) != (dst, int(sn[j, e])):
                out.append((j, e, src, int(so[j, e]), dst, int(sn[j, e])))
    return out


def migrate_local(models: Sequence, new_assign: np.ndarray) -> int:
    """G virtual ranks in one process: returns the number of experts moved
    between ranks (slot shuffles inside a rank not counted)."""
    import torch
    G = models[0].config.world_size
    old = models[0].assign
    moves = plan(old, new_assign, G)
    by_layer: Dict[int, list] = {}
    for mv in moves:
        by_layer.setdefault(mv[0], []).append(mv)
    torch.cuda.synchronize()
    for j, mvs in by_layer.items():
        staged = []
        for (_, e, src, ss, dst, ds) in mvs:
            staged.append((dst, ds, [t.clone() for t in models[src].expert_storage(j, ss)]))
        for dst, ds, tensors in staged:
            for d_t, s_t in zip(models[dst].expert_storage(j, ds), tensors):
                d_t.copy_(s_t)
    torch.cuda.synchronize()
    for m in models:
        m.set_placement(new_assign)
    return sum(1 for mv in moves if mv[2] != mv[4])


def _wire(t):
    """NCCL-transferable view of a weight slot (int16 bf16 bits -> bfloat16; fp32 as is)."""
    import torch
    return t.view(torch.bfloat16) if t.dtype == torch.int16 else t


def warm_up(group=None) -> None:
    """Open the NCCL peer-to-peer connections between every pair of ranks
    (one tiny send/recv per pair): NCCL sets them up lazily on first use,
    which would otherwise land inside the first timed migration."""
    import torch
    import torch.distributed as dist
    G, rank = dist.get_world_size(group), dist.get_rank(group)
    dist.barrier(group=group)
    dev = torch.device("cuda", torch.cuda.current_device())
    send = [torch.zeros(1, device=dev) for _ in range(G)]
    recv = [torch.empty(1, device=dev) for _ in range(G)]
    ops = []
    for p in range(G):
        if p != rank:
            ops.append(dist.P2POp(dist.isend, send[p], p, group=group))
            ops.append(dist.P2POp(dist.irecv, recv[p], p, group=group))
    if ops:
        for r in dist.batch_isend_irecv(ops):
            r.wait()
    torch.cuda.synchronize()


def migrate_nccl(model, new_assign: np.ndarray, group=None) -> int:
    """One process per GPU (every rank calls it with the same table): the old
    owner sends each moved expert's weights over NCCL, the new owner receives
    them into staging buffers, then copies into the new slots."""
    import torch
    import torch.distributed as dist
    G, rank = model.config.world_size, model.config.rank
    moves = plan(model.assign, new_assign, G)
    by_layer: Dict[int, list] = {}
    for mv in moves:
        by_layer.setdefault(mv[0], []).append(mv)
    torch.cuda.synchronize()
    # every rank joins one collective on the group first: PyTorch creates the
    # NCCL communicator lazily, and its first batch_isend_irecv must include
    # every rank of the group (a rank without moves in the first moving layer
    # would otherwise leave the others' communicator init hanging)
    dist.barrier(group=group)
    for j, mvs in sorted(by_layer.items()):
        ops, staged = [], []
        for (_, e, src, ss, dst, ds) in mvs:
            if src == rank and dst == rank:  # slot shuffle on this GPU
                staged.append((ds, [t.clone() for t in model.expert_storage(j, ss)]))
            elif src == rank:  # (bf16 views of int16 storage: NCCL has no int16 type)
                for t in model.expert_storage(j, ss):
                    ops.append(dist.P2POp(dist.isend, _wire(t), dst, group=group))
            elif dst == rank:
                bufs = [_wire(torch.empty_like(t)) for t in model.expert_storage(j, ds)]
                for b in bufs:
                    ops.append(dist.P2POp(dist.irecv, b, src, group=group))
                staged.append((ds, bufs))
        if ops:
            for r in dist.batch_isend_irecv(ops):
                r.wait()
        torch.cuda.synchronize()
        for ds, bufs in staged:
            for d_t, b in zip(model.expert_storage(j, ds), bufs):
                d_t.copy_(b.view(d_t.dtype))
    torch.cuda.synchronize()
    model.set_placement(new_assign)
    return sum(1 for mv in moves if mv[2] != mv[4])
