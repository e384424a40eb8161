"""Host-side multi-rank plumbing over torch.distributed (one process per GPU).

Only control-plane traffic goes through torch.distributed: the 64-byte CUDA
IPC handles of every rank's symmetric receive region, the exact int64 sum of
the per-rank affinity histograms, and the placement agreed from it. The data
path (dispatch, AllGather) is the P2P kernels in libexflow_b200.so.
Works with NCCL (GPU) and gloo (CPU tests) process groups.
"""
from __future__ import annotations

from typing import List, Sequence

import numpy as np


def _dist():
    import torch.distributed as dist
    return dist


def exchange_handles(handle: bytes, group=None) -> List[bytes]:
    """All-gather the 64-byte IPC handle of every rank, in rank order."""
    dist = _dist()
    if len(handle) != 64:
        raise ValueError("an IPC handle is 64 bytes")
    out = [None] * dist.get_world_size(group)
    dist.all_gather_object(out, handle, group=group)
    return out


def sum_counts(counts: np.ndarray, group=None, device=None) -> np.ndarray:
    """Exact int64 sum of per-rank histograms (order-independent, bit-exact)."""
    import torch
    dist = _dist()
    t = torch.from_numpy(np.ascontiguousarray(counts, dtype=np.int64))
    if device is not None:
        t = t.to(device)
    dist.all_reduce(t, group=group)
    return t.cpu().numpy()


def agree_placement(counts: np.ndarray, topology, params=None, group=None) -> np.ndarray:
    """Rank 0 solves solve_staged on the global histogram (CPU) and broadcasts
    the [L][E] placement so every rank loads the same expert table."""
    from . import placement as pl
    dist = _dist()
    payload = [None]
    if dist.get_rank(group) == 0:
        assign, report = pl.solve_staged(counts, topology, params or pl.AnnealParams())
        payload = [(assign.tolist(), report.objective)]
    dist.broadcast_object_list(payload, src=0, group=group)
    return np.asarray(payload[0][0], dtype=np.int32)


def merge_routes(routes: np.ndarray, group=None) -> np.ndarray:
    """Union of the per-rank token-indexed route tables (-1 = not seen here)."""
    dist = _dist()
    allr = [None] * dist.get_world_size(group)
    dist.all_gather_object(allr, np.ascontiguousarray(routes))
    return np.max(np.stack(allr), axis=0)


def max_over_ranks(value: float, group=None, device=None) -> float:
    import torch
    dist = _dist()
    t = torch.tensor([value], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
    return float(t.item())
