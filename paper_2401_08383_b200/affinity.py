"""Affinity statistics and routing replay -- Python mirror of the reference
surface that this framework accelerates (proj/include/exflow/trace.hpp:58-90,
proj/include/exflow/sim.hpp:28-65). Compute goes through the C-ABI
(libexflow_b200.so); only the fp64 post-processing that the reference also
keeps on the host (conditional_probabilities, most_affiliated, the SimReport
ratios) runs here.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from typing import Optional, Sequence

import numpy as np

from . import _capi

VANILLA, COHERENT = 0, 1


@dataclass
class TransitionCounts:
    """proj/include/exflow/trace.hpp:61-69; matrices[j][a, b] (row-major)."""
    num_experts: int
    num_layers: int
    gap: int
    matrices: np.ndarray      # [L-gap][E][E] int64
    row_totals: np.ndarray    # [L-gap][E] int64

    def num_layer_pairs(self) -> int:
        return int(self.matrices.shape[0])


def count_transitions(paths: np.ndarray, num_experts: int, gap: int = 1) -> TransitionCounts:
    """GPU kernel (5) through exf_count_transitions_host.

    Mirrors exflow::count_transitions(trace, gap) (proj/src/trace.cpp:191-215),
    including its std::invalid_argument cases (raised as
    ExflowInvalidArgument with the reference's messages).
    """
    paths = np.ascontiguousarray(paths, dtype=np.int32)
    if paths.ndim != 2:
        raise _capi.ExflowInvalidArgument("paths must be a [T][L] matrix")
    T, L = paths.shape
    pairs = max(L - gap, 1)
    counts = np.zeros((pairs, num_experts, num_experts), np.int64)
    totals = np.zeros((pairs, num_experts), np.int64)
    _capi.call("exf_count_transitions_host", paths.ctypes.data, T, L, num_experts, gap,
               counts.ctypes.data, totals.ctypes.data)
    return TransitionCounts(num_experts, L, gap, counts, totals)


def count_transitions_device(d_paths, T: int, L: int, E: int, gap: int, d_counts, d_totals,
                             d_workspace, stream: int = 0) -> None:
    """Device-pointer entry (torch tensors' data_ptr()); asynchronous on `stream`."""
    _capi.call("exf_count_transitions", d_paths, T, L, E, gap, d_counts, d_totals, d_workspace,
               stream)


def count_transitions_workspace_bytes(T: int, L: int, E: int, gap: int = 1) -> int:
    n = _capi.load().exf_count_transitions_workspace_bytes(T, L, E, gap)
    if n < 0:
        _capi.check(_capi.EXF_INVALID)
    return int(n)


@dataclass
class AffinityMatrix:
    """proj/include/exflow/trace.hpp:76-84."""
    num_experts: int
    num_layers: int
    gap: int
    matrices: np.ndarray  # fp64
    seen: np.ndarray      # bool


def conditional_probabilities(counts: TransitionCounts) -> AffinityMatrix:
    """Host fp64 row normalisation (proj/src/trace.cpp:217-240); unseen rows stay 0."""
    tot = counts.row_totals.astype(np.float64)
    seen = counts.row_totals > 0
    with np.errstate(divide="ignore", invalid="ignore"):
        probs = np.where(seen[:, :, None], counts.matrices / tot[:, :, None], 0.0)
    return AffinityMatrix(counts.num_experts, counts.num_layers, counts.gap, probs, seen)


def most_affiliated(affinity: AffinityMatrix, source_layer: int, expert: int) -> int:
    """proj/src/trace.cpp:242-260 (first maximum = lowest-index tie-break)."""
    pairs = affinity.matrices.shape[0]
    if source_layer < 0 or source_layer >= pairs:
        raise _capi.ExflowInvalidArgument(
            f"source layer {source_layer} out of range [0,{pairs})")
    if expert < 0 or expert >= affinity.num_experts:
        raise _capi.ExflowInvalidArgument(f"expert {expert} out of range")
    if not affinity.seen[source_layer, expert]:
        raise _capi.ExflowInvalidArgument(
            f"no observations for expert {expert} at layer {source_layer}")
    return int(np.argmax(affinity.matrices[source_layer, expert]))


@dataclass
class SimReport:
    """proj/include/exflow/sim.hpp:49-63."""
    hops_intra_node: int
    hops_inter_node: int
    locality_gpu: float
    locality_node: float
    p: float
    p_star: float
    alltoall_count: int
    allgather_count: int
    setup_allgather_count: int
    volume_units: float
    estimated_latency: float

    def total_crossings(self) -> int:
        return self.hops_intra_node + self.hops_inter_node


def token_hops(path, home_gpu: int, assign: np.ndarray, mode: int, topology: "Topology"):
    """exflow::token_hops (proj/src/sim.cpp:34-76) through exf_token_hops:
    per layer (crossed, tier, hops); tier 0 intra-GPU, 1 intra-node, 2 inter-node."""
    p = np.ascontiguousarray(path, dtype=np.int32)
    a = np.ascontiguousarray(assign, dtype=np.int32)
    L = p.shape[0]
    if a.ndim != 2:
        raise _capi.ExflowInvalidArgument("assign must be [L][E]")
    crossed, tier, hops = (np.zeros(L, np.int32) for _ in range(3))
    _capi.call("exf_token_hops", p.ctypes.data, L, home_gpu, a.ctypes.data, a.shape[1],
               topology.num_nodes, topology.gpus_per_node, mode, crossed.ctypes.data,
               tier.ctypes.data, hops.ctypes.data)
    return crossed.astype(bool), tier, hops


@dataclass
class Topology:
    """proj/include/exflow/placement.hpp:16-25."""
    num_nodes: int = 1
    gpus_per_node: int = 1
    intra_node_hop_cost: float = 1.0
    inter_node_hop_cost: float = 4.0

    def total_gpus(self) -> int:
        return self.num_nodes * self.gpus_per_node


@dataclass
class SimConfig:
    """proj/include/exflow/sim.hpp:32-41."""
    mode: int = VANILLA
    topology: Topology = field(default_factory=Topology)
    tokens_per_gpu: int = 1
    iterations: int = 1
    homes: Optional[Sequence[int]] = None


def simulate(paths: np.ndarray, assign: np.ndarray, config: SimConfig) -> SimReport:
    """Routing replay on the GPU (exf_simulate_host); mirrors exflow::simulate
    (proj/src/sim.cpp:78-169) including validation and SimReport derivation."""
    paths = np.ascontiguousarray(paths, dtype=np.int32)
    assign = np.ascontiguousarray(assign, dtype=np.int32)
    if paths.ndim != 2 or assign.ndim != 2:
        raise _capi.ExflowInvalidArgument("paths and assign must be matrices")
    T, L = paths.shape
    if assign.shape[0] != L:
        raise _capi.ExflowInvalidArgument("trace and placement shapes disagree")
    if config.iterations < 1:
        raise _capi.ExflowInvalidArgument("iterations must be >= 1")
    homes_ptr = None
    if config.homes is not None:
        homes = np.ascontiguousarray(config.homes, dtype=np.int32)
        if homes.shape[0] != T:
            raise _capi.ExflowInvalidArgument("homes must list one GPU per token")
        homes_ptr = homes.ctypes.data
    rep = _capi.SimReportC()
    topo = config.topology
    _capi.call("exf_simulate_host", paths.ctypes.data, T, L, assign.shape[1], assign.ctypes.data,
               topo.num_nodes, topo.gpus_per_node, topo.intra_node_hop_cost,
               topo.inter_node_hop_cost, config.tokens_per_gpu, config.mode, homes_ptr,
               C.byref(rep))
    return SimReport(**{f: getattr(rep, f) for f, _ in _capi.SimReportC._fields_})
