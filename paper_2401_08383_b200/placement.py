"""Expert-placement table and the host (CPU) integer-program placement solver.

Python mirror of proj/include/exflow/placement.hpp over the C-ABI
(libexflow_b200.so, csrc/host/placement.cpp). Placements are [L][E] int32
arrays of GPU ids; counts are gap-1 transition counts [L-1][E][E] int64 (the
GPU histogram's output).
"""
from __future__ import annotations

import ctypes as C
import json
from dataclasses import dataclass
from typing import Optional

import numpy as np

from . import _capi
from .affinity import Topology

NODE, GPU = 0, 1
DEFAULT_STATE_CAP = 10000


@dataclass
class AnnealParams:
    """proj/include/exflow/placement.hpp:106-114."""
    restarts: int = 8
    max_iters: int = 0
    initial_temperature: float = 0.0
    cooling: float = 0.999
    seed: int = 0

    def _c(self) -> _capi.AnnealParamsC:
        return _capi.AnnealParamsC(self.restarts, self.max_iters, self.initial_temperature,
                                   self.cooling, self.seed)


@dataclass
class SolveReport:
    """proj/include/exflow/placement.hpp:120-130."""
    solver: str
    objective: float
    seed: int
    iterations: int
    restarts: int
    optimality_gap: Optional[float] = None
    inter_node_crossings: Optional[float] = None
    intra_node_crossings: Optional[float] = None
    weighted_cost: Optional[float] = None


def _report(r: _capi.SolveReportC) -> SolveReport:
    return SolveReport(r.solver.decode(), r.objective, r.seed, r.iterations, r.restarts,
                       r.optimality_gap if r.has_optimality_gap else None,
                       r.inter_node_crossings if r.has_tiers else None,
                       r.intra_node_crossings if r.has_tiers else None,
                       r.weighted_cost if r.has_tiers else None)


def _counts(counts) -> np.ndarray:
    c = np.ascontiguousarray(getattr(counts, "matrices", counts), dtype=np.int64)
    if c.ndim != 3 or c.shape[1] != c.shape[2]:
        raise _capi.ExflowInvalidArgument("counts must be [L-1][E][E]")
    if getattr(counts, "gap", 1) != 1:
        raise _capi.ExflowInvalidArgument("placement solving requires gap-1 transition counts")
    return c


def contiguous_placement(num_experts: int, num_layers: int, topology: Topology) -> np.ndarray:
    """Vanilla placement: expert i -> GPU i/(E/G) (proj/src/placement.cpp:482-502)."""
    a = np.empty((num_layers, num_experts), np.int32)
    _capi.call("exf_contiguous_placement", num_experts, num_layers, topology.num_nodes,
               topology.gpus_per_node, a.ctypes.data)
    return a


def random_placement(num_experts, num_layers, topology: Topology, seed: int) -> np.ndarray:
    a = np.empty((num_layers, num_experts), np.int32)
    _capi.call("exf_random_placement", num_experts, num_layers, topology.num_nodes,
               topology.gpus_per_node, seed, a.ctypes.data)
    return a


def validate_placement(assign: np.ndarray, topology: Topology) -> None:
    a = np.ascontiguousarray(assign, dtype=np.int32)
    _capi.call("exf_validate_placement", a.ctypes.data, a.shape[0], a.shape[1],
               topology.num_nodes, topology.gpus_per_node)


def objective_crossings(counts, assign, topology: Topology = Topology(), level: int = GPU,
                        gap: int = 1) -> float:
    c = np.ascontiguousarray(getattr(counts, "matrices", counts), dtype=np.int64)
    a = np.ascontiguousarray(assign, dtype=np.int32)
    out = C.c_double()
    _capi.call("exf_objective_crossings", c.ctypes.data, a.shape[0], a.shape[1], gap,
               a.ctypes.data, topology.num_nodes, topology.gpus_per_node, level, C.byref(out))
    return out.value


def balanced_assignment_count(items: int, parts: int, cap: int = DEFAULT_STATE_CAP) -> int:
    n = _capi.load().exf_balanced_assignment_count(items, parts, cap)
    if n < 0:
        _capi.check(_capi.EXF_INVALID)
    return int(n)


def solve_exact_dp(counts, partitions: int, state_cap: int = DEFAULT_STATE_CAP):
    c = _counts(counts)
    a = np.empty((c.shape[0] + 1, c.shape[1]), np.int32)
    rep = _capi.SolveReportC()
    _capi.call("exf_solve_exact_dp", c.ctypes.data, c.shape[0] + 1, c.shape[1], partitions,
               state_cap, a.ctypes.data, C.byref(rep))
    return a, _report(rep)


def solve_local_search(counts, partitions: int, params: AnnealParams = AnnealParams()):
    c = _counts(counts)
    a = np.empty((c.shape[0] + 1, c.shape[1]), np.int32)
    rep = _capi.SolveReportC()
    p = params._c()
    _capi.call("exf_solve_local_search", c.ctypes.data, c.shape[0] + 1, c.shape[1], partitions,
               C.byref(p), a.ctypes.data, C.byref(rep))
    return a, _report(rep)


def solve_staged(counts, topology: Topology, params: AnnealParams = AnnealParams(),
                 state_cap: int = DEFAULT_STATE_CAP):
    """Affinity placement from gap-1 counts (proj/src/placement.cpp:720-821)."""
    c = _counts(counts)
    a = np.empty((c.shape[0] + 1, c.shape[1]), np.int32)
    rep = _capi.SolveReportC()
    p = params._c()
    _capi.call("exf_solve_staged", c.ctypes.data, c.shape[0] + 1, c.shape[1], topology.num_nodes,
               topology.gpus_per_node, topology.intra_node_hop_cost,
               topology.inter_node_hop_cost, C.byref(p), state_cap, a.ctypes.data, C.byref(rep))
    return a, _report(rep)


def generate_markov_trace(num_experts, num_layers, num_tokens, affinity_strength,
                          planted_groups, seed) -> np.ndarray:
    """Seeded forced-routing workload (proj/src/synth.cpp:30-53), host C++."""
    out = np.empty((num_tokens, num_layers), np.int32)
    _capi.call("exf_generate_markov_trace", num_experts, num_layers, num_tokens,
               affinity_strength, planted_groups, seed, out.ctypes.data)
    return out


def placement_to_json(assign: np.ndarray, topology: Topology) -> str:
    """Placement JSON (proj/src/json_io.cpp:30-43)."""
    return json.dumps({"experts": int(assign.shape[1]), "layers": int(assign.shape[0]),
                       "nodes": topology.num_nodes, "gpus_per_node": topology.gpus_per_node,
                       "assign": assign.tolist()})


def placement_from_json(text: str):
    """proj/src/json_io.cpp:45-64: returns (assign, topology); validates balance."""
    j = json.loads(text)
    topo = Topology(int(j["nodes"]), int(j["gpus_per_node"]))
    assign = np.array(j["assign"], dtype=np.int32)
    if assign.shape[0] != int(j["layers"]):
        raise _capi.ExflowInvalidArgument("placement assign table has wrong layer count")
    if assign.ndim != 2 or assign.shape[1] != int(j["experts"]):
        raise _capi.ExflowInvalidArgument("placement assign row has wrong expert count")
    validate_placement(assign, topo)
    return assign, topo
