"""numpy/ctypes front-end for the CPU oracle (oracle/liboracle.so).

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and
bench.py's cpu_baseline / --impl reference legs. The product package
(paper_2401_08383_b200) never imports this module.

Every wrapper mirrors a reference function; see exflow_oracle.h for the
file:line each C routine restates.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "liboracle.so")
_lib = None

I32P = np.ctypeslib.ndpointer(dtype=np.int32, flags="C_CONTIGUOUS")
I64P = np.ctypeslib.ndpointer(dtype=np.int64, flags="C_CONTIGUOUS")
U16P = np.ctypeslib.ndpointer(dtype=np.uint16, flags="C_CONTIGUOUS")
F32P = np.ctypeslib.ndpointer(dtype=np.float32, flags="C_CONTIGUOUS")
F64P = np.ctypeslib.ndpointer(dtype=np.float64, flags="C_CONTIGUOUS")
U8P = np.ctypeslib.ndpointer(dtype=np.uint8, flags="C_CONTIGUOUS")


class OracleError(ValueError):
    """Mirrors std::invalid_argument raised by the reference validators."""


class _SimReport(C.Structure):
    _fields_ = [
        ("hops_intra_node", C.c_int64),
        ("hops_inter_node", C.c_int64),
        ("gpu_local_events", C.c_int64),
        ("node_local_events", C.c_int64),
        ("away_from_home_events", C.c_int64),
        ("coherent_moves", C.c_int64),
        ("locality_gpu", C.c_double),
        ("locality_node", C.c_double),
        ("p", C.c_double),
        ("p_star", C.c_double),
        ("alltoall_count", C.c_int64),
        ("allgather_count", C.c_int64),
        ("setup_allgather_count", C.c_int64),
        ("volume_units", C.c_double),
        ("estimated_latency", C.c_double),
    ]


def build() -> str:
    """Compile liboracle.so from the C restatement (make in oracle/)."""
    subprocess.run(["make", "-s", "-C", _HERE], check=True)
    return _LIB_PATH


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            build()
        L = C.CDLL(_LIB_PATH)
        L.orc_last_error.restype = C.c_char_p
        L.orc_rng_next.restype = C.c_uint64
        L.orc_rng_below.restype = C.c_uint64
        L.orc_rng_below.argtypes = [C.c_void_p, C.c_uint64]
        L.orc_rng_uniform01.restype = C.c_double
        L.orc_seed_stream.restype = C.c_uint64
        L.orc_seed_stream.argtypes = [C.c_uint64, C.c_uint64]
        L.orc_rng_init.argtypes = [C.c_void_p, C.c_uint64]
        L.orc_rng_next.argtypes = [C.c_void_p]
        L.orc_rng_uniform01.argtypes = [C.c_void_p]
        L.orc_generate_markov_trace.argtypes = [C.c_int32, C.c_int32, C.c_int64, C.c_double,
                                                C.c_int32, C.c_uint64, I32P]
        L.orc_expected_planted_locality.restype = C.c_double
        L.orc_expected_planted_locality.argtypes = [C.c_double, C.c_int32]
        L.orc_count_transitions.argtypes = [I32P, C.c_int64, C.c_int32, C.c_int32, C.c_int32,
                                            I64P, I64P]
        L.orc_count_transitions_mt.argtypes = [I32P, C.c_int64, C.c_int32, C.c_int32, C.c_int32,
                                               I64P, I64P, C.c_int32]
        L.orc_conditional_probabilities.argtypes = [I64P, I64P, C.c_int32, C.c_int32, F64P, U8P]
        L.orc_most_affiliated.argtypes = [F64P, U8P, C.c_int32, C.c_int32, C.c_int32, C.c_int32]
        L.orc_permute_experts.argtypes = [I32P, C.c_int64, C.c_int32, C.c_int32, I32P, I32P]
        L.orc_validate_placement.argtypes = [I32P, C.c_int32, C.c_int32, C.c_int32]
        L.orc_contiguous_placement.argtypes = [C.c_int32, C.c_int32, C.c_int32, I32P]
        L.orc_random_placement.argtypes = [C.c_int32, C.c_int32, C.c_int32, C.c_uint64, I32P]
        L.orc_objective_crossings.restype = C.c_double
        L.orc_objective_crossings.argtypes = [I64P, C.c_int32, C.c_int32, C.c_int32, I32P,
                                              C.c_int32, C.c_int32]
        L.orc_balanced_assignment_count.restype = C.c_int64
        L.orc_balanced_assignment_count.argtypes = [C.c_int32, C.c_int32, C.c_int64]
        L.orc_brute_force_optimum.restype = C.c_double
        L.orc_brute_force_optimum.argtypes = [I64P, C.c_int32, C.c_int32, C.c_int32]
        L.orc_token_hops.argtypes = [I32P, C.c_int32, C.c_int32, I32P, C.c_int32, C.c_int32,
                                     C.c_int32, C.c_int32, I32P, I32P, I32P]
        L.orc_simulate_mt.argtypes = [I32P, C.c_int64, C.c_int32, C.c_int32, I32P, C.c_int32,
                                      C.c_int32, C.c_double, C.c_double, C.c_int32, C.c_int32,
                                      C.c_void_p, C.POINTER(_SimReport), C.c_int32]
        L.orc_volume_table1.restype = C.c_double
        L.orc_volume_table1.argtypes = [C.c_int32, C.c_int32, C.c_int32, C.c_double, C.c_int32,
                                        C.c_int32]
        L.orc_gate_logits.argtypes = [U16P, U16P, C.c_int32, C.c_int32, F32P]
        L.orc_gate_top1.restype = C.c_int
        L.orc_gate_top1.argtypes = [F32P, C.c_int32, C.c_void_p]
        L.orc_expert_ffn.argtypes = [U16P, U16P, U16P, U16P, U16P, C.c_int32, C.c_int32,
                                     C.c_float, C.c_void_p, C.c_void_p]
        L.orc_gate_logits_f32.argtypes = [F32P, F32P, C.c_int32, C.c_int32, F32P]
        L.orc_expert_ffn_f32.argtypes = [F32P, F32P, F32P, F32P, F32P, C.c_int32, C.c_int32,
                                         C.c_float, C.c_void_p]
        _lib = L
    return _lib


def _check(rc: int):
    if rc != 0:
        raise OracleError(lib().orc_last_error().decode())


# ---------------------------------------------------------------- rng
class Rng:
    """proj/include/exflow/rng.hpp:17-66."""

    def __init__(self, seed: int):
        self._state = (C.c_uint64 * 4)()
        lib().orc_rng_init(C.byref(self._state), C.c_uint64(seed & (2**64 - 1)))

    def next(self) -> int:
        return lib().orc_rng_next(C.byref(self._state))

    def below(self, bound: int) -> int:
        return lib().orc_rng_below(C.byref(self._state), bound)

    def below_int(self, bound: int) -> int:
        return int(self.below(bound))

    def uniform01(self) -> float:
        return lib().orc_rng_uniform01(C.byref(self._state))

    def shuffle(self, values: list) -> None:
        for i in range(len(values), 1, -1):
            j = self.below(i)
            values[i - 1], values[j] = values[j], values[i - 1]


def seed_stream(seed: int, stream: int) -> int:
    return lib().orc_seed_stream(seed, stream)


# ---------------------------------------------------------------- synth / trace
def generate_markov_trace(num_experts, num_layers, num_tokens, affinity_strength,
                          planted_groups, seed) -> np.ndarray:
    """proj/src/synth.cpp:30-53 -> paths [T][L] int32."""
    out = np.empty((num_tokens, num_layers), dtype=np.int32)
    _check(lib().orc_generate_markov_trace(num_experts, num_layers, num_tokens,
                                           affinity_strength, planted_groups, seed, out))
    return out


def expected_planted_locality(alpha, groups) -> float:
    return lib().orc_expected_planted_locality(alpha, groups)


def count_transitions(paths: np.ndarray, num_experts: int, gap: int = 1, threads: int = 1):
    """proj/src/trace.cpp:191-215 -> (counts [L-gap][E][E] int64, row_totals [L-gap][E])."""
    paths = np.ascontiguousarray(paths, dtype=np.int32)
    T, L = paths.shape
    pairs = max(L - gap, 1)
    counts = np.zeros((pairs, num_experts, num_experts), dtype=np.int64)
    totals = np.zeros((pairs, num_experts), dtype=np.int64)
    _check(lib().orc_count_transitions_mt(paths, T, L, num_experts, gap, counts, totals,
                                          threads))
    return counts, totals


def conditional_probabilities(counts: np.ndarray, row_totals: np.ndarray):
    """proj/src/trace.cpp:217-240 -> (probs fp64, seen bool)."""
    pairs, E, _ = counts.shape
    probs = np.zeros(counts.shape, dtype=np.float64)
    seen = np.zeros((pairs, E), dtype=np.uint8)
    lib().orc_conditional_probabilities(np.ascontiguousarray(counts),
                                        np.ascontiguousarray(row_totals), pairs, E, probs, seen)
    return probs, seen.astype(bool)


def most_affiliated(probs, seen, source_layer, expert) -> int:
    pairs, E, _ = probs.shape
    r = lib().orc_most_affiliated(np.ascontiguousarray(probs),
                                  np.ascontiguousarray(seen.astype(np.uint8)), pairs, E,
                                  source_layer, expert)
    if r < 0:
        raise OracleError(lib().orc_last_error().decode())
    return r


def export_heatmap_csv(probs, source_layer) -> str:
    """proj/src/trace.cpp:262-283 (%.6f, comma-separated, one row per line)."""
    if source_layer < 0 or source_layer >= probs.shape[0]:
        raise OracleError("source layer out of range")
    return "".join(",".join("%.6f" % v for v in row) + "\n" for row in probs[source_layer])


def permute_experts(paths, num_experts, perm) -> np.ndarray:
    paths = np.ascontiguousarray(paths, dtype=np.int32)
    out = np.empty_like(paths)
    _check(lib().orc_permute_experts(paths, paths.shape[0], paths.shape[1], num_experts,
                                     np.ascontiguousarray(perm, dtype=np.int32), out))
    return out


# ---------------------------------------------------------------- placement
def contiguous_placement(num_experts, num_layers, gpus) -> np.ndarray:
    a = np.empty((num_layers, num_experts), dtype=np.int32)
    _check(lib().orc_contiguous_placement(num_experts, num_layers, gpus, a))
    return a


def random_placement(num_experts, num_layers, gpus, seed) -> np.ndarray:
    a = np.empty((num_layers, num_experts), dtype=np.int32)
    _check(lib().orc_random_placement(num_experts, num_layers, gpus, seed, a))
    return a


def validate_placement(assign, gpus) -> None:
    assign = np.ascontiguousarray(assign, dtype=np.int32)
    _check(lib().orc_validate_placement(assign, assign.shape[0], assign.shape[1], gpus))


def objective_crossings(counts, assign, gap=1, gpus_per_node=1, level_node=False) -> float:
    counts = np.ascontiguousarray(counts, dtype=np.int64)
    return lib().orc_objective_crossings(counts, counts.shape[0], counts.shape[1], gap,
                                         np.ascontiguousarray(assign, dtype=np.int32),
                                         gpus_per_node, int(level_node))


def balanced_assignment_count(items, parts, cap=10000) -> int:
    return lib().orc_balanced_assignment_count(items, parts, cap)


def brute_force_optimum(counts, parts) -> float:
    counts = np.ascontiguousarray(counts, dtype=np.int64)
    return lib().orc_brute_force_optimum(counts, counts.shape[0] + 1, counts.shape[1], parts)


# ---------------------------------------------------------------- simulator
VANILLA, COHERENT = 0, 1


@dataclass
class SimReport:
    hops_intra_node: int
    hops_inter_node: int
    gpu_local_events: int
    node_local_events: int
    away_from_home_events: int
    coherent_moves: int
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


def token_hops(path, home, assign, num_nodes, gpus_per_node, mode):
    path = np.ascontiguousarray(path, dtype=np.int32)
    assign = np.ascontiguousarray(assign, dtype=np.int32)
    L = path.shape[0]
    if assign.shape[0] != L:
        raise OracleError("path length does not match placement layers")
    hops = np.zeros(L, np.int32)
    crossed = np.zeros(L, np.int32)
    tier = np.zeros(L, np.int32)
    _check(lib().orc_token_hops(path, L, home, assign, assign.shape[1], num_nodes,
                                gpus_per_node, mode, hops, crossed, tier))
    return hops, crossed, tier


def simulate(paths, assign, num_nodes=1, gpus_per_node=1, mode=COHERENT, homes=None,
             intra_cost=1.0, inter_cost=4.0, tokens_per_gpu=1, threads=1) -> SimReport:
    """proj/src/sim.cpp:78-169."""
    paths = np.ascontiguousarray(paths, dtype=np.int32)
    assign = np.ascontiguousarray(assign, dtype=np.int32)
    T, L = paths.shape
    if assign.shape[0] != L:
        raise OracleError("trace and placement shapes disagree")
    rep = _SimReport()
    hp = None
    if homes is not None:
        homes = np.ascontiguousarray(homes, dtype=np.int32)
        if homes.shape[0] != T:
            raise OracleError("homes must list one GPU per token")
        hp = homes.ctypes.data_as(C.c_void_p)
    _check(lib().orc_simulate_mt(paths, T, L, assign.shape[1], assign, num_nodes, gpus_per_node,
                                 intra_cost, inter_cost, tokens_per_gpu, mode, hp, C.byref(rep),
                                 threads))
    return SimReport(**{f: getattr(rep, f) for f, _ in _SimReport._fields_})


def volume_table1(gpus, tokens_per_gpu, layers, ratio, gating=0, method=0) -> float:
    v = lib().orc_volume_table1(gpus, tokens_per_gpu, layers, ratio, gating, method)
    if v != v:
        raise OracleError("volume arguments out of range")
    return v


# ---------------------------------------------------------------- model oracle
def bf16_bits_to_f32(a: np.ndarray) -> np.ndarray:
    return (np.asarray(a, dtype=np.uint16).astype(np.uint32) << 16).view(np.float32)


def f32_to_bf16_bits(a: np.ndarray) -> np.ndarray:
    u = np.ascontiguousarray(a, dtype=np.float32).view(np.uint32).astype(np.uint64)
    r = ((u + 0x7FFF + ((u >> 16) & 1)) >> 16).astype(np.uint16)
    return r


def gate_logits(x_bits: np.ndarray, wg_bits: np.ndarray) -> np.ndarray:
    """Fixed-order fp32 gate logits (see exflow_model_oracle.c). x [n][d], wg [E][d]."""
    x_bits = np.ascontiguousarray(x_bits, dtype=np.uint16)
    wg_bits = np.ascontiguousarray(wg_bits, dtype=np.uint16)
    n, d = x_bits.shape
    E = wg_bits.shape[0]
    out = np.empty((n, E), np.float32)
    row = np.empty(E, np.float32)
    for t in range(n):
        lib().orc_gate_logits(np.ascontiguousarray(x_bits[t]), wg_bits, d, E, row)
        out[t] = row
    return out


def gate_logits_f32(x: np.ndarray, wg: np.ndarray) -> np.ndarray:
    """fp32-mode gate logits: the fixed fmaf order on fp32 inputs. x [n][d], wg [E][d]."""
    x = np.ascontiguousarray(x, dtype=np.float32)
    wg = np.ascontiguousarray(wg, dtype=np.float32)
    n, d = x.shape
    E = wg.shape[0]
    out = np.empty((n, E), np.float32)
    row = np.empty(E, np.float32)
    for t in range(n):
        lib().orc_gate_logits_f32(np.ascontiguousarray(x[t]), wg, d, E, row)
        out[t] = row
    return out


def expert_ffn_f32(x, w1, b1, w2, b2, prob) -> np.ndarray:
    """One fp32 token through one fp32 expert, evaluated in fp64: [d] float64."""
    d = x.shape[0]
    dff = w1.shape[0]
    out = np.empty(d, np.float64)
    f = lambda a: np.ascontiguousarray(a, dtype=np.float32)
    lib().orc_expert_ffn_f32(f(x), f(w1), f(b1), f(w2), f(b2), d, dff, float(prob),
                             out.ctypes.data_as(C.c_void_p))
    return out


def gate_top1(logits: np.ndarray):
    """argmax (lowest index on ties) + softmax prob of the winner."""
    n, E = logits.shape
    idx = np.empty(n, np.int32)
    prob = np.empty(n, np.float32)
    p = C.c_float()
    for t in range(n):
        idx[t] = lib().orc_gate_top1(np.ascontiguousarray(logits[t]), E, C.byref(p))
        prob[t] = p.value
    return idx, prob


def expert_ffn(x_bits, w1, b1, w2, b2, prob):
    """One token through one expert: returns (bf16 bits, fp32 value) [d]."""
    d = x_bits.shape[0]
    dff = w1.shape[0]
    out = np.empty(d, np.uint16)
    outf = np.empty(d, np.float32)
    lib().orc_expert_ffn(np.ascontiguousarray(x_bits, dtype=np.uint16),
                         np.ascontiguousarray(w1, dtype=np.uint16),
                         np.ascontiguousarray(b1, dtype=np.uint16),
                         np.ascontiguousarray(w2, dtype=np.uint16),
                         np.ascontiguousarray(b2, dtype=np.uint16), d, dff, float(prob),
                         out.ctypes.data_as(C.c_void_p), outf.ctypes.data_as(C.c_void_p))
    return out, outf
