"""Teacher-forced CPU oracle of one context-coherent MoE layer across G ranks.

TEST INFRASTRUCTURE ONLY. Given each rank's resident tokens (bf16 bits +
token ids) BEFORE layer j, it reproduces:
  * the gate routing (fixed-order fp32 logits, top-1 lowest-index ties) --
    bit-exact contract with the sm_100a gate kernel;
  * the coherent dispatch rule (proj/src/sim.cpp:65-71): a token moves to the
    GPU of its layer-j expert and stays there; the per-rank canonical order
    after dispatch is (local expert slot, source rank, source order) -- the
    stable bucketing the dispatch kernel implements;
  * the expert FFN (fp64 accumulate) as the tolerance reference.
"""
from __future__ import annotations

import numpy as np

from oracle import oracle as orc


def slots_of(assign_row: np.ndarray, G: int) -> np.ndarray:
    """slot[e] = rank of expert e among the experts placed on its GPU."""
    E = assign_row.shape[0]
    slot = np.zeros(E, np.int32)
    seen = np.zeros(G, np.int32)
    for e in range(E):
        g = assign_row[e]
        slot[e] = seen[g]
        seen[g] += 1
    return slot


def route(x_bits: np.ndarray, wg: np.ndarray, forced=None):
    """Gate routing; with `forced` expert ids the decision is overridden and the
    scale is the softmax probability of the forced expert."""
    logits = orc.gate_logits(x_bits, wg)
    if forced is None:
        return orc.gate_top1(logits)
    e = np.asarray(forced, np.int32)
    z = np.exp(logits.astype(np.float64) - logits.max(axis=1, keepdims=True))
    p = (z[np.arange(len(e)), e] / z.sum(axis=1)).astype(np.float32)
    return e, p


def dispatch(resident, experts, assign_row, G):
    """resident[g] = token ids (in resident order); experts[g] = expert per token.
    Returns per destination rank the canonical list of (src_rank, src_index)."""
    E = assign_row.shape[0]
    E_loc = E // G
    slot = slots_of(assign_row, G)
    out = []
    for p in range(G):
        lst = []
        for s in range(E_loc):
            for g in range(G):
                for i, e in enumerate(experts[g]):
                    if assign_row[e] == p and slot[e] == s:
                        lst.append((g, i))
        out.append(lst)
    return out


def ffn_ref(x_bits_row, weights, prob):
    w1, b1, w2, b2 = weights
    return orc.expert_ffn(x_bits_row, w1, b1, w2, b2, prob)
