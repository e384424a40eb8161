"""CPU oracle for coherent decode attention (exf_coherent_attention).

TEST INFRASTRUCTURE ONLY: imported by tests/ and tools/ as the checker; the
product package never imports it.

The reference has no attention code; the protocol is
PAPER.md:180-184: every GPU holds the replicated context (one AllGather per
step, proj/src/sim.cpp:161-162), so a token attends over its own sequence's
cache rows wherever the dispatch left it. Parity is therefore pinned only by
this restatement of standard softmax attention (fp64 on the bf16 inputs).
"""
from __future__ import annotations

import numpy as np


def bf16_round(x: np.ndarray) -> np.ndarray:
    """Round fp32 to bf16 (nearest-even) and return as fp32."""
    u = np.ascontiguousarray(x, np.float32).view(np.uint32).astype(np.uint64)
    u = ((u + 0x7FFF + ((u >> 16) & 1)) >> 16) << 16
    return u.astype(np.uint32).view(np.float32)


def coherent_attention(q, seq, ctx_len, k, v, scale):
    """q [N][H][Dh], seq [N], ctx_len [S], k/v [S][H][C][Dh] (float arrays
    holding bf16 values) -> out [N][H][Dh] fp64. Empty context -> 0."""
    N, H, Dh = q.shape
    out = np.zeros((N, H, Dh), np.float64)
    for n in range(N):
        s = int(seq[n])
        L = int(ctx_len[s])
        if L == 0:
            continue
        kk = k[s, :, :L, :].astype(np.float64)          # [H][L][Dh]
        vv = v[s, :, :L, :].astype(np.float64)
        sc = np.einsum("hd,hld->hl", q[n].astype(np.float64), kk) * scale
        sc -= sc.max(axis=1, keepdims=True)
        p = np.exp(sc)
        p /= p.sum(axis=1, keepdims=True)
        out[n] = np.einsum("hl,hld->hd", p, vv)
    return out


def kv_append(k_new, v_new, seq, k_cache, v_cache, ctx_len):
    """In-place restatement of exf_kv_append on one replica (numpy arrays).
    Returns the number of tokens skipped because their sequence was full."""
    C = k_cache.shape[2]
    overflow = 0
    for n in range(k_new.shape[0]):
        s = int(seq[n])
        pos = int(ctx_len[s])
        if pos >= C:
            overflow += 1
            continue
        k_cache[s, :, pos, :] = k_new[n]
        v_cache[s, :, pos, :] = v_new[n]
        ctx_len[s] = pos + 1
    return overflow
