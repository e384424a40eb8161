"""CPU implementation of the whole ExFlow decode path, for the baseline arm.

TEST/BENCH INFRASTRUCTURE ONLY (bench.py cpu_baseline leg and --impl
reference). The reference itself implements only the routing bookkeeping of
this path on the CPU -- count_transitions (proj/src/trace.cpp:191-215) and
the coherent replay of simulate (proj/src/sim.cpp:110-145) -- which run here
through the C restatement (liboracle.so, multi-threaded integer-sum variant
allowed by SPEC.md:102/:339). The gate and expert FFN that the reference
leaves out are a numpy fp32 port (multi-threaded BLAS),
so the CPU number covers the same work per token as the GPU path:
  gate GEMM + softmax/top-1 -> affinity histogram -> coherent dispatch
  (stable bucketing by destination GPU / expert) -> grouped expert FFN
  (GELU, residual, gate-prob scale) for every layer.
"""
from __future__ import annotations

import math
import os
import time

import numpy as np

from . import oracle as orc


def _gelu(v: np.ndarray) -> np.ndarray:
    # erf GELU (same activation as the GPU path), vectorised
    from scipy.special import erf
    return 0.5 * v * (1.0 + erf(v * (1.0 / math.sqrt(2.0))))


class CpuDecodePath:
    """Every one of the L layers runs each step. To bound host memory, the
    expert weights come from `weight_sets` distinct sets (layer j uses set
    j % weight_sets; each set is E x 2 x d x dff fp32, far larger than the
    CPU caches, so nothing is served from cache that HBM-sized weights would
    not be)."""

    def __init__(self, E, L, d, dff, tokens, G, assign, seed=0, weight_sets=2):
        self.E, self.L, self.d, self.dff, self.T, self.G = E, L, d, dff, tokens, G
        self.assign = np.ascontiguousarray(assign, np.int32)
        rng = np.random.default_rng(seed)
        self.wg = [rng.standard_normal((E, d), dtype=np.float32) / math.sqrt(d) for _ in range(L)]
        nset = max(1, min(weight_sets, L))
        sets = []
        for _ in range(nset):
            sets.append(([rng.standard_normal((dff, d), dtype=np.float32) * 0.02 for _ in range(E)],
                         [rng.standard_normal(dff, dtype=np.float32) * 0.02 for _ in range(E)],
                         [rng.standard_normal((d, dff), dtype=np.float32) * 0.02 for _ in range(E)],
                         [rng.standard_normal(d, dtype=np.float32) * 0.02 for _ in range(E)]))
        self.w = [sets[j % nset] for j in range(L)]
        self.slot = np.zeros_like(self.assign)
        for j in range(L):
            seen = np.zeros(G, np.int32)
            for e in range(E):
                g = self.assign[j, e]
                self.slot[j, e] = seen[g]
                seen[g] += 1

    def step(self, x: np.ndarray, threads: int):
        """One decode step over all G*B tokens and all L layers; returns
        (x_out, routes, counts, report)."""
        T = self.T
        routes = np.zeros((T, self.L), np.int32)
        for j in range(self.L):
            w1, b1, w2, b2 = self.w[j]
            logits = x @ self.wg[j].T
            e = np.argmax(logits, axis=1).astype(np.int32)   # first max = lowest index
            z = np.exp(logits - logits.max(axis=1, keepdims=True))
            prob = 1.0 / z.sum(axis=1)
            routes[:, j] = e
            dest = self.assign[j][e]
            # coherent dispatch: stable bucketing by (destination GPU, local slot)
            order = np.lexsort((np.arange(T), self.slot[j][e], dest))
            xs = x[order]
            es = e[order]
            out = np.empty_like(xs)
            for ex in range(self.E):
                sel = np.nonzero(es == ex)[0]
                if sel.size == 0:
                    continue
                h = _gelu(xs[sel] @ w1[ex].T + b1[ex])
                y = h @ w2[ex].T + b2[ex]
                out[sel] = xs[sel] + prob[order][sel, None] * y
            x = np.empty_like(out)
            x[order] = out
        # the reference's own CPU path on this step's routes: affinity
        # histogram + coherent replay (C restatement, integer sums)
        counts, _ = orc.count_transitions(routes, self.E, 1, threads=threads)
        rep = orc.simulate(routes, self.assign, 1, self.G, orc.COHERENT, threads=threads)
        return x, routes, counts, rep


def time_cpu_path(E, L, d, dff, tokens, G, assign, steps=None, seed=0, min_seconds=8.0,
                  max_steps=20):
    """Times whole decode steps (all L layers, nothing extrapolated): at least
    `steps` steps if given, else as many as fit `min_seconds` (>= 1, <=
    max_steps). Returns (tokens_per_s, seconds measured, sample str, threads,
    steps timed)."""
    threads = os.cpu_count() or 1
    # BLAS on every host core even under torchrun, which exports
    # OMP_NUM_THREADS=1 to each rank (the CPU baseline would otherwise run
    # single-threaded at N > 1)
    try:
        from threadpoolctl import threadpool_limits
        limiter = threadpool_limits(limits=threads)
    except Exception:  # threadpoolctl absent: the environment's setting stands
        limiter = None
    try:
        return _time_steps(E, L, d, dff, tokens, G, assign, steps, seed, min_seconds, max_steps, threads)
    finally:
        if limiter is not None:
            limiter.restore_original_limits()


def _time_steps(E, L, d, dff, tokens, G, assign, steps, seed, min_seconds, max_steps, threads):
    path = CpuDecodePath(E, L, d, dff, tokens, G, assign, seed)
    rng = np.random.default_rng(seed + 1)
    x = rng.standard_normal((tokens, d), dtype=np.float32)
    path.step(x, threads)  # warm-up (BLAS threads, page faults)
    n = 0
    t0 = time.perf_counter()
    while True:
        path.step(x, threads)
        n += 1
        dt = time.perf_counter() - t0
        if (steps is not None and n >= steps) or (steps is None and (dt >= min_seconds or n >= max_steps)):
            break
    sample = (f"{n} full decode steps x {L}/{L} layers x {tokens} tokens (numpy fp32 gate+FFN on "
              f"{threads} threads, C oracle histogram+replay); no extrapolation")
    return n * tokens / dt, dt, sample, threads, n


def time_reference_routing(paths: np.ndarray, E: int, assign: np.ndarray, G: int, threads: int,
                           min_seconds: float = 2.0):
    """The reference's own CPU path alone (count_transitions + coherent
    simulate on the given trace): tokens/s."""
    T = paths.shape[0]
    n = 0
    t0 = time.perf_counter()
    while True:
        orc.count_transitions(paths, E, 1, threads=threads)
        orc.simulate(paths, assign, 1, G, orc.COHERENT, threads=threads)
        n += 1
        dt = time.perf_counter() - t0
        if dt >= min_seconds:
            break
    return n * T / dt
