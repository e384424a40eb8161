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
    def __init__(self, E, L, d, dff, tokens, G, assign, seed=0, layers=None):
        self.E, self.L, self.d, self.dff, self.T, self.G = E, L, d, dff, tokens, G
        self.assign = np.ascontiguousarray(assign, np.int32)
        self.layers = list(range(L)) if layers is None else list(layers)
        rng = np.random.default_rng(seed)
        self.wg = {j: (rng.standard_normal((E, d), dtype=np.float32) / math.sqrt(d))
                   for j in self.layers}
        self.w1 = {}
        self.w2 = {}
        self.b1 = {}
        self.b2 = {}
        for j in self.layers:
            self.w1[j] = [rng.standard_normal((dff, d), dtype=np.float32) * 0.02 for _ in range(E)]
            self.w2[j] = [rng.standard_normal((d, dff), dtype=np.float32) * 0.02 for _ in range(E)]
            self.b1[j] = [rng.standard_normal(dff, dtype=np.float32) * 0.02 for _ in range(E)]
            self.b2[j] = [rng.standard_normal(d, dtype=np.float32) * 0.02 for _ in range(E)]
        self.slot = np.zeros_like(self.assign)
        for j in range(L):
            seen = np.zeros(G, np.int32)
            for e in range(E):
                g = self.assign[j, e]
                self.slot[j, e] = seen[g]
                seen[g] += 1

    def step(self, x: np.ndarray, threads: int):
        """One decode step over all G*B tokens; returns (x_out, routes)."""
        T = self.T
        routes = np.zeros((T, self.L), np.int32)
        loc = np.arange(T) % self.G
        for j in self.layers:
            logits = x @ self.wg[j].T
            e = np.argmax(logits, axis=1).astype(np.int32)   # first max = lowest index
            z = np.exp(logits - logits.max(axis=1, keepdims=True))
            prob = 1.0 / z.sum(axis=1)
            routes[:, j] = e
            dest = self.assign[j][e]
            # coherent dispatch: stable bucketing by (destination GPU, local slot)
            order = np.lexsort((np.arange(T), self.slot[j][e], dest))
            loc = dest
            xs = x[order]
            es = e[order]
            out = np.empty_like(xs)
            for ex in range(self.E):
                sel = np.nonzero(es == ex)[0]
                if sel.size == 0:
                    continue
                h = _gelu(xs[sel] @ self.w1[j][ex].T + self.b1[j][ex])
                y = h @ self.w2[j][ex].T + self.b2[j][ex]
                out[sel] = xs[sel] + prob[order][sel, None] * y
            x = np.empty_like(out)
            x[order] = out
        # the reference's own CPU path on this step's routes: affinity
        # histogram + coherent replay (C restatement, integer sums)
        counts, _ = orc.count_transitions(routes, self.E, 1, threads=threads)
        rep = orc.simulate(routes, self.assign, 1, self.G, orc.COHERENT, threads=threads)
        return x, routes, counts, rep


def time_cpu_path(E, L, d, dff, tokens, G, assign, layers_sample, steps, seed=0):
    """Times `steps` steps over `layers_sample` of the L layers; returns
    (tokens_per_s extrapolated to all L layers, seconds measured, sample str, threads)."""
    threads = os.cpu_count() or 1
    layers = list(range(min(layers_sample, L)))
    path = CpuDecodePath(E, L, d, dff, tokens, G, assign, seed, layers)
    rng = np.random.default_rng(seed + 1)
    x = rng.standard_normal((tokens, d), dtype=np.float32)
    path.step(x, threads)  # warm-up (BLAS threads, page faults)
    t0 = time.perf_counter()
    for _ in range(steps):
        path.step(x, threads)
    dt = time.perf_counter() - t0
    per_step_full = dt / steps * (L / len(layers))
    sample = (f"{steps} steps x {len(layers)}/{L} layers x {tokens} tokens (numpy fp32 gate+FFN, "
              f"C oracle histogram+replay), extrapolated linearly to {L} layers")
    return tokens / per_step_full, dt, sample, threads


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
