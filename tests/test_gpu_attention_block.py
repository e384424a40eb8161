"""The coherent attention block inside the decode step (
PAPER.md:180-184) against the CPU oracle, teacher-forced per layer:

  * setup AllGather: after exf_model_context_setup every replica holds the
    same prompt K/V for every sequence and the length is the prompt length;
  * K/V append (the per-step context AllGather of the new tokens): the row
    written at position len of every replica equals the oracle projection
    k, v = x Wk^T + bk, x Wv^T + bv (bf16, <= 1e-2 relative), identical on
    every replica, and every length advances by one per step;
  * attention + output projection: the post-attention token state equals
    x + softmax(q K^T / sqrt(Dh)) V Wo^T + bo over the token's own sequence
    in the local replica (fp64 oracle on the bf16 operands, <= 1e-2 relative);
  * the MoE layer that follows routes the post-attention states exactly as
    the oracle gate does (bit-exact) and its outputs stay within 1e-2.
Shapes: one GPU on the fused MoE path, and two lock-step ranks on one GPU
(two-kernel MoE path) whose tokens move between ranks, so attention runs on
the GPU the dispatch left each token on.
"""
import numpy as np
import pytest

import coherent_oracle as co
from oracle import attention as oatt

pytestmark = pytest.mark.gpu

REL_TOL = 1e-2


def _bf(a):
    return co.orc.bf16_bits_to_f32(a).astype(np.float64)


def _rel(a, b):
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-30))


def _models(G, assign, **kw):
    from paper_2401_08383_b200.model import MoeModel, MoeModelConfig
    models = [MoeModel(MoeModelConfig(world_size=G, rank=r, **kw), assign) for r in range(G)]
    if G > 1:
        MoeModel.connect_local(models)
    return models


def run_attention_checked(torch, models, assign, steps=2, seed=0):
    from paper_2401_08383_b200.model import (PHASE_ATTN, PHASE_BEGIN, PHASE_DISPATCH, PHASE_FFN, PHASE_FUSED,
                                             PHASE_GATHER_SEND, PHASE_GATHER_WAIT)
    cfg = models[0].config
    G, L, d, H = cfg.world_size, cfg.num_layers, cfg.d_model, cfg.attn_heads
    Dh = d // H
    fused = G == 1 and models[0].describe().get("path") == "fused"
    for m in models:
        m.context_setup(phase=1)
    for m in models:
        m.context_setup(phase=2)
    torch.cuda.synchronize()
    P = cfg.context_prefix
    # setup AllGather: every replica identical, lengths = prompt
    for j in range(L):
        for m in models:
            assert (m.kv_len(j) == P).all()
    for s in (0, cfg.capacity - 1):
        ref = models[0].kv_rows(L - 1, s, 0, P)
        for m in models[1:]:
            got = m.kv_rows(L - 1, s, 0, P)
            assert np.array_equal(got[0], ref[0]) and np.array_equal(got[1], ref[1])
    g = torch.Generator().manual_seed(seed)
    for step in range(steps):
        xs = [torch.randn(cfg.tokens_per_gpu, d, generator=g).to(torch.bfloat16).cuda() for _ in models]
        for m in models:
            m.reset_stats()
        for r, m in enumerate(models):
            m.phase(PHASE_BEGIN, 0, xs[r])
        for j in range(L):
            pos = P + step  # position of this step's row in every sequence
            before = [m.resident(j % 2) for m in models]
            for m in models:
                m.phase(PHASE_ATTN, j)
            torch.cuda.synchronize()
            mid = [m.resident(j % 2) for m in models]
            wqkv, bqkv, wo, bo = (_bf(w) for w in models[0].attn_weights(j))
            for r in range(G):
                xb, meta = before[r]
                xm, meta_m = mid[r]
                assert np.array_equal(meta[:, 0], meta_m[:, 0])
                qkv = _bf(xb) @ wqkv.T + bqkv
                qkv = co.orc.bf16_bits_to_f32(co.orc.f32_to_bf16_bits(qkv.astype(np.float32))).astype(np.float64)
                lens = models[r].kv_len(j)
                for i in range(len(meta)):
                    s = int(meta[i, 0])
                    assert lens[s] == pos + 1, f"layer {j} seq {s}: length {lens[s]} != {pos + 1}"
                    k_all, v_all = models[r].kv_rows(j, s, 0, pos + 1)
                    # the appended row: oracle projection, identical in every replica
                    assert _rel(_bf(k_all[pos]).ravel(), qkv[i, d:2 * d]) <= REL_TOL
                    assert _rel(_bf(v_all[pos]).ravel(), qkv[i, 2 * d:]) <= REL_TOL
                    for m2 in models:
                        k2, v2 = m2.kv_rows(j, s, pos, 1)
                        assert np.array_equal(k2[0], k_all[pos]) and np.array_equal(v2[0], v_all[pos])
                    # attention over the local replica + output projection + residual
                    q = qkv[i, :d].reshape(1, H, Dh)
                    kk = _bf(k_all).transpose(1, 0, 2)[None]   # [1][H][pos+1][Dh]
                    vv = _bf(v_all).transpose(1, 0, 2)[None]
                    att = oatt.coherent_attention(q, np.array([0]), np.array([pos + 1]), kk, vv, Dh ** -0.5)
                    att = co.orc.bf16_bits_to_f32(co.orc.f32_to_bf16_bits(att.reshape(-1).astype(np.float32)))
                    want = _bf(xb[i]) + att.astype(np.float64) @ wo.T + bo
                    err = _rel(_bf(xm[i]), want)
                    assert err <= REL_TOL, f"layer {j} token {s}: post-attention rel err {err:.3e}"
            # the MoE layer on the post-attention states (routes exact)
            if fused:
                models[0].phase(PHASE_FUSED, j)
            else:
                for m in models:
                    m.phase(PHASE_DISPATCH, j)
                for m in models:
                    m.phase(PHASE_FFN, j)
            torch.cuda.synchronize()
            routes = np.full_like(models[0].routes(), -1)
            for m in models:
                routes = np.where(m.routes() >= 0, m.routes(), routes)
            wg = models[0].gate_weights(j)
            for r in range(G):
                xm, meta_m = mid[r]
                e, _ = co.route(xm, wg, None)
                assert (routes[meta_m[:, 0], j] == e).all(), f"routing mismatch after attention, layer {j}"
        for m in models:
            m.phase(PHASE_GATHER_SEND)
        for m in models:
            m.phase(PHASE_GATHER_WAIT)
        torch.cuda.synchronize()
        for m in models:
            m.check()
        for j in range(L):
            for m in models:
                assert (m.kv_len(j) == P + step + 1).all()


@pytest.fixture(scope="module")
def torch_cuda():
    import torch
    from paper_2401_08383_b200 import _capi
    assert torch.cuda.is_available()
    if _capi.load().exf_device_ok() != 1:
        pytest.fail("no sm_100 GPU visible to libexflow_b200.so")
    return torch


def test_attention_block_one_gpu_fused(torch_cuda):
    from paper_2401_08383_b200 import placement as pl
    from paper_2401_08383_b200.affinity import Topology
    E, L = 8, 2
    assign = pl.contiguous_placement(E, L, Topology(1, 1))
    models = _models(1, assign, num_experts=E, num_layers=L, d_model=512, d_ffn=1024, tokens_per_gpu=32,
                     seed=3, gate_affinity=0.7, attn_heads=8, context_len=256, context_prefix=40)
    assert models[0].describe()["attention"]["heads"] == 8
    run_attention_checked(torch_cuda, models, assign, steps=2, seed=1)
    for m in models:
        m.close()


def test_attention_block_two_ranks_tokens_move(torch_cuda):
    from paper_2401_08383_b200 import placement as pl
    from paper_2401_08383_b200.affinity import Topology
    E, L = 8, 3
    assign = pl.random_placement(E, L, Topology(1, 2), seed=4)
    models = _models(2, assign, num_experts=E, num_layers=L, d_model=1024, d_ffn=2048, tokens_per_gpu=16,
                     seed=5, gate_affinity=0.5, attn_heads=16, context_len=300, context_prefix=100)
    run_attention_checked(torch_cuda, models, assign, steps=2, seed=2)
    for m in models:
        m.close()


def test_attention_step_graph_replays(torch_cuda):
    """The public one-call step (CUDA graph) with the attention block: each
    replay appends one row per sequence and layer, and equals the phased run."""
    import torch
    from paper_2401_08383_b200 import placement as pl
    from paper_2401_08383_b200.affinity import Topology
    E, L = 8, 2
    assign = pl.contiguous_placement(E, L, Topology(1, 1))
    kw = dict(num_experts=E, num_layers=L, d_model=512, d_ffn=1024, tokens_per_gpu=64, seed=9,
              gate_affinity=0.7, attn_heads=8, context_len=128, context_prefix=16)
    (m,) = _models(1, assign, **kw)
    (ref,) = _models(1, assign, **kw)
    x = torch.randn(64, 512, generator=torch.Generator().manual_seed(4)).to(torch.bfloat16).cuda()
    s = torch.cuda.Stream()
    for mm in (m, ref):
        mm.context_setup(s)
    s.synchronize()
    m.capture(x, s)
    for step in range(3):
        m.replay(s)
        ref.step(x, s)
        s.synchronize()
        m.check()
        assert torch.equal(m.output(), ref.output()), f"step {step}"
        assert (m.kv_len(0) == 16 + step + 1).all()
    assert m.launches_per_step() == 1 + (3 + 1) * L + 2  # qkv (+ folded K/V append), attention, o-proj, MoE
    m.close()
    ref.close()
