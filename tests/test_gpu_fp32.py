"""fp32 mode of the decode layer stack (BASELINE.json north_star: layer outputs
within 1e-5 relative error in fp32 mode) against the CPU oracle.

Per layer, teacher-forced on the GPU's own fp32 layer inputs:
  * routing: bit-exact -- the oracle runs the same fixed-order fmaf gate on the
    same fp32 inputs (oracle/exflow_model_oracle.c orc_gate_logits_f32);
  * permutation: exact canonical (slot, source, order) token order per rank;
  * outputs: every checked token within REL_TOL_F32 = 1e-5 relative L2 of the
    fp64 evaluation of the same fp32 expert (orc_expert_ffn_f32).
Per step: AllGather output identical across ranks and equal to the final
resident rows; crossed counters == simulate() coherent moves; fused histogram
== count_transitions of the emitted trace.
Shapes: BASELINE configs[0] (E=8, L=4, d=512, 256 tokens, one device) and
configs[1]'s layer shape (E=8, d=1024, d_ffn=4096, 64 tokens per rank) on 1
and 2 lock-step ranks.
"""
import numpy as np
import pytest

import coherent_oracle as co

pytestmark = pytest.mark.gpu

REL_TOL_F32 = 1e-5


def _models(G, assign, **kw):
    from paper_2401_08383_b200.model import DTYPE_F32, MoeModel, MoeModelConfig
    models = [MoeModel(MoeModelConfig(world_size=G, rank=r, dtype=DTYPE_F32, **kw), assign)
              for r in range(G)]
    if G > 1:
        MoeModel.connect_local(models)
    return models


def _route_f32(x, wg):
    logits = co.orc.gate_logits_f32(x, wg)
    return co.orc.gate_top1(logits)


def run_checked_f32(torch, models, assign, samples, seed):
    from paper_2401_08383_b200.model import (PHASE_BEGIN, PHASE_DISPATCH, PHASE_FFN,
                                             PHASE_GATHER_SEND, PHASE_GATHER_WAIT)
    cfg = models[0].config
    G, L, E = cfg.world_size, cfg.num_layers, cfg.num_experts
    g = torch.Generator().manual_seed(seed)
    xs = [torch.randn(cfg.tokens_per_gpu, cfg.d_model, generator=g).float().cuda() for _ in models]
    rng = np.random.default_rng(seed)
    for m in models:
        m.reset_stats()
        assert m.describe()["dtype"] == "f32"
    for r, m in enumerate(models):
        m.phase(PHASE_BEGIN, 0, xs[r])
    moves = np.zeros(L, np.int64)
    worst = 0.0
    for j in range(L):
        before = [m.resident(j % 2) for m in models]
        if j == 0:
            for r in range(G):
                assert np.array_equal(before[r][0], xs[r].cpu().numpy()), "step begin copy"
        for m in models:
            m.phase(PHASE_DISPATCH, j)
        for m in models:
            m.phase(PHASE_FFN, j)
        torch.cuda.synchronize()
        after = [m.resident((j + 1) % 2) for m in models]
        routes = np.full_like(models[0].routes(), -1)
        for m in models:
            mine = m.routes()
            routes = np.where(mine >= 0, mine, routes)
        wg = models[0].gate_weights(j)
        assert wg.dtype == np.float32
        experts, probs = [], []
        for r in range(G):
            xb, meta = before[r]
            e, p = _route_f32(xb, wg)
            assert (routes[meta[:, 0], j] == e).all(), f"fp32 routing mismatch layer {j} rank {r}"
            experts.append(e)
            probs.append(p)
            moves[j] += int((assign[j][e] != r).sum())
        plan = co.dispatch([b[1][:, 0] for b in before], experts, assign[j], G)
        weights = {}
        for pr in range(G):
            xa, meta_a = after[pr]
            want = np.array([before[gg][1][i, 0] for gg, i in plan[pr]], np.int32)
            assert (meta_a[:, 0] == want).all(), f"permutation mismatch layer {j} rank {pr}"
            idx = np.arange(len(plan[pr]))
            if len(idx) > samples:
                idx = rng.choice(idx, samples, replace=False)
            for k in idx:
                gg, i = plan[pr][k]
                e = int(experts[gg][i])
                if e not in weights:
                    weights[e] = models[assign[j][e]].expert_weights(j, e)
                ref = co.orc.expert_ffn_f32(before[gg][0][i], *weights[e], probs[gg][i])
                err = float(np.linalg.norm(xa[k].astype(np.float64) - ref) / np.linalg.norm(ref))
                worst = max(worst, err)
                assert err <= REL_TOL_F32, f"layer {j} token {want[k]}: fp32 rel err {err:.3e}"
    finals = [m.resident(L % 2) for m in models]
    for m in models:
        m.phase(PHASE_GATHER_SEND)
    for m in models:
        m.phase(PHASE_GATHER_WAIT)
    torch.cuda.synchronize()
    for m in models:
        m.check()
    outs = [m.output().cpu().numpy() for m in models]
    for o in outs[1:]:
        assert np.array_equal(o, outs[0])
    for xf, meta in finals:
        assert np.array_equal(outs[0][meta[:, 0]], xf)
    routes = np.full_like(models[0].routes(), -1)
    for m in models:
        routes = np.where(m.routes() >= 0, m.routes(), routes)
    crossed = sum(m.crossed() for m in models)
    assert (crossed == moves).all()
    rep = co.orc.simulate(routes, assign, 1, G, co.orc.COHERENT)
    assert int(crossed.sum()) == rep.coherent_moves
    want_hist, _ = co.orc.count_transitions(routes, E)
    assert np.array_equal(sum(m.affinity_counts() for m in models), want_hist)
    return worst


@pytest.fixture(scope="module")
def torch_cuda():
    import torch
    from paper_2401_08383_b200 import _capi
    assert torch.cuda.is_available()
    if _capi.load().exf_device_ok() != 1:
        pytest.fail("no sm_100 GPU visible to libexflow_b200.so")
    return torch


def test_fp32_configs0_tiny(torch_cuda):
    """BASELINE configs[0]: 4 MoE layers, 8 experts, d_model 512, 256 tokens."""
    from paper_2401_08383_b200 import placement as pl
    from paper_2401_08383_b200.affinity import Topology
    E, L = 8, 4
    assign = pl.contiguous_placement(E, L, Topology(1, 1))
    models = _models(1, assign, num_experts=E, num_layers=L, d_model=512, d_ffn=2048,
                     tokens_per_gpu=256, seed=42, gate_affinity=0.8)
    worst = run_checked_f32(torch_cuda, models, assign, samples=24, seed=1)
    assert worst < REL_TOL_F32
    for m in models:
        m.close()


@pytest.mark.parametrize("G", [1, 2])
def test_fp32_configs1_layer_shape(torch_cuda, G):
    """configs[1] layer shape (d 1024, d_ffn 4096, 8 experts, 64 tokens per rank),
    G lock-step ranks with a random placement (tokens cross GPUs)."""
    from paper_2401_08383_b200 import placement as pl
    from paper_2401_08383_b200.affinity import Topology
    E, L = 8, 3
    assign = pl.random_placement(E, L, Topology(1, G), seed=5)
    models = _models(G, assign, num_experts=E, num_layers=L, d_model=1024, d_ffn=4096,
                     tokens_per_gpu=64, seed=7, gate_affinity=0.5)
    run_checked_f32(torch_cuda, models, assign, samples=12, seed=2)
    for m in models:
        m.close()


def test_fp32_step_graph_matches_phases(torch_cuda):
    """exf_model_step (the public one-call step, CUDA-graph captured) gives
    the same fp32 outputs as the phased run, bit for bit."""
    import torch
    from paper_2401_08383_b200 import placement as pl
    from paper_2401_08383_b200.affinity import Topology
    from paper_2401_08383_b200.model import (PHASE_BEGIN, PHASE_DISPATCH, PHASE_FFN,
                                             PHASE_GATHER_SEND, PHASE_GATHER_WAIT)
    E, L = 8, 4
    assign = pl.contiguous_placement(E, L, Topology(1, 1))
    (m,) = _models(1, assign, num_experts=E, num_layers=L, d_model=512, d_ffn=2048,
                   tokens_per_gpu=128, seed=3, gate_affinity=0.8)
    x = torch.randn(128, 512, generator=torch.Generator().manual_seed(9)).cuda()
    m.phase(PHASE_BEGIN, 0, x)
    for j in range(L):
        m.phase(PHASE_DISPATCH, j)
        m.phase(PHASE_FFN, j)
    m.phase(PHASE_GATHER_SEND)
    m.phase(PHASE_GATHER_WAIT)
    torch.cuda.synchronize()
    ref = m.output().clone()
    s = torch.cuda.Stream()
    m.capture(x, s)
    m.replay(s)
    s.synchronize()
    m.check()
    assert torch.equal(m.output(), ref)
    assert m.launches_per_step() == 1 + 3 * L + 2
    m.close()
