"""GPU parity of the full decode layer stack against the CPU oracle.

Per layer, teacher-forced on the GPU's own layer inputs (bf16, exact):
  * routing decisions: bit-exact (fixed-order fp32 gate, lowest-index ties)
  * token permutation after the coherent dispatch: exact token order per rank
  * layer outputs: <= 1e-2 relative L2 error per token (bf16 tolerance of
    BASELINE.json north_star), written in the assertion below
Per step: context AllGather output identical on every rank and equal to the
final resident states; crossed-token counters == simulate() coherent moves
(proj/src/sim.cpp:124-125) on the emitted trace; fused histogram ==
count_transitions (proj/src/trace.cpp:191-215) on the emitted trace.
Multi-rank cases run G ranks in one process on one GPU in lock-step phases
(dispatch of every rank, then every rank's FFN), which exercises the same
peer-pointer stores and flags as the multi-GPU path.
"""
import numpy as np
import pytest

import coherent_oracle as co

pytestmark = pytest.mark.gpu

REL_TOL = 1e-2


@pytest.fixture(scope="module")
def torch_cuda():
    import torch
    from paper_2401_08383_b200 import _capi
    assert torch.cuda.is_available()
    if _capi.load().exf_device_ok() != 1:
        pytest.fail("no sm_100 GPU visible to libexflow_b200.so")
    return torch


def _models(G, assign, **kw):
    from paper_2401_08383_b200.model import MoeModel, MoeModelConfig
    models = [MoeModel(MoeModelConfig(world_size=G, rank=r, **kw), assign) for r in range(G)]
    if G > 1:
        MoeModel.connect_local(models)
    return models


def _inputs(torch, models, seed):
    g = torch.Generator().manual_seed(seed)
    cfg = models[0].config
    return [torch.randn(cfg.tokens_per_gpu, cfg.d_model, generator=g).to(torch.bfloat16).cuda()
            for _ in models]


def _bf16_bits(t):
    import torch
    return t.view(torch.int16).cpu().numpy().view(np.uint16)


def _union_routes(models):
    r = np.full_like(models[0].routes(), -1)
    for m in models:
        mine = m.routes()
        r = np.where(mine >= 0, mine, r)
    return r


def run_checked(torch, models, xs, assign, ffn_samples=48, seed=0, forced=None, fused=False, streams=None):
    """Lock-step phased run with per-layer oracle checks; returns final routes.
    fused=True drives the one-launch-per-layer kernel (layer_fused.cu). With
    ep_mode EP_VANILLA every layer is followed by the combine (outputs back to
    the home ranks), checked as an exact copy in home order."""
    from paper_2401_08383_b200.model import (EP_VANILLA, PHASE_BEGIN, PHASE_COMBINE_SEND,
                                             PHASE_COMBINE_WAIT, PHASE_DISPATCH, PHASE_FFN, PHASE_FUSED,
                                             PHASE_GATHER_SEND, PHASE_GATHER_WAIT)
    cfg = models[0].config
    vanilla = cfg.ep_mode == EP_VANILLA
    G, L, E = cfg.world_size, cfg.num_layers, cfg.num_experts
    rng = np.random.default_rng(seed)
    for m in models:
        m.reset_stats()
    for r, m in enumerate(models):
        m.phase(PHASE_BEGIN, 0, xs[r])
    weights = {}
    moves = np.zeros(L, np.int64)
    for j in range(L):
        before = [m.resident(j % 2) for m in models]
        if j == 0:
            for r in range(G):
                assert (before[r][1][:, 0] == cfg.home_tokens(r)).all()
        if fused:
            # one rank per GPU, or co-resident ranks (EXF_FUSED_CTAS) on their
            # own streams: every rank's layer kernel must run concurrently
            assert G == 1 or streams is not None, "the fused layer kernel needs concurrent ranks"
            for r, m in enumerate(models):
                m.phase(PHASE_FUSED, j, stream=None if streams is None else streams[r])
            torch.cuda.synchronize()
        else:
            for m in models:
                m.phase(PHASE_DISPATCH, j)
            for m in models:
                m.phase(PHASE_FFN, j)
        after = [m.resident((j + 1) % 2) for m in models]
        routes = _union_routes(models)
        wg = models[0].gate_weights(j)
        experts, probs = [], []
        for r in range(G):
            xb, meta = before[r]
            toks = meta[:, 0]
            e, p = co.route(xb, wg, None if forced is None else forced[toks, j])
            # (1) routing decisions bit-exact
            assert (routes[toks, j] == e).all(), f"routing mismatch at layer {j} rank {r}"
            experts.append(e)
            probs.append(p)
            moves[j] += int((assign[j][e] != r).sum())
        # (2) permutation: canonical (slot, source, order) token order per rank
        plan = co.dispatch([b[1][:, 0] for b in before], experts, assign[j], G)
        for p_rank in range(G):
            xa, meta_a = after[p_rank]
            want_tok = np.array([before[g][1][i, 0] for g, i in plan[p_rank]], np.int32)
            assert (meta_a[:, 0] == want_tok).all(), f"permutation mismatch layer {j} rank {p_rank}"
            want_exp = np.array([experts[g][i] for g, i in plan[p_rank]], np.int32)
            assert (meta_a[:, 1] == want_exp).all()
            # (3) FFN outputs within tolerance on a sample of tokens
            idx = np.arange(len(plan[p_rank]))
            if len(idx) > ffn_samples:
                idx = rng.choice(idx, ffn_samples, replace=False)
            for k in idx:
                g, i = plan[p_rank][k]
                e = int(experts[g][i])
                if (j, e) not in weights:
                    weights[(j, e)] = models[assign[j][e]].expert_weights(j, e)
                _, ref = co.ffn_ref(before[g][0][i], weights[(j, e)], probs[g][i])
                got = co.orc.bf16_bits_to_f32(xa[k])
                err = np.linalg.norm(got - ref) / np.linalg.norm(ref)
                assert err <= REL_TOL, f"layer {j} token {want_tok[k]} rel err {err}"
                # the FFN update itself (out - x) to 5%, plus the bf16 rounding
                # floor of the stored output (2^-8 relative to |out|)
                xin = co.orc.bf16_bits_to_f32(before[g][0][i])
                budget = 5e-2 * np.linalg.norm(ref - xin) + 2.0 ** -8 * np.linalg.norm(ref)
                assert np.linalg.norm(got - ref) <= budget, \
                    f"layer {j} token {want_tok[k]} FFN-delta error above budget"
        if vanilla:
            # combine: every token's row back to slot t / G of home rank t % G
            for m in models:
                m.phase(PHASE_COMBINE_SEND, j)
            for m in models:
                m.phase(PHASE_COMBINE_WAIT, j)
            row_of = {}
            for p_rank in range(G):
                xa, meta_a = after[p_rank]
                for k in range(len(meta_a)):
                    row_of[int(meta_a[k, 0])] = (xa[k], int(meta_a[k, 1]))
            for r in range(G):
                xh, meta_h = models[r].resident((j + 1) % 2)
                assert (meta_h[:, 0] == cfg.home_tokens(r)).all(), f"combine order layer {j} rank {r}"
                for k, t in enumerate(meta_h[:, 0]):
                    assert np.array_equal(xh[k], row_of[int(t)][0]), f"combine row layer {j} token {t}"
                    assert meta_h[k, 1] == row_of[int(t)][1]
    final = [m.resident(L % 2) for m in models]
    for m in models:
        m.phase(PHASE_GATHER_SEND)
    for m in models:
        m.phase(PHASE_GATHER_WAIT)
    for m in models:
        m.check()
    # context AllGather: every rank sees every token's final state
    outs = [_bf16_bits(m.output()) for m in models]
    for o in outs[1:]:
        assert np.array_equal(o, outs[0])
    for r in range(G):
        xf, meta = final[r]
        assert np.array_equal(outs[0][meta[:, 0]], xf)
    routes = _union_routes(models)
    assert (routes >= 0).all()
    # crossed counters == coherent moves (vanilla: away-from-home events) of
    # the replay on the emitted trace
    crossed = sum(m.crossed() for m in models)
    assert (crossed == moves).all()
    if vanilla:
        rep = co.orc.simulate(routes, assign, 1, G, co.orc.VANILLA)
        assert int(crossed.sum()) == rep.away_from_home_events
    else:
        rep = co.orc.simulate(routes, assign, 1, G, co.orc.COHERENT)
        assert int(crossed.sum()) == rep.coherent_moves
    # fused histogram == count_transitions of the emitted trace (bit-exact)
    hist = sum(m.affinity_counts() for m in models)
    want, _ = co.orc.count_transitions(routes, E)
    assert np.array_equal(hist, want)
    return routes


def test_tiny_config_single_device(torch_cuda, orc):
    # BASELINE configs[0]: 4 MoE layers, 8 experts top-1, d_model 512, 256 tokens, 1 device
    assign = orc.contiguous_placement(8, 4, 1)
    models = _models(1, assign, num_experts=8, num_layers=4, d_model=512, d_ffn=2048,
                     tokens_per_gpu=256, seed=42, gate_affinity=0.5)
    xs = _inputs(torch_cuda, models, 1)
    run_checked(torch_cuda, models, xs, assign)


FUSED_CONFIGS = [(8, 4, 512, 2048, 256), (8, 4, 1024, 4096, 64), (16, 3, 256, 512, 8),
                 (64, 3, 1024, 1024, 96), (32, 2, 2048, 2048, 48),
                 # > 4 jobs per CTA: TMEM accumulator buffers wrap around
                 (8, 2, 1024, 8192, 64), (16, 2, 1024, 4096, 64),
                 # BASELINE configs[3] (1.3B: E=32, d=2048, d_ffn=4d) at the largest
                 # decode batch of its sweep (B=512 > #SMs: dispatch path, 4 tokens
                 # per CTA) and configs[4] (E=64, d=1024, d_ffn=4d)
                 (32, 2, 2048, 8192, 512), (64, 2, 1024, 4096, 64)]


@pytest.mark.parametrize("E,L,d,dff,B", FUSED_CONFIGS)
def test_fused_layer_kernel_single_device(torch_cuda, orc, E, L, d, dff, B):
    # the one-launch-per-layer kernel (dense single-GPU mode where C <= #SMs):
    # gate, routing, GEMM1 -> GEMM2 with in-kernel dependencies; oracle per layer
    assign = orc.contiguous_placement(E, L, 1)
    models = _models(1, assign, num_experts=E, num_layers=L, d_model=d, d_ffn=dff,
                     tokens_per_gpu=B, seed=42 + E, gate_affinity=0.5)
    xs = _inputs(torch_cuda, models, 1)
    run_checked(torch_cuda, models, xs, assign, ffn_samples=24, fused=True)


@pytest.mark.parametrize("E,L,d,dff,B", FUSED_CONFIGS[:2] + FUSED_CONFIGS[5:])
def test_fused_layer_kernel_dispatch_path(torch_cuda, orc, monkeypatch, E, L, d, dff, B):
    # the same kernel with the single-GPU dense mode off: gate, bucketing,
    # dispatch exchange, split-K pieces over the dispatched rows
    monkeypatch.setenv("EXF_DENSE", "0")
    assign = orc.contiguous_placement(E, L, 1)
    models = _models(1, assign, num_experts=E, num_layers=L, d_model=d, d_ffn=dff,
                     tokens_per_gpu=B, seed=7 + E, gate_affinity=0.5)
    assert models[0].describe()["layer_kernel"]["dense"] is False
    xs = _inputs(torch_cuda, models, 2)
    run_checked(torch_cuda, models, xs, assign, ffn_samples=24, fused=True)


def test_fused_layer_kernel_forced_skew(torch_cuda, orc):
    # every token on one expert: empty experts, multi-chunk tiles, split-K slots
    E, L, B = 8, 3, 200
    assign = orc.contiguous_placement(E, L, 1)
    models = _models(1, assign, num_experts=E, num_layers=L, d_model=512, d_ffn=1024,
                     tokens_per_gpu=B, seed=2)
    forced = np.full((B, L), 3, np.int32)
    models[0].set_forced_routes(forced)
    xs = _inputs(torch_cuda, models, 5)
    routes = run_checked(torch_cuda, models, xs, assign, ffn_samples=8, forced=forced, fused=True)
    assert (routes == 3).all()


@pytest.mark.parametrize("G,placement", [(2, "contiguous"), (4, "random"), (8, "contiguous"),
                                         (8, "random")])
def test_multi_rank_lockstep(torch_cuda, orc, G, placement):
    E, L = 8, 3
    assign = (orc.contiguous_placement(E, L, G) if placement == "contiguous"
              else orc.random_placement(E, L, G, 7))
    models = _models(G, assign, num_experts=E, num_layers=L, d_model=256, d_ffn=512,
                     tokens_per_gpu=24, seed=3, gate_affinity=0.8)
    xs = _inputs(torch_cuda, models, G)
    run_checked(torch_cuda, models, xs, assign, ffn_samples=16)


@pytest.mark.parametrize("B", [40, 100])
def test_forced_skew_all_tokens_one_expert(torch_cuda, orc, B):
    # worst-case skew: every token routed to expert 0 (empty experts elsewhere,
    # multi-chunk token tiles, all tokens converge on one GPU)
    G, E, L = 2, 4, 3
    assign = orc.contiguous_placement(E, L, G)
    models = _models(G, assign, num_experts=E, num_layers=L, d_model=256, d_ffn=256,
                     tokens_per_gpu=B, seed=5)
    forced = np.zeros((G * B, L), np.int32)
    for m in models:
        m.set_forced_routes(forced)
    xs = _inputs(torch_cuda, models, 9)
    routes = run_checked(torch_cuda, models, xs, assign, ffn_samples=8, forced=forced)
    assert (routes == 0).all()


def test_forced_markov_routes_replay_parity(torch_cuda, orc):
    # forced-routing mode: routes from generate_markov_trace; the measured
    # crossed fraction must equal simulate()'s p_star on the same trace/homes
    G, E, L, B = 4, 16, 6, 32
    forced = orc.generate_markov_trace(E, L, G * B, 0.8, 4, 11)
    for assign in (orc.contiguous_placement(E, L, G), orc.random_placement(E, L, G, 2)):
        models = _models(G, assign, num_experts=E, num_layers=L, d_model=256, d_ffn=256,
                         tokens_per_gpu=B, seed=1)
        for m in models:
            m.set_forced_routes(forced)
        xs = _inputs(torch_cuda, models, 4)
        routes = run_checked(torch_cuda, models, xs, assign, ffn_samples=4, forced=forced)
        assert np.array_equal(routes, forced)
        crossed = sum(m.crossed() for m in models)
        rep = orc.simulate(forced, assign, 1, G, orc.COHERENT)
        assert crossed.sum() / (G * B * L) == rep.p_star


@pytest.mark.parametrize("E,B,dense", [(8, 128, "1"), (8, 128, "0"), (64, 8, "0")])
def test_full_step_and_graph_replay_match_phased(torch_cuda, orc, monkeypatch, E, B, dense):
    # eager exf_model_step (dispatch path: layer kernels chained on exit
    # generations), graph replays (PDL waits) and the phased run give the same
    # bits; dense single-GPU mode, the dispatch path, and sparse decode with
    # virtual expert slots (E=64, 8 tokens)
    torch = torch_cuda
    monkeypatch.setenv("EXF_DENSE", dense)
    assign = orc.contiguous_placement(E, 4, 1)
    kw = dict(num_experts=E, num_layers=4, d_model=512, d_ffn=1024, tokens_per_gpu=B, seed=8,
              gate_affinity=0.5)
    m = _models(1, assign, **kw)[0]
    x = _inputs(torch, [m], 2)[0]
    m.step(x)
    m.check()
    a = _bf16_bits(m.output()).copy()
    r1 = m.routes().copy()
    stream = torch.cuda.Stream()
    m.capture(x, stream)
    for _ in range(3):
        m.replay(stream)
    stream.synchronize()
    m.check()
    assert np.array_equal(_bf16_bits(m.output()), a)  # deterministic step
    assert np.array_equal(m.routes(), r1)
    # the same step driven layer by layer (fused kernel) gives the same bits
    m2 = _models(1, assign, **kw)[0]
    run_checked(torch, [m2], [x], assign, ffn_samples=8, fused=True)
    assert np.array_equal(_bf16_bits(m2.output()), a)


def test_model_rejects_bad_configs(torch_cuda, orc):
    from paper_2401_08383_b200 import _capi
    assign = orc.contiguous_placement(8, 4, 1)
    with pytest.raises(_capi.ExflowInvalidArgument, match="top-1"):
        _models(1, assign, num_experts=8, num_layers=4, d_model=512, d_ffn=1024,
                tokens_per_gpu=8, top_k=2)
    with pytest.raises(_capi.ExflowInvalidArgument, match="multiple of 256"):
        _models(1, assign, num_experts=8, num_layers=4, d_model=500, d_ffn=1024, tokens_per_gpu=8)
    bad = assign.copy()
    with pytest.raises(_capi.ExflowInvalidArgument):
        _models(2, bad, num_experts=8, num_layers=4, d_model=256, d_ffn=256, tokens_per_gpu=8)


@pytest.mark.parametrize("G", [2, 4])
def test_vanilla_ep_lockstep(torch_cuda, orc, G):
    # vanilla expert parallelism (dispatch + combine back home every layer,
    # proj/src/sim.cpp:60-64): same routes and FFN math, tokens at home after
    # every layer, crossed counters == simulate(VANILLA) away-from-home events
    from paper_2401_08383_b200.model import EP_VANILLA
    E, L = 8, 3
    assign = orc.random_placement(E, L, G, 11)
    models = _models(G, assign, num_experts=E, num_layers=L, d_model=256, d_ffn=512,
                     tokens_per_gpu=24, seed=5, gate_affinity=0.8, ep_mode=EP_VANILLA)
    xs = _inputs(torch_cuda, models, 40 + G)
    run_checked(torch_cuda, models, xs, assign, ffn_samples=16)


def test_vanilla_ep_single_device_fused(torch_cuda, orc):
    from paper_2401_08383_b200.model import EP_VANILLA
    E, L, B = 8, 3, 64
    assign = orc.contiguous_placement(E, L, 1)
    models = _models(1, assign, num_experts=E, num_layers=L, d_model=1024, d_ffn=4096,
                     tokens_per_gpu=B, seed=9, gate_affinity=0.8, ep_mode=EP_VANILLA)
    xs = _inputs(torch_cuda, models, 77)
    run_checked(torch_cuda, models, xs, assign, ffn_samples=8, fused=True)


def test_emitted_trace_round_trip(torch_cuda, orc, tmp_path):
    # a GPU run's routes saved as EXFLOW-TRACE v1 and read back reproduce the
    # run's fused histogram (count_transitions) and crossed counters (simulate)
    from paper_2401_08383_b200 import traceio
    E, L, B = 8, 4, 64
    assign = orc.contiguous_placement(E, L, 1)
    models = _models(1, assign, num_experts=E, num_layers=L, d_model=512, d_ffn=2048,
                     tokens_per_gpu=B, seed=21, gate_affinity=0.8)
    m = models[0]
    xs = _inputs(torch_cuda, models, 5)
    m.reset_stats()
    m.step(xs[0])
    torch_cuda.cuda.synchronize()
    m.check()
    f = tmp_path / "run.trace"
    m.save_trace(f)
    paths, e = traceio.load_trace(f)
    assert e == E and np.array_equal(paths, m.routes())
    want, _ = orc.count_transitions(paths, E)
    assert np.array_equal(m.affinity_counts(), want)
    rep = orc.simulate(paths, assign, 1, 1, orc.COHERENT)
    assert int(m.crossed().sum()) == rep.coherent_moves


def test_expert_migration_local(torch_cuda, orc):
    # online placement change (histogram -> solver -> migration): after
    # migrate_local every rank's slots hold exactly the weights a model built
    # on the new placement has, and a decode step matches it bit for bit
    from paper_2401_08383_b200 import migrate
    from paper_2401_08383_b200.model import (PHASE_BEGIN, PHASE_DISPATCH, PHASE_FFN,
                                             PHASE_GATHER_SEND, PHASE_GATHER_WAIT)
    E, L, G = 8, 3, 2
    p0 = orc.contiguous_placement(E, L, G)
    p1 = orc.random_placement(E, L, G, 5)
    kw = dict(num_experts=E, num_layers=L, d_model=256, d_ffn=512, tokens_per_gpu=16, seed=13,
              gate_affinity=0.7)
    models = _models(G, p0, **kw)
    fresh = _models(G, p1, **kw)
    moved = migrate.migrate_local(models, p1)
    assert moved == sum(int((p0[j] != p1[j]).sum()) for j in range(L))
    for j in range(L):
        for e in range(E):
            g = int(p1[j][e])
            got, want = models[g].expert_weights(j, e), fresh[g].expert_weights(j, e)
            assert all(np.array_equal(a, b) for a, b in zip(got, want)), f"layer {j} expert {e}"
    xs = _inputs(torch_cuda, models, 3)
    outs = []
    for ms in (models, fresh):
        for r, m in enumerate(ms):
            m.phase(PHASE_BEGIN, 0, xs[r])
        for j in range(L):
            for m in ms:
                m.phase(PHASE_DISPATCH, j)
            for m in ms:
                m.phase(PHASE_FFN, j)
        for m in ms:
            m.phase(PHASE_GATHER_SEND)
        for m in ms:
            m.phase(PHASE_GATHER_WAIT)
        for m in ms:
            m.check()
        outs.append((_bf16_bits(ms[0].output()), _union_routes(ms)))
    assert np.array_equal(outs[0][0], outs[1][0]) and np.array_equal(outs[0][1], outs[1][1])


@pytest.mark.parametrize("E,L,d,dff,B,remap", [(64, 2, 1024, 4096, 8, "1"), (16, 3, 256, 512, 8, "1"),
                                               (16, 3, 256, 512, 8, "0"), (64, 2, 512, 1024, 40, "1"),
                                               # BASELINE configs[3] (1.3B: E=32, d=2048) at B=16
                                               (32, 2, 2048, 8192, 16, "1")])
def test_fused_dispatch_virtual_expert_slots(torch_cuda, orc, monkeypatch, E, L, d, dff, B, remap):
    # sparse decode (fewer tokens than 2 per local expert): the schedule's
    # expert ids are virtual slots bound to the experts in descending token
    # count per layer (FusedArgs.remap). Oracle per layer, and the step output
    # bit-identical with the binding off (a tile's split-K parts still reduce
    # in k order, whichever CTAs run them).
    monkeypatch.setenv("EXF_DENSE", "0")
    monkeypatch.setenv("EXF_REMAP", remap)
    assign = orc.contiguous_placement(E, L, 1)
    kw = dict(num_experts=E, num_layers=L, d_model=d, d_ffn=dff, tokens_per_gpu=B, seed=5 + E, gate_affinity=0.6)
    models = _models(1, assign, **kw)
    assert models[0].describe()["layer_kernel"]["virtual_expert_slots"] is (remap == "1")
    xs = _inputs(torch_cuda, models, 3)
    run_checked(torch_cuda, models, xs, assign, ffn_samples=16, fused=True)
    out = _bf16_bits(models[0].output())
    monkeypatch.setenv("EXF_REMAP", "0" if remap == "1" else "1")
    other = _models(1, assign, **kw)
    run_checked(torch_cuda, other, xs, assign, ffn_samples=4, fused=True)
    assert np.array_equal(_bf16_bits(other[0].output()), out)
    for m in models + other:
        m.close()


@pytest.mark.parametrize("E,B,ep", [(8, 16, "coherent"), (8, 64, "coherent"), (64, 8, "coherent"), (16, 16, "vanilla")])
def test_fused_dispatch_path_eight_ranks_one_gpu(torch_cuda, orc, monkeypatch, E, B, ep):
    # the fused dispatch path at G = 8 (BASELINE configs[1] one expert per GPU,
    # configs[4] eight experts per GPU) without eight GPUs: 8 ranks share this
    # device with 18-CTA layer kernels (EXF_FUSED_CTAS), all co-resident, each
    # on its own stream; route flags, receive regions and peers as across GPUs
    from paper_2401_08383_b200.model import EP_VANILLA
    monkeypatch.setenv("EXF_FUSED_CTAS", "18")
    G, L = 8, 3
    assign = orc.random_placement(E, L, G, 11)
    kw = dict(ep_mode=EP_VANILLA) if ep == "vanilla" else {}
    models = _models(G, assign, num_experts=E, num_layers=L, d_model=1024, d_ffn=4096, tokens_per_gpu=B,
                     seed=21 + E, gate_affinity=0.6, **kw)
    d = models[0].describe()
    assert d["path"] == "fused" and d["layer_kernel"]["ctas"] == 18
    streams = [torch_cuda.cuda.Stream() for _ in models]
    xs = _inputs(torch_cuda, models, 4)
    run_checked(torch_cuda, models, xs, assign, ffn_samples=6, fused=True, streams=streams)
    for m in models:
        m.close()
