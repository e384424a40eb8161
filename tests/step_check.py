"""One checked decode step of a running multi-rank model (every rank calls it).

TEST/BENCH CHECKER ONLY: bench.py runs it outside its timed regions, once per
placement, so every bench line carries its own parity verdict; it uses the
CPU oracle only as the checker. Each rank checks its own part of one full
decode step, layer by layer, teacher-forced on the inputs the GPU layer
actually received:

  * routes: the oracle gate (fixed-order fp32 logits, top-1, lowest index on
    ties) of every token equals the route the fused kernel recorded -- exact;
  * permutation: the tokens resident here after the layer are exactly the
    canonical (local slot, source rank, source order) list of the coherent
    dispatch rule (proj/src/sim.cpp:65-71) -- exact, with their experts;
  * outputs: `rows_per_layer` sampled rows of this rank's layer output vs the
    fp64 expert FFN on the same inputs, relative L2 <= 1e-2 (bf16 bar);
  * crossed: the sum over ranks of the per-layer crossed counters equals the
    moves of the oracle routes, and their total equals coherent_moves of
    simulate() on the emitted trace (p_star, proj/src/sim.cpp:151);
  * histogram: the sum over ranks of the fused affinity histogram equals
    count_transitions of the emitted trace (proj/src/trace.cpp:191-215);
  * AllGather: every rank's step output is identical and equals the final
    resident rows.
Returns a JSON-able dict; "parity" is "ok" only if every check passed on
every rank.
"""
from __future__ import annotations

import numpy as np

import coherent_oracle as co

REL_TOL = 1e-2       # bf16 mode (BASELINE north_star)
REL_TOL_F32 = 1e-5   # fp32 mode


def check_step(model, x_dev, assign, rows_per_layer=2, seed=0, group=None):
    import torch
    import torch.distributed as dist
    from paper_2401_08383_b200.model import (PHASE_ATTN, PHASE_BEGIN, PHASE_COMBINE_SEND,
                                             PHASE_COMBINE_WAIT, PHASE_DISPATCH, PHASE_FFN, PHASE_FUSED,
                                             PHASE_GATHER_SEND, PHASE_GATHER_WAIT)
    cfg = model.config
    G, rank, L, E = cfg.world_size, cfg.rank, cfg.num_layers, cfg.num_experts
    dist_on = G > 1

    def allgather(obj):
        if not dist_on:
            return [obj]
        out = [None] * G
        dist.all_gather_object(out, obj, group=group)
        return out

    fused = model.describe().get("path") == "fused"
    vanilla = cfg.ep_mode == 1
    f32 = getattr(cfg, "dtype", 0) == 1
    tol = REL_TOL_F32 if f32 else REL_TOL

    def route(xb, wg):
        if f32:
            return co.orc.gate_top1(co.orc.gate_logits_f32(xb, wg))
        return co.route(xb, wg, None)

    def ffn(x_row, w, p):
        if f32:
            return co.orc.expert_ffn_f32(x_row, *w, p)
        return co.ffn_ref(x_row, w, p)[1]

    def as_f64(row):
        return row.astype(np.float64) if f32 else co.orc.bf16_bits_to_f32(row).astype(np.float64)

    attn = getattr(cfg, "attn_heads", 0) > 0
    attn_worst = 0.0

    def check_attention(j, before_mine, mid_mine):
        """Post-attention rows of sampled resident tokens vs the fp64 oracle on
        the local replica; the appended K/V row identical on every rank."""
        nonlocal attn_worst
        from oracle import attention as oatt
        d, H = cfg.d_model, cfg.attn_heads
        Dh = d // H
        xb, meta = before_mine
        xm, _ = mid_mine
        lens = model.kv_len(j)
        wqkv, bqkv, wo, bo = (co.orc.bf16_bits_to_f32(w).astype(np.float64) for w in model.attn_weights(j))
        pick = rng.choice(len(meta), min(rows_per_layer, len(meta)), replace=False) if len(meta) else []
        rows = []
        for i in pick:
            s_ = int(meta[i, 0])
            pos = int(lens[s_]) - 1
            k_all, v_all = model.kv_rows(j, s_, 0, pos + 1)
            xq = co.orc.bf16_bits_to_f32(xb[i]).astype(np.float64)
            qkv = xq @ wqkv.T + bqkv
            qkv = co.orc.bf16_bits_to_f32(co.orc.f32_to_bf16_bits(qkv.astype(np.float32))).astype(np.float64)
            kf = co.orc.bf16_bits_to_f32(k_all).astype(np.float64)
            vf = co.orc.bf16_bits_to_f32(v_all).astype(np.float64)
            ek = np.linalg.norm(kf[pos].ravel() - qkv[d:2 * d]) / max(np.linalg.norm(qkv[d:2 * d]), 1e-30)
            att = oatt.coherent_attention(qkv[:d].reshape(1, H, Dh), np.array([0]), np.array([pos + 1]),
                                          kf.transpose(1, 0, 2)[None], vf.transpose(1, 0, 2)[None], Dh ** -0.5)
            att = co.orc.bf16_bits_to_f32(co.orc.f32_to_bf16_bits(att.reshape(-1).astype(np.float32)))
            want = xq + att.astype(np.float64) @ wo.T + bo
            got = co.orc.bf16_bits_to_f32(xm[i]).astype(np.float64)
            err = float(np.linalg.norm(got - want) / max(np.linalg.norm(want), 1e-30))
            attn_worst = max(attn_worst, err, float(ek))
            if err > REL_TOL or ek > REL_TOL:
                fails.append(f"layer {j} token {s_}: attention rel err {err:.3e}, appended k rel err {ek:.3e}")
            rows.append((s_, pos, k_all[pos].copy(), v_all[pos].copy()))
        # the appended rows must be identical in every rank's replica
        for r_rows in allgather(rows):
            for s_, pos, kr, vr in r_rows:
                k2, v2 = model.kv_rows(j, s_, pos, 1)
                if not (np.array_equal(k2[0], kr) and np.array_equal(v2[0], vr)):
                    fails.append(f"layer {j} seq {s_}: replicas differ at position {pos}")
    rng = np.random.default_rng(seed + rank)
    fails = []
    worst = 0.0
    moves = np.zeros(L, np.int64)
    model.reset_stats()
    torch.cuda.synchronize()
    if dist_on:
        dist.barrier(group=group)
    model.phase(PHASE_BEGIN, 0, x_dev)
    for j in range(L):
        torch.cuda.synchronize()
        if attn:  # the attention block first, checked on its own
            pre = model.resident(j % 2)
            if dist_on:
                dist.barrier(group=group)
            model.phase(PHASE_ATTN, j)
            torch.cuda.synchronize()
            if dist_on:
                dist.barrier(group=group)  # every rank's appends landed
            check_attention(j, pre, model.resident(j % 2))
        before = allgather(model.resident(j % 2))
        if dist_on:
            dist.barrier(group=group)
        if fused:
            model.phase(PHASE_FUSED, j)
        else:
            model.phase(PHASE_DISPATCH, j)
            torch.cuda.synchronize()
            if dist_on:
                dist.barrier(group=group)
            model.phase(PHASE_FFN, j)
        torch.cuda.synchronize()
        xa, meta_a = model.resident((j + 1) % 2)
        wg = model.gate_weights(j)
        experts, probs = [], []
        for r in range(G):
            xb, meta = before[r]
            e, p = route(xb, wg)
            experts.append(e)
            probs.append(p)
            moves[j] += int((assign[j][e] != r).sum())
        # this rank's recorded routes of the tokens it gated
        mine_tok = before[rank][1][:, 0]
        rec = model.routes()[mine_tok, j]
        if not (rec == experts[rank]).all():
            fails.append(f"layer {j}: routes differ from the oracle gate "
                         f"({int((rec != experts[rank]).sum())} tokens)")
        plan = co.dispatch([b[1][:, 0] for b in before], experts, assign[j], G)[rank]
        want_tok = np.array([before[g][1][i, 0] for g, i in plan], np.int32)
        want_exp = np.array([experts[g][i] for g, i in plan], np.int32)
        if len(want_tok) != len(meta_a) or not (meta_a[:, 0] == want_tok).all() or \
                not (meta_a[:, 1] == want_exp).all():
            fails.append(f"layer {j}: permutation differs from the canonical dispatch order")
        elif len(plan):
            idx = rng.choice(len(plan), min(rows_per_layer, len(plan)), replace=False)
            wcache = {}
            for k in idx:
                g, i = plan[k]
                e = int(experts[g][i])
                if e not in wcache:
                    wcache[e] = model.expert_weights(j, e)
                ref = ffn(before[g][0][i], wcache[e], probs[g][i])
                got = as_f64(xa[k])
                err = float(np.linalg.norm(got - ref) / max(np.linalg.norm(ref), 1e-30))
                worst = max(worst, err)
                if err > tol:
                    fails.append(f"layer {j} token {want_tok[k]}: rel err {err:.3e}")
        if dist_on:
            dist.barrier(group=group)
        if vanilla:
            model.phase(PHASE_COMBINE_SEND, j)
            model.phase(PHASE_COMBINE_WAIT, j)
            torch.cuda.synchronize()
            if dist_on:
                dist.barrier(group=group)
    final = model.resident(L % 2)
    model.phase(PHASE_GATHER_SEND)
    model.phase(PHASE_GATHER_WAIT)
    torch.cuda.synchronize()
    model.check()
    out = model.output().cpu().numpy() if f32 else \
        model.output().view(torch.int16).cpu().numpy().view(np.uint16)
    outs = allgather(out)
    finals = allgather(final)
    crossed = sum(allgather(model.crossed()))
    hist = sum(allgather(model.affinity_counts()))
    routes = np.max(np.stack(allgather(model.routes())), axis=0)
    for o in outs[1:]:
        if not np.array_equal(o, outs[0]):
            fails.append("AllGather outputs differ across ranks")
            break
    for xf, meta in finals:
        if not np.array_equal(outs[0][meta[:, 0]], xf):
            fails.append("AllGather output differs from the final resident rows")
            break
    if (routes < 0).any():
        fails.append("some token-layer has no recorded route")
    if vanilla:
        rep = co.orc.simulate(routes, assign, 1, G, co.orc.VANILLA)
        want_cross = rep.away_from_home_events
    else:
        rep = co.orc.simulate(routes, assign, 1, G, co.orc.COHERENT)
        want_cross = rep.coherent_moves
        if not (crossed == moves).all():
            fails.append(f"per-layer crossed counters {crossed.tolist()} != oracle moves {moves.tolist()}")
    if int(crossed.sum()) != want_cross:
        fails.append(f"crossed {int(crossed.sum())} != simulate {want_cross}")
    want_hist, _ = co.orc.count_transitions(routes, E)
    if not np.array_equal(hist, want_hist):
        fails.append("fused affinity histogram != count_transitions of the emitted trace")
    all_fails = allgather(fails)
    worst_all = max(allgather(worst))
    flat = [f"rank {r}: {f}" for r, fs in enumerate(all_fails) for f in fs]
    return {"parity": "ok" if not flat else "FAIL", "dtype": "f32" if f32 else "bf16",
            "checked": "one full decode step, every layer, every rank: routes + permutation exact, "
                       f"{rows_per_layer} sampled output rows/layer/rank <= {tol} rel L2 vs fp64, "
                       "crossed == simulate, histogram == count_transitions, AllGather equal",
            "routed_fraction_checked_step": float(crossed.sum()) / (cfg.capacity * L),
            "simulate_p_star": rep.p_star if not vanilla else None,
            "max_rel_err_sampled": worst_all,
            "attention_max_rel_err_sampled": max(allgather(attn_worst)) if attn else None,
            "failures": flat[:8]}
