"""Real multi-GPU parity worker (one process per GPU, launched by torchrun from
tests/test_multi_gpu.py): every rank runs the decode layers through the fused
one-launch-per-layer kernel (or the two-kernel path with --phased), the ranks'
kernels exchanging tokens over NVLink P2P; after each layer rank 0 gathers
every rank's resident tokens and checks them against the CPU oracle exactly as
tests/test_gpu_model.py::run_checked does for single-device virtual ranks:
bit-exact routes, exact canonical (slot, source, order) permutation, FFN
outputs within the bf16 tolerance, AllGather equality, crossed counters ==
coherent moves of simulate(), fused histogram == count_transitions."""
import argparse
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import coherent_oracle as co  # noqa: E402

REL_TOL = 1e-2


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--experts", type=int, default=8)
    p.add_argument("--layers", type=int, default=3)
    p.add_argument("--d-model", type=int, default=256)
    p.add_argument("--d-ffn", type=int, default=512)
    p.add_argument("--batch", type=int, default=16)
    p.add_argument("--phased", action="store_true")
    p.add_argument("--vanilla", action="store_true", help="vanilla EP: combine back home every layer")
    p.add_argument("--migrate", action="store_true",
                   help="start from the contiguous placement and migrate the experts (NCCL) to the "
                        "random one before the checked steps")
    p.add_argument("--steps", type=int, default=2)
    a = p.parse_args()

    import torch
    import torch.distributed as dist
    from paper_2401_08383_b200 import dist as xd, placement as pl
    from paper_2401_08383_b200.affinity import Topology
    from paper_2401_08383_b200.model import (EP_COHERENT, EP_VANILLA, PHASE_BEGIN, PHASE_COMBINE_SEND,
                                             PHASE_COMBINE_WAIT, PHASE_DISPATCH, PHASE_FFN, PHASE_FUSED,
                                             PHASE_GATHER_SEND, PHASE_GATHER_WAIT, MoeModel,
                                             MoeModelConfig)
    rank = int(os.environ["RANK"])
    G = int(os.environ["WORLD_SIZE"])
    torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", rank)))
    dist.init_process_group("gloo")
    E, L = a.experts, a.layers
    assign = pl.random_placement(E, L, Topology(1, G), seed=7)
    cfg = MoeModelConfig(num_experts=E, num_layers=L, d_model=a.d_model, d_ffn=a.d_ffn,
                         tokens_per_gpu=a.batch, world_size=G, rank=rank, seed=99, gate_affinity=0.6,
                         ep_mode=EP_VANILLA if a.vanilla else EP_COHERENT)
    if a.migrate:
        from paper_2401_08383_b200 import migrate
        m = MoeModel(cfg, pl.contiguous_placement(E, L, Topology(1, G)))
        m.connect(xd.exchange_handles(m.ipc_handle()))
        nccl = dist.new_group(backend="nccl")
        moved = migrate.migrate_nccl(m, assign, group=nccl)
        # the migrated slots hold exactly what a model built on the new
        # placement generates for them
        ref = MoeModel(cfg, assign)
        for j in range(L):
            for e in range(E):
                if assign[j][e] == rank:
                    got, want = m.expert_weights(j, e), ref.expert_weights(j, e)
                    assert all(np.array_equal(x, y) for x, y in zip(got, want)), f"layer {j} expert {e}"
        ref.close()
        if rank == 0:
            print(f"[mgpu] migrated {moved} experts over NCCL", flush=True)
    else:
        m = MoeModel(cfg, assign)
        m.connect(xd.exchange_handles(m.ipc_handle()))
    fused = m.describe().get("path") == "fused" and not a.phased
    g = torch.Generator().manual_seed(1000 + rank)
    rng = np.random.default_rng(0)

    def gather(obj):
        out = [None] * G if rank == 0 else None
        dist.gather_object(obj, out, dst=0)
        return out

    for step in range(a.steps):
        x = torch.randn(a.batch, a.d_model, generator=g).to(torch.bfloat16).cuda()
        m.reset_stats()
        m.phase(PHASE_BEGIN, 0, x)
        moves = np.zeros(L, np.int64)
        for j in range(L):
            torch.cuda.synchronize()
            before = gather(m.resident(j % 2))
            dist.barrier()
            if fused:
                m.phase(PHASE_FUSED, j)
            else:
                m.phase(PHASE_DISPATCH, j)
                torch.cuda.synchronize()
                dist.barrier()
                m.phase(PHASE_FFN, j)
            torch.cuda.synchronize()
            after = gather(m.resident((j + 1) % 2))
            routes = xd.merge_routes(m.routes())
            # expert weights of this layer, from their owners
            mine = {e: m.expert_weights(j, e) for e in range(E) if assign[j][e] == rank}
            allw = gather(mine)
            if rank == 0:
                weights = {}
                for d in allw:
                    weights.update(d)
                wg = m.gate_weights(j)
                experts, probs = [], []
                for r in range(G):
                    xb, meta = before[r]
                    toks = meta[:, 0]
                    e, pr = co.route(xb, wg, None)
                    assert (routes[toks, j] == e).all(), f"step {step} layer {j} rank {r}: routing mismatch"
                    experts.append(e)
                    probs.append(pr)
                    moves[j] += int((assign[j][e] != r).sum())
                plan = co.dispatch([b[1][:, 0] for b in before], experts, assign[j], G)
                for pr_ in range(G):
                    xa, meta_a = after[pr_]
                    want_tok = np.array([before[gg][1][i, 0] for gg, i in plan[pr_]], np.int32)
                    assert (meta_a[:, 0] == want_tok).all(), f"layer {j} rank {pr_}: permutation mismatch"
                    want_exp = np.array([experts[gg][i] for gg, i in plan[pr_]], np.int32)
                    assert (meta_a[:, 1] == want_exp).all()
                    idx = np.arange(len(plan[pr_]))
                    if len(idx) > 24:
                        idx = rng.choice(idx, 24, replace=False)
                    for k in idx:
                        gg, i = plan[pr_][k]
                        e = int(experts[gg][i])
                        _, ref = co.ffn_ref(before[gg][0][i], weights[e], probs[gg][i])
                        got = co.orc.bf16_bits_to_f32(xa[k])
                        err = np.linalg.norm(got - ref) / np.linalg.norm(ref)
                        assert err <= REL_TOL, f"layer {j} token {want_tok[k]} rel err {err}"
            dist.barrier()
            if a.vanilla:  # outputs back to the home ranks, exact copies in home order
                m.phase(PHASE_COMBINE_SEND, j)
                m.phase(PHASE_COMBINE_WAIT, j)
                torch.cuda.synchronize()
                home = gather(m.resident((j + 1) % 2))
                if rank == 0:
                    row_of = {}
                    for xa, meta_a in after:
                        for k in range(len(meta_a)):
                            row_of[int(meta_a[k, 0])] = (xa[k], int(meta_a[k, 1]))
                    for r in range(G):
                        xh, meta_h = home[r]
                        assert (meta_h[:, 0] == cfg.home_tokens(r)).all(), f"layer {j} rank {r}: combine order"
                        for k, t in enumerate(meta_h[:, 0]):
                            assert np.array_equal(xh[k], row_of[int(t)][0]), f"layer {j} token {t}: combine row"
                            assert meta_h[k, 1] == row_of[int(t)][1]
                dist.barrier()
        final = m.resident(L % 2)
        m.phase(PHASE_GATHER_SEND)
        m.phase(PHASE_GATHER_WAIT)
        torch.cuda.synchronize()
        m.check()
        out = m.output().view(torch.int16).cpu().numpy().view(np.uint16)
        outs = gather(out)
        finals = gather(final)
        crossed = gather(m.crossed())
        hists = gather(m.affinity_counts())
        routes = xd.merge_routes(m.routes())
        if rank == 0:
            for o in outs[1:]:
                assert np.array_equal(o, outs[0]), "AllGather outputs differ across ranks"
            for xf, meta in finals:
                assert np.array_equal(outs[0][meta[:, 0]], xf)
            assert (routes >= 0).all()
            c = sum(crossed)
            assert (c == moves).all(), f"crossed {c} != moves {moves}"
            if a.vanilla:
                rep = co.orc.simulate(routes, assign, 1, G, co.orc.VANILLA)
                assert int(c.sum()) == rep.away_from_home_events
            else:
                rep = co.orc.simulate(routes, assign, 1, G, co.orc.COHERENT)
                assert int(c.sum()) == rep.coherent_moves
            want, _ = co.orc.count_transitions(routes, E)
            assert np.array_equal(sum(hists), want)
            print(f"[mgpu] step {step}: G={G} {'fused' if fused else 'two-kernel'} path "
                  f"{'vanilla' if a.vanilla else 'coherent'} OK "
                  f"(crossed {int(c.sum())} of {a.batch * G * L} token-layers)", flush=True)
        dist.barrier()
    m.close()
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
