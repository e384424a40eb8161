"""Per-CTA timeline of the fused layer kernel (diagnostics): GEMM-phase start,
per-job MMA start/end (first/last k-block issued) and exit, for the last
layer of a decode step at the bench config. Usage: python tools/fused_timeline.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ.setdefault("EXF_FFN_TIMELINE", "1")


def main():
    import numpy as np
    import torch
    from paper_2401_08383_b200 import _capi, placement as pl
    from paper_2401_08383_b200.affinity import Topology
    from paper_2401_08383_b200.model import MoeModel, MoeModelConfig
    E = int(os.environ.get("E", "8"))
    B = int(os.environ.get("B", "64"))
    G = int(os.environ.get("WORLD_SIZE", "1"))  # under torchrun: one process per GPU
    rank = int(os.environ.get("RANK", "0"))
    if G > 1:
        import torch.distributed as dist
        from paper_2401_08383_b200 import dist as xd
        torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", rank)))
        dist.init_process_group("gloo")
    cfg = MoeModelConfig(num_experts=E, num_layers=4, d_model=1024, d_ffn=4096, tokens_per_gpu=B,
                         seed=1234, gate_affinity=0.8, world_size=G, rank=rank)
    m = MoeModel(cfg, pl.contiguous_placement(E, 4, Topology(1, G)))
    if G > 1:
        m.connect(xd.exchange_handles(m.ipc_handle()))
    x = torch.randn(B, 1024).to(torch.bfloat16).cuda()
    s = torch.cuda.Stream()
    for _ in range(3):
        m.step(x, s)
    s.synchronize()
    m.check()
    if G > 1:
        dist.barrier()
        if rank != 0:
            return
    ctas = 148
    buf = np.zeros((6, ctas, 16), np.uint64)
    _capi.call("exf_model_read_ffn_timeline", m.handle, buf.ctypes.data, ctas)
    t = buf[0].astype(np.int64)
    t0 = t[:, 0].min()
    rel = (t - t0) / 1000.0
    print(f"span {rel[:, 15].max():.2f} us; GEMM phase start mean {rel[:, 1].mean():.2f} "
          f"(min {rel[:, 1].min():.2f} max {rel[:, 1].max():.2f})")
    prev_end = rel[:, 1]
    for j in range(6):
        st, en = rel[:, 2 + 2 * j], rel[:, 3 + 2 * j]
        ok = t[:, 2 + 2 * j] > 0
        if not ok.any():
            break
        print(f"job {j}: ctas {ok.sum():3d}  start {st[ok].mean():6.2f} (wait after prev "
              f"{(st - prev_end)[ok].mean():5.2f})  mma span {(en - st)[ok].mean():5.2f} "
              f"[{(en - st)[ok].min():5.2f},{(en - st)[ok].max():5.2f}]  end {en[ok].mean():6.2f} "
              f"max {en[ok].max():6.2f}")
        prev_end = np.where(ok, en, prev_end)
    print(f"exit mean {rel[:, 15].mean():.2f} max {rel[:, 15].max():.2f}")
    t2 = buf[1].astype(np.int64)
    r2 = (t2 - t0) / 1000.0
    j0 = rel[:, 2]
    print("GEMM1 epilogue store-loop cycles, job 0 (median over CTAs):", int(np.median(t2[:, 0])),
          "; first token-row stage: issue -> landed %.2f us (issued %.2f us after layer entry stamp)" % (
              np.median((t2[:, 2] - t2[:, 1]) / 1e3), np.median((t2[:, 1] - t[:, 0]) / 1e3)))
    b_start = buf[3][:, 8].astype(np.int64)
    mma_full_b = buf[3][:, 9].astype(np.int64)
    print("  rel. token-row producer start: rows ready %.2f, first stage issued %.2f, landed %.2f, MMA role entry "
          "%.2f, MMA saw it %.2f us" % tuple(np.median((v - b_start) / 1e3)
                                            for v in (t2[:, 9], t2[:, 1], t2[:, 2], t2[:, 3], mma_full_b)))
    if G == 1:  # dense: epilogue per job (accumulator ready -> done), by kind
        t4 = buf[4]
        for j in range(5):
            st = t4[:, 2 * j].astype(np.int64)
            en_raw = t4[:, 2 * j + 1]
            ok = (st > 0) & (en_raw > 0)
            if not ok.any():
                break
            kind = (en_raw >> np.uint64(62)).astype(np.int64)
            en = (en_raw & np.uint64((1 << 62) - 1)).astype(np.int64)
            mma_end = t[:, 3 + 2 * j]
            for kd, nm in ((0, "direct"), (2, "finisher"), (1, "park")):
                sel = ok & (kind == kd)
                if sel.any():
                    print(f"  epilogue job {j} {nm:8s} ctas {sel.sum():3d}: acc ready {np.median((st - mma_end)[sel]) / 1e3:5.2f} "
                          f"after last MMA, duration median {np.median((en - st)[sel]) / 1e3:5.2f} max "
                          f"{((en - st)[sel]).max() / 1e3:5.2f} us")
    if G > 1:  # dispatch path: epilogue per job: acc ready, park done, counter done, done
        t4 = buf[4]
        for j in range(4):
            st = t4[:, 2 * j].astype(np.int64)
            en_raw = t4[:, 2 * j + 1]
            ok = (st > 0) & (en_raw > 0)
            if not ok.any():
                break
            kind = (en_raw >> np.uint64(62)).astype(np.int64)
            en = (en_raw & np.uint64((1 << 62) - 1)).astype(np.int64)
            pk = t4[:, 8 + 2 * j].astype(np.int64)
            ct = t4[:, 9 + 2 * j].astype(np.int64)
            for kd, nm in ((0, "direct"), (2, "finisher"), (1, "park")):
                sel = ok & (kind == kd)
                if sel.any():
                    hasp = sel & (pk > 0)
                    print(f"  epilogue job {j} {nm:8s} ctas {sel.sum():3d}: acc ready {np.median((st - t[:, 3 + 2 * j])[sel]) / 1e3:5.2f} "
                          f"after last MMA, duration median {np.median((en - st)[sel]) / 1e3:5.2f} max "
                          f"{((en - st)[sel]).max() / 1e3:5.2f} us" +
                          (f"; park {np.median((pk - st)[hasp]) / 1e3:5.2f} counter {np.median((ct - pk)[hasp]) / 1e3:5.2f}"
                           if hasp.any() else "") + f"; done rel first entry max {((en[sel] - t0) / 1e3).max():.2f}")
                    if kd == 2 and j == 0:
                        f12, f13, f14 = (t4[:, k].astype(np.int64) for k in (12, 13, 14))
                        f15 = t4[:, 15].astype(np.int64)
                        print(f"    finisher: partial sums of the first 16 columns ready {np.median((f15 - f12)[sel]) / 1e3:5.2f} us after loop start")
                        print(f"    finisher: counter -> loop start {np.median((f12 - ct)[sel]) / 1e3:5.2f}, first 16 cols "
                              f"{np.median((f13 - f12)[sel]) / 1e3:5.2f}, loop end {np.median((f14 - f12)[sel]) / 1e3:5.2f}, "
                              f"-> done {np.median((en - f14)[sel]) / 1e3:5.2f} us; ncols? n/a")
    t5 = buf[5].astype(np.int64)
    print("  token-row stage issue (emptyB passed) rel. job 0 first MMA, median us, it 0..15:",
          [round(float(np.median((t5[:, i] - t[:, 2]) / 1e3)), 2) for i in range(16)])
    print("  job 0 last MMA rel. its first: median %.2f" % np.median((t[:, 3] - t[:, 2]) / 1e3))
    its = np.maximum(t2[:, 7], 1)
    print(f"weight stage hold (MMA issue -> stage freed): median {np.median(t2[:, 4]):.0f} ns; "
          f"MMA warp blocked per stage on token rows {np.median(t2[:, 5] / its):.0f} ns, "
          f"on weights {np.median(t2[:, 6] / its):.0f} ns (stages/CTA {int(np.median(t2[:, 7]))})")
    print(f"job 1 MMA: fullB ready {(r2[:, 8] - rel[:, 3]).mean():.2f}, A ready {(r2[:, 9] - rel[:, 3]).mean():.2f} "
          f"after job 0 last MMA")
    print(f"job 0 epilogue: tmem_full at {(r2[:, 10] - rel[:, 3]).mean():.2f} after last MMA, "
          f"done {(r2[:, 11] - r2[:, 10]).mean():.2f} later")
    for k, nm in ((12, "epilogue"), (13, "B producer"), (14, "A producer"), (15, "MMA")):
        print(f"{nm} done mean {r2[:, k].mean():.2f} max {r2[:, k].max():.2f} (argmax cta {r2[:, k].argmax()})")
    w = rel[:, 15].argmax()
    print(f"slowest cta {w}: jobs", [(round(rel[w, 2 + 2 * j], 2), round(rel[w, 3 + 2 * j], 2)) for j in range(5)
                                    if t[w, 2 + 2 * j] > 0])
    # token phase of the last layer (L=4 -> odd row 3) against the previous
    # layer's exits (even row 2)
    cur = buf[3].astype(np.int64)
    prv = buf[2].astype(np.int64)
    z = prv[:, 15].max()
    names = ["entry", "pdl wait", "gate", "scan", "flags", "dispatch", "completion", "tables"]
    print(f"token phase rel. previous layer's last exit (prev exit min {(prv[:, 15].min() - z) / 1e3:.2f}):")
    def rel_us(col):  # stamps never written (this mode's path skips them) -> nan
        return np.where(col > 0, (col - z) / 1e3, np.nan)

    for k, nm in enumerate(names):
        v = rel_us(cur[:, k])
        if np.isnan(v).all():
            print(f"  {nm:10s} (not stamped on this path)")
            continue
        print(f"  {nm:10s} min {np.nanmin(v):7.2f} mean {np.nanmean(v):7.2f} max {np.nanmax(v):7.2f}")
    print(f"  first MMA  min {(t[:, 2] - z).min() / 1e3:7.2f} mean {(t[:, 2] - z).mean() / 1e3:7.2f}")
    print("  dense token warp (rel. prev exit; median/max): gate %s ranks %s barrier %s published %s flag %s" % tuple(
        "%.2f/%.2f" % (np.median((cur[:, k] - z) / 1e3), ((cur[:, k] - z) / 1e3).max()) for k in (12, 13, 14, 7, 2)))
    r10 = buf[1][:, 10].astype(np.int64)
    print("  dense GEMM1 epilogue of job 0 (us after tmem_full): tmem-ld %.2f route-wait %.2f stores %.2f bar %.2f "
          "red %.2f" % tuple(np.median((cur[:, k] - r10) / 1e3) for k in (3, 14, 4, 5, 6)))
    print("  tmem_full of job 0 rel. prev exit: median %.2f; route tables ready median %.2f" % (
        np.median((r10 - z) / 1e3), np.median((cur[:, 2] - z) / 1e3)))
    print("  gate detail (n loaded / Wg ready / dot products done / rows staged):")
    for c in range(4):
        print(f"   cta {c}: " + " ".join(f"{(cur[c, k] - z) / 1e3:6.2f}" for k in (11, 12, 13, 14)))
    print("  per CTA (0..9, 147):", " / ".join(names))
    for c in list(range(10)) + [ctas - 1]:
        print(f"   cta {c:3d}: " + " ".join(f"{(cur[c, k] - z) / 1e3:6.2f}" for k in range(8)) +
              f" | B start {(cur[c, 8] - z) / 1e3:6.2f} fullB {(cur[c, 9] - z) / 1e3:6.2f} "
              f"fullA {(cur[c, 10] - z) / 1e3:6.2f} mma {(t[c, 2] - z) / 1e3:6.2f}")
    print(f"  exit       min {(cur[:, 15] - z).min() / 1e3:7.2f} max {(cur[:, 15] - z).max() / 1e3:7.2f}")
    ok = t[:, 12] > 0
    print(f"job 1 first A TMA issued {(rel[:, 12] - rel[:, 3])[ok].mean():.2f} us after job 0's last MMA; "
          f"first B gather {(rel[:, 13] - rel[:, 3])[ok].mean():.2f}; job 1 first MMA "
          f"{(rel[:, 4] - rel[:, 3])[ok].mean():.2f}")


if __name__ == "__main__":
    main()
