"""FFN kernel timeline (diagnostics): per-CTA globaltimer stamps of the last
GEMM1/GEMM2 launch of a decode step at the bench config.
Usage: EXF_FFN_TIMELINE=1 python tools/ffn_timeline.py"""
import ctypes as C
import os
import statistics
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
    cfg = MoeModelConfig(num_experts=E, num_layers=4, d_model=1024, d_ffn=4096,
                         tokens_per_gpu=B, seed=1234, gate_affinity=0.8)
    m = MoeModel(cfg, pl.contiguous_placement(E, 4, Topology(1, 1)))
    plan = m.describe()
    print("plan", plan)
    x = torch.randn(B, 1024).to(torch.bfloat16).cuda()
    s = torch.cuda.Stream()
    for _ in range(3):
        m.step(x, s)
    s.synchronize()
    m.check()
    ctas = 4096
    buf = np.zeros((6, ctas, 16), np.uint64)
    _capi.call("exf_model_read_ffn_timeline", m.handle, buf.ctypes.data, ctas)
    for g, key in ((0, "gemm1"), (1, "gemm2")):
        n = plan[key]["clusters"] * plan[key]["ksplit"]
        t = buf[g, :n].astype(np.int64)
        t0 = t[:, 0].min()
        rel = (t - t0) / 1000.0
        span = rel[:, 15].max()
        pro = rel[:, 1] - rel[:, 0]
        print(f"{key}: ctas {n}, span {span:.2f} us, entry skew {rel[:, 0].max():.2f} us, "
              f"prologue mean {pro.mean():.2f} max {pro.max():.2f} us")
        for j in range(3):
            st, en = rel[:, 2 + 2 * j], rel[:, 3 + 2 * j]
            ok = t[:, 2 + 2 * j] > 0
            if not ok.any():
                continue
            d = (en - st)[ok]
            print(f"  job {j}: ctas {ok.sum()}, first-stage at {st[ok].mean():.2f} us (after "
                  f"prologue {(st - rel[:, 1])[ok].mean():.2f}), stream {d.mean():.2f} us "
                  f"(min {d.min():.2f} max {d.max():.2f}), done at {en[ok].mean():.2f}")
        print(f"  epilogue done {rel[:, 14].mean():.2f} us, exit mean {rel[:, 15].mean():.2f} "
              f"max {rel[:, 15].max():.2f}")


if __name__ == "__main__":
    main()
