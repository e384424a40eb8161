"""Decode-step timeline (diagnostics): for each layer and kernel
(gate_dispatch, GEMM1, GEMM2) the first CTA entry, first/last
griddepcontrol.wait return and last CTA exit, relative to the step start,
from a CUDA-graph replay at the bench config.
Usage: python tools/step_timeline.py   (sets EXF_FFN_TIMELINE=1)"""
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
    L = int(os.environ.get("L", "24"))
    cfg = MoeModelConfig(num_experts=E, num_layers=L, d_model=1024, d_ffn=4096, tokens_per_gpu=B,
                         seed=1234, gate_affinity=0.8)
    m = MoeModel(cfg, pl.contiguous_placement(E, L, Topology(1, 1)))
    print("plan", m.describe())
    x = torch.randn(B, 1024).to(torch.bfloat16).cuda()
    s = torch.cuda.Stream()
    m.capture(x, s)
    for _ in range(3):
        m.replay(s)
    s.synchronize()
    buf = np.zeros((L, 3, 8), np.uint64)
    _capi.call("exf_model_read_step_timeline", m.handle, None, 1)
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev0.record(s)
    m.replay(s)
    ev1.record(s)
    s.synchronize()
    m.check()
    _capi.call("exf_model_read_step_timeline", m.handle, buf.ctypes.data, 0)
    t = buf.astype(np.int64)
    t0 = t[0, 0, 0]
    rel = (t - t0) / 1000.0
    print(f"step (events) {ev0.elapsed_time(ev1) * 1000:.1f} us; timeline span {rel[-1, 2, 3]:.1f} us")
    names = ["gate_disp", "gemm1", "gemm2"]
    print("layer kernel   entry  wait0  wait1   exit | run(after wait1)  gap-from-prev-exit")
    prev_exit = None
    for j in range(L):
        for k in range(3):
            e, w0, w1, x_ = rel[j, k, :4]
            gap = (w1 - prev_exit) if prev_exit is not None else 0.0
            if j < 3 or j == L - 1:
                print(f"{j:5d} {names[k]:9s} {e:6.1f} {w0:6.1f} {w1:6.1f} {x_:6.1f} | "
                      f"{x_ - w1:6.1f}  {gap:6.1f}")
            prev_exit = x_
    per = np.diff(rel[:, 0, 0])
    run = rel[:, :, 3] - rel[:, :, 2]
    ph = rel[:, 0, 4:8] - rel[:, 0, 2:3]
    print("gate_disp phases after wait (mean us): staged Wg %.2f, gate %.2f, barrier %.2f, copy %.2f, exit %.2f"
          % (ph[:, 0].mean(), ph[:, 1].mean(), ph[:, 2].mean(), ph[:, 3].mean(),
             (rel[:, 0, 3] - rel[:, 0, 2]).mean()))
    print(f"per-layer period mean {per.mean():.2f} us; kernel run (exit - last wait) mean "
          f"gate_disp {run[:, 0].mean():.2f} gemm1 {run[:, 1].mean():.2f} gemm2 {run[:, 2].mean():.2f}")
    gaps = rel[:, 1:, 2] - rel[:, :-1, 3]
    print(f"wait-release lag after predecessor exit: gemm1 {gaps[:, 0].mean():.2f} gemm2 "
          f"{gaps[:, 1].mean():.2f}; gate_disp {np.mean(rel[1:, 0, 2] - rel[:-1, 2, 3]):.2f}")


if __name__ == "__main__":
    main()
