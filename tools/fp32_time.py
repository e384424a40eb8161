"""fp32-mode step time at BASELINE configs[1] (diagnostics)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

if __name__ == "__main__":
    import torch
    from paper_2401_08383_b200 import placement as pl
    from paper_2401_08383_b200.affinity import Topology
    from paper_2401_08383_b200.model import DTYPE_F32, MoeModel, MoeModelConfig
    cfg = MoeModelConfig(num_experts=8, num_layers=24, d_model=1024, d_ffn=4096, tokens_per_gpu=64, seed=1,
                         gate_affinity=0.8, dtype=DTYPE_F32)
    m = MoeModel(cfg, pl.contiguous_placement(8, 24, Topology(1, 1)))
    x = torch.randn(64, 1024).cuda()
    s = torch.cuda.Stream()
    m.capture(x, s)
    for _ in range(3):
        m.replay(s)
    s.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    for _ in range(10):
        m.replay(s)
    e1.record(s)
    e1.synchronize()
    m.check()
    ms = e0.elapsed_time(e1) / 10
    print(f"fp32 step {ms:.3f} ms, {64 / ms * 1e3:.0f} tok/s, weights {24 * 8 * 33.5e6 / (ms * 1e-3) / 1e12:.2f} TB/s")
