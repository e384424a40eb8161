"""Profiling driver: builds the bench model (BASELINE configs[1], N=1) and runs
decode steps through the phased (non-graph) API so every kernel launch is
visible to ncu. Usage: python tools/profile_step.py [--steps N]."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--steps", type=int, default=2)
    p.add_argument("--batch", type=int, default=64)
    p.add_argument("--experts", type=int, default=8)
    p.add_argument("--layers", type=int, default=24)
    a = p.parse_args()
    import torch
    from paper_2401_08383_b200 import placement as pl
    from paper_2401_08383_b200.affinity import Topology
    from paper_2401_08383_b200.model import MoeModel, MoeModelConfig
    cfg = MoeModelConfig(num_experts=a.experts, num_layers=a.layers, d_model=1024, d_ffn=4096,
                         tokens_per_gpu=a.batch, seed=1234, gate_affinity=0.8)
    m = MoeModel(cfg, pl.contiguous_placement(a.experts, a.layers, Topology(1, 1)))
    x = torch.randn(a.batch, 1024).to(torch.bfloat16).cuda()
    s = torch.cuda.Stream()
    for _ in range(a.steps):
        m.step(x, s)
    s.synchronize()
    m.check()
    print("profile_step ok")


if __name__ == "__main__":
    main()
