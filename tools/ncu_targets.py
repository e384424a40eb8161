"""Small driver for ncu captures (diagnostics): python tools/ncu_targets.py WHAT
  step      -- 3 bf16 decode steps at BASELINE configs[1] (layer_fused_kernel)
  fp32      -- 2 fp32-mode steps at configs[1] (gate_dispatch f32, ffn_f32_kernel)
  routing   -- exf_count_transitions + exf_route_replay on a 2^21 x 24 trace (E=8, E=64)
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    what = sys.argv[1] if len(sys.argv) > 1 else "step"
    import numpy as np
    import torch
    from paper_2401_08383_b200 import _capi, affinity, placement as pl
    from paper_2401_08383_b200.model import DTYPE_F32, MoeModel, MoeModelConfig
    if what in ("step", "fp32"):
        f32 = what == "fp32"
        cfg = MoeModelConfig(num_experts=8, num_layers=24, d_model=1024, d_ffn=4096, tokens_per_gpu=64,
                             seed=1234, gate_affinity=0.8, dtype=DTYPE_F32 if f32 else 0)
        m = MoeModel(cfg, pl.contiguous_placement(8, 24, affinity.Topology(1, 1)))
        x = torch.randn(64, 1024).cuda()
        x = x if f32 else x.to(torch.bfloat16)
        s = torch.cuda.Stream()
        for _ in range(2 if f32 else 3):
            m.step(x, s)
        s.synchronize()
        m.check()
        print("ok", m.describe())
        return
    lib = _capi.load()
    T, L = 1 << 21, 24
    for E in (8, 64):
        paths = pl.generate_markov_trace(E, L, T, 0.8, 8, 3)
        assign = pl.contiguous_placement(E, L, affinity.Topology(1, 8))
        dp = torch.from_numpy(paths).cuda()
        da = torch.from_numpy(np.ascontiguousarray(assign, np.int32)).cuda()
        cnt = torch.empty((L - 1) * E * E, dtype=torch.int64, device="cuda")
        tot = torch.empty((L - 1) * E, dtype=torch.int64, device="cuda")
        ws = torch.empty(max(lib.exf_count_transitions_workspace_bytes(T, L, E, 1), 1), dtype=torch.uint8,
                         device="cuda")
        ctr = torch.empty(6, dtype=torch.int64, device="cuda")
        for _ in range(2):
            _capi.call("exf_count_transitions", dp.data_ptr(), T, L, E, 1, cnt.data_ptr(), tot.data_ptr(),
                       ws.data_ptr(), None)
            _capi.call("exf_route_replay", dp.data_ptr(), None, da.data_ptr(), T, L, E, 1, 8, 1,
                       ctr.data_ptr(), None)
        torch.cuda.synchronize()
    print("ok routing")


if __name__ == "__main__":
    main()
