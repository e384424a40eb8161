"""Diagnostics: build a model of the given shape (E L d d_ffn B), run two steps and
report the fused kernel's timeout channel (exf_debug_last_timeout) on failure.
Usage: python tools/probe_config.py E L d dff B"""
import os, sys, ctypes as C, numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2401_08383_b200 import placement as pl
from paper_2401_08383_b200.affinity import Topology
from paper_2401_08383_b200.model import MoeModel, MoeModelConfig
E, L, d, f, B = map(int, sys.argv[1:6])
m = MoeModel(MoeModelConfig(num_experts=E, num_layers=L, d_model=d, d_ffn=f, tokens_per_gpu=B, seed=3),
             pl.contiguous_placement(E, L, Topology(1, 1)))
print(m.describe(), flush=True)
x = torch.randn(B, d).to(torch.bfloat16).cuda()
try:
    for _ in range(2):
        m.step(x)
    torch.cuda.synchronize()
    m.check()
except Exception as ex:
    from paper_2401_08383_b200 import _capi
    w = (C.c_int32 * 12)()
    _capi.load().exf_debug_last_timeout(w)
    print("FAILED", E, L, d, f, B, "timeout words", list(w), str(ex)[:80], flush=True)
    sys.exit(1)
print("OK", E, L, d, f, B, os.environ.get("EXF_DENSE"), flush=True)
