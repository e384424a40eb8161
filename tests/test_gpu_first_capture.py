"""The public one-call step captured as the FIRST work of a fresh process
(exf_model_capture before any eager step): every host-side setup that is
illegal inside a stream capture (synchronous symbol copies, mapped host
allocations) must already have happened at model create. Regression: the
fused layer kernel's diagnostics channel was set up lazily on the first
launch, and a capture that contained that launch was invalidated.

Runs in a subprocess so that no earlier test has warmed the launchers."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

SCRIPT = r"""
import sys, torch
sys.path.insert(0, {root!r})
from paper_2401_08383_b200 import placement as pl
from paper_2401_08383_b200.affinity import Topology
from paper_2401_08383_b200.model import MoeModel, MoeModelConfig
kw = dict(num_experts={E}, num_layers=3, d_model=1024, d_ffn=2048, tokens_per_gpu=8, seed=11, gate_affinity=0.8,
          attn_heads={H}, context_len=512, context_prefix=100)
assign = pl.contiguous_placement({E}, 3, Topology(1, 1))
m = MoeModel(MoeModelConfig(**kw), assign)
s = torch.cuda.Stream()
if {H}:
    m.context_setup(s, phase=3)
    s.synchronize()
x = torch.randn(8, 1024, generator=torch.Generator().manual_seed(1)).to(torch.bfloat16).cuda()
m.capture(x, s)
m.replay(s)
s.synchronize()
m.check()
ref = MoeModel(MoeModelConfig(**kw), assign)
if {H}:
    ref.context_setup(s, phase=3)
ref.step(x, s)
s.synchronize()
ref.check()
assert torch.equal(m.output(), ref.output())
print("FIRST_CAPTURE_OK")
"""


@pytest.mark.parametrize("E,H", [(8, 0), (64, 16)])
def test_capture_before_any_eager_step(E, H):
    code = SCRIPT.format(root=ROOT, E=E, H=H)
    r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0 and "FIRST_CAPTURE_OK" in r.stdout, r.stdout[-2000:] + r.stderr[-4000:]
