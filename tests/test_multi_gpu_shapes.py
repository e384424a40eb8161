"""Real multi-GPU parity at the BASELINE.json shapes (needs >= G visible
B200s; skipped otherwise). One process per GPU (torchrun), the ranks'
kernels exchanging tokens over NVLink peer memory; every rank checks its own
part of one full decode step against the CPU oracle (tests/step_check.py):
  configs[1]  E=8,  d=1024, d_ffn=4096, B=64     at G=2 and G=4 (fused path)
  configs[2]  E=16, d=1024, d_ffn=4096, B=64     at G=2 and G=4
  configs[3]  E=32, d=2048, d_ffn=8192, B=64/256/512 at G=4
  fp32 mode   configs[1] shape                   at G=2 (<= 1e-5)
  attention   configs[1] layer + 16-head attention block at G=2, configs[4]
              (E=64, 8 sequences/GPU) at G=4: setup AllGather across GPUs,
              K/V rows appended into every GPU's replica, attention on the
              GPU the dispatch left each token on
"""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

HERE = os.path.dirname(os.path.abspath(__file__))

CASES = [
    # (G, experts, d, dff, batch, dtype, port)
    (2, 8, 1024, 4096, 64, "bf16", 29711),
    (4, 8, 1024, 4096, 64, "bf16", 29712),
    (2, 16, 1024, 4096, 64, "bf16", 29713),
    (4, 16, 1024, 4096, 64, "bf16", 29714),
    (4, 32, 2048, 8192, 64, "bf16", 29715),
    (4, 32, 2048, 8192, 256, "bf16", 29716),
    # G*C = 8192 route slots: the largest the fused dispatch path takes
    (4, 32, 2048, 8192, 512, "bf16", 29720),
    # 5120 route slots with a 64-token natural tile: the 128-token variant is forced
    (4, 64, 1024, 4096, 320, "bf16", 29721),
    (2, 8, 1024, 4096, 64, "f32", 29717),
]
ATTN_CASES = [
    # (G, experts, batch, heads, context, port)
    (2, 8, 16, 16, 512, 29718),
    (4, 64, 8, 16, 1024, 29719),
]


def _gpus():
    import torch
    return torch.cuda.device_count() if torch.cuda.is_available() else 0


@pytest.mark.parametrize("G,E,d,dff,B,dtype,port", CASES,
                         ids=[f"G{c[0]}-E{c[1]}-d{c[2]}-B{c[4]}-{c[5]}" for c in CASES])
def test_baseline_shape_parity(G, E, d, dff, B, dtype, port):
    if _gpus() < G:
        pytest.skip(f"needs {G} GPUs")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", str(G),
           "--master-addr", "127.0.0.1", "--master-port", str(port),
           os.path.join(HERE, "mgpu_step_worker.py"), "--experts", str(E), "--d-model", str(d),
           "--d-ffn", str(dff), "--batch", str(B), "--dtype", dtype]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    assert " OK" in r.stdout, r.stdout[-2000:]
    print(r.stdout.strip().splitlines()[-1])


@pytest.mark.parametrize("G,E,B,H,ctx,port", ATTN_CASES,
                         ids=[f"G{c[0]}-E{c[1]}-B{c[2]}-attn" for c in ATTN_CASES])
def test_attention_block_across_gpus(G, E, B, H, ctx, port):
    if _gpus() < G:
        pytest.skip(f"needs {G} GPUs")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", str(G),
           "--master-addr", "127.0.0.1", "--master-port", str(port),
           os.path.join(HERE, "mgpu_step_worker.py"), "--experts", str(E), "--batch", str(B),
           "--attn-heads", str(H), "--context", str(ctx), "--rows", "2"]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    assert " OK" in r.stdout, r.stdout[-2000:]
    print(r.stdout.strip().splitlines()[-1])
