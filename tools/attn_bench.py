"""Measure exf_coherent_attention on B200 (one JSON line per shape).

Workload: BASELINE configs[4] (d=1024 -> 16 heads x 64, context 16k, B=8
decode tokens resident per GPU per layer) plus a wider B. Algorithmic bytes
per call = sum_tokens H * ctx_len * Dh * 2 (K) * 2 (V) + q + out; the K/V set
(268 MB at B=8) is larger than the 126 MB L2, so no flush is needed between
iterations. Times the launch(es) with CUDA events on the launching stream.
Usage: python tools/attn_bench.py [--iters 50]
"""
import argparse
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2401_08383_b200 import _capi  # noqa: E402
from paper_2401_08383_b200.attention import coherent_attention  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--iters", type=int, default=50)
    a = ap.parse_args()
    peaks = {}
    pk = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                      "MEASURED_PEAKS.json")
    if os.path.exists(pk):
        peaks = json.load(open(pk))
    peak = float(peaks.get("hbm_gbs", 6558.1))
    for (B, H, Dh, Cap) in [(8, 16, 64, 16384), (32, 16, 64, 16384), (8, 8, 128, 16384)]:
        g = torch.Generator(device="cuda").manual_seed(0)
        q = torch.randn(B, H, Dh, device="cuda", generator=g).to(torch.bfloat16)
        k = torch.randn(B, H, Cap, Dh, device="cuda", generator=g).to(torch.bfloat16)
        v = torch.randn(B, H, Cap, Dh, device="cuda", generator=g).to(torch.bfloat16)
        seq = torch.randperm(B, device="cuda").to(torch.int32)
        ctx = torch.full((B,), Cap, dtype=torch.int32, device="cuda")
        out = torch.empty_like(q)
        ws = torch.zeros(max(_capi.load().exf_coherent_attention_workspace_bytes(B, H, Dh, Cap), 1),
                         dtype=torch.uint8, device="cuda")
        for _ in range(5):
            coherent_attention(q, seq, ctx, k, v, out=out, workspace=ws)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(a.iters):
            coherent_attention(q, seq, ctx, k, v, out=out, workspace=ws)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / a.iters
        byts = B * H * Cap * Dh * 2 * 2 + 2 * B * H * Dh * 2
        gbs = byts / (ms * 1e-3) / 1e9
        print(json.dumps({"kernel": "coherent_attn_kernel (split-KV, in-kernel merge)", "tokens": B, "heads": H,
                          "head_dim": Dh, "context": Cap, "ms_per_call": ms,
                          "bytes_per_call": byts, "achieved_gbs": gbs, "peak_gbs": peak,
                          "frac": gbs / peak, "tokens_per_s_per_layer": B / (ms * 1e-3),
                          "peak_source": "MEASURED_PEAKS.json hbm_gbs" if peaks else "fallback"}))


if __name__ == "__main__":
    main()
