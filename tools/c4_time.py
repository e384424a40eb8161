"""configs[4]-shaped decode step time (diagnostics): E experts top-1, attention
block over the replicated context (H heads, ctx keys), B sequences per GPU;
under torchrun one process per GPU. Usage: python tools/c4_time.py [E B ctx]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

if __name__ == "__main__":
    import torch
    from paper_2401_08383_b200 import placement as pl
    from paper_2401_08383_b200.affinity import Topology
    from paper_2401_08383_b200.model import MoeModel, MoeModelConfig
    E = int(sys.argv[1]) if len(sys.argv) > 1 else 64
    B = int(sys.argv[2]) if len(sys.argv) > 2 else 8
    ctx = int(sys.argv[3]) if len(sys.argv) > 3 else 16384
    G = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if G > 1:
        import torch.distributed as dist
        from paper_2401_08383_b200 import dist as xd
        torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", rank)))
        dist.init_process_group("gloo")
    cfg = MoeModelConfig(num_experts=E, num_layers=24, d_model=1024, d_ffn=4096, tokens_per_gpu=B, world_size=G,
                         rank=rank, seed=4321, gate_affinity=0.8, attn_heads=16, context_len=ctx,
                         context_prefix=ctx - 64)
    m = MoeModel(cfg, pl.contiguous_placement(E, 24, Topology(1, G)))
    if G > 1:
        m.connect(xd.exchange_handles(m.ipc_handle()))
    s = torch.cuda.Stream()
    m.context_setup(s, phase=3)
    x = torch.randn(B, 1024).to(torch.bfloat16).cuda()
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
    if G > 1:
        t = torch.tensor([ms], dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    if rank == 0:
        kv = B * G * 16 * ctx * 64 * 4 / G  # K+V bytes read per layer per GPU (avg)
        print(f"c4 G={G} E={E} B={B} ctx={ctx}: {ms:.3f} ms/step, {B * G / ms * 1e3:.0f} tok/s, "
              f"attention K/V {kv * 24 / (ms * 1e-3) / 1e12:.2f} TB/s of the step")
