"""Quick step-time probe (diagnostics): the bench model (BASELINE configs[1],
N=1, contiguous placement) captured in a CUDA graph and replayed; prints the
mean device time per decode step. Knobs come from the EXF_* environment.
Usage: python tools/step_time.py [--reps N] [--batch B]"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--reps", type=int, default=50)
    p.add_argument("--batch", type=int, default=64)
    p.add_argument("--experts", type=int, default=8)
    p.add_argument("--layers", type=int, default=24)
    p.add_argument("--d-model", type=int, default=1024)
    p.add_argument("--d-ffn", type=int, default=4096)
    p.add_argument("--eager", action="store_true", help="time exf_model_step calls instead of graph replays")
    a = p.parse_args()
    import torch
    from paper_2401_08383_b200 import placement as pl
    from paper_2401_08383_b200.affinity import Topology
    from paper_2401_08383_b200.model import MoeModel, MoeModelConfig
    G = int(os.environ.get("WORLD_SIZE", "1"))  # under torchrun: one process per GPU
    rank = int(os.environ.get("RANK", "0"))
    if G > 1:
        import torch.distributed as dist
        from paper_2401_08383_b200 import dist as xd
        torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", rank)))
        dist.init_process_group("gloo")
    cfg = MoeModelConfig(num_experts=a.experts, num_layers=a.layers, d_model=a.d_model, d_ffn=a.d_ffn,
                         tokens_per_gpu=a.batch, seed=1234, gate_affinity=0.8, world_size=G, rank=rank)
    m = MoeModel(cfg, pl.contiguous_placement(a.experts, a.layers, Topology(1, G)))
    if G > 1:
        m.connect(xd.exchange_handles(m.ipc_handle()))
    x = torch.randn(a.batch, a.d_model).to(torch.bfloat16).cuda()
    s = torch.cuda.Stream()
    for _ in range(3):
        m.step(x, s)
    run = (lambda: m.step(x, s)) if a.eager else (lambda: m.replay(s))
    if not a.eager:
        m.capture(x, s)
    for _ in range(5):
        run()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.synchronize()
    e0.record(s)
    for _ in range(a.reps):
        run()
    e1.record(s)
    e1.synchronize()
    m.check()
    us = e0.elapsed_time(e1) * 1000.0 / a.reps
    if G > 1:
        t = torch.tensor([us], dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        us = float(t.item())
        if rank != 0:
            return
    knobs = {k: v for k, v in os.environ.items() if k.startswith("EXF_")}
    wbytes = a.experts // G * 2 * a.d_model * a.d_ffn * 2  # every local expert active (weights dominate)
    print(f"G={G} step {us:.1f} us  ({us / a.layers:.2f} us/layer, {a.batch * G / us * 1e6:.0f} tok/s, "
          f"weights {wbytes / (us / a.layers * 1e-6) / 1e12:.2f} TB/s, {m.describe().get('path')}"
          f"{' dense' if m.describe().get('layer_kernel', {}).get('dense') else ''})  {knobs}")


if __name__ == "__main__":
    main()
