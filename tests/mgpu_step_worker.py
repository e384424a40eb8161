"""Multi-GPU parity at the BASELINE shapes (one process per GPU under torchrun,
launched by tests/test_multi_gpu_shapes.py). Builds the decode stack at the
requested shape on a random placement (tokens cross GPUs), runs two warm
steps through the public one-call step, then one fully checked step through
tests/step_check.check_step: every rank checks its own part of every layer
(routes and permutation exact, sampled output rows within the dtype's bar,
crossed == simulate, histogram == count_transitions, AllGather equal).
Prints "[mgpu-shape] ... OK" on rank 0 when every rank passed."""
import argparse
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--experts", type=int, default=8)
    p.add_argument("--layers", type=int, default=3)
    p.add_argument("--d-model", type=int, default=1024)
    p.add_argument("--d-ffn", type=int, default=4096)
    p.add_argument("--batch", type=int, default=64)
    p.add_argument("--dtype", choices=["bf16", "f32"], default="bf16")
    p.add_argument("--rows", type=int, default=3, help="sampled output rows per layer per rank")
    p.add_argument("--attn-heads", type=int, default=0, help="attention block per layer (0: MoE stack only)")
    p.add_argument("--context", type=int, default=512, help="context capacity per sequence (attention)")
    a = p.parse_args()
    import torch
    import torch.distributed as dist
    from paper_2401_08383_b200 import dist as xd, placement as pl
    from paper_2401_08383_b200.affinity import Topology
    from paper_2401_08383_b200.model import DTYPE_BF16, DTYPE_F32, MoeModel, MoeModelConfig
    from step_check import check_step
    rank = int(os.environ["RANK"])
    G = int(os.environ["WORLD_SIZE"])
    torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", rank)))
    dist.init_process_group("gloo")
    E, L = a.experts, a.layers
    assign = pl.random_placement(E, L, Topology(1, G), seed=11)
    f32 = a.dtype == "f32"
    cfg = MoeModelConfig(num_experts=E, num_layers=L, d_model=a.d_model, d_ffn=a.d_ffn,
                         tokens_per_gpu=a.batch, world_size=G, rank=rank, seed=2024,
                         gate_affinity=0.6, dtype=DTYPE_F32 if f32 else DTYPE_BF16,
                         attn_heads=a.attn_heads, context_len=a.context if a.attn_heads else 0,
                         context_prefix=a.context // 2 if a.attn_heads else 0)
    m = MoeModel(cfg, assign)
    m.connect(xd.exchange_handles(m.ipc_handle()))
    if a.attn_heads:
        # setup AllGather across the GPUs: every replica holds every prompt
        m.context_setup(torch.cuda.current_stream())
        torch.cuda.synchronize()
        dist.barrier()
    g = torch.Generator().manual_seed(500 + rank)
    x = torch.randn(a.batch, a.d_model, generator=g)
    x = (x if f32 else x.to(torch.bfloat16)).cuda()
    s = torch.cuda.Stream()
    for _ in range(2):
        m.step(x, s)
    s.synchronize()
    m.check()
    dist.barrier()
    res = check_step(m, x, assign, rows_per_layer=a.rows)
    # the eager step (layer kernels chained on exit generations, FusedArgs.chain)
    # and a graph replay (griddepcontrol.wait between layers) give the same bits
    # (without attention: with it every step appends a context row)
    if a.attn_heads:
        path = m.describe().get("path")
        if rank == 0:
            tag = (f"G={G} E={E} L={L} d={a.d_model} B={a.batch} attention heads={a.attn_heads} path={path} "
                   f"max rel err {res['max_rel_err_sampled']:.2e} attention {res['attention_max_rel_err_sampled']:.2e}")
            print(f"[mgpu-shape] {tag} {'OK' if res['parity'] == 'ok' else 'FAIL ' + str(res['failures'])}",
                  flush=True)
        dist.barrier()
        m.close()
        dist.destroy_process_group()
        sys.exit(0 if res["parity"] == "ok" else 1)
    m.step(x, s)
    s.synchronize()
    eager = m.output().clone()
    dist.barrier()
    m.capture(x, s)
    m.replay(s)
    s.synchronize()
    m.check()
    if not torch.equal(eager, m.output()):
        res["parity"] = "FAIL"
        res["failures"] = res.get("failures", []) + ["eager (chained) step != graph replay"]
    dist.barrier()
    path = m.describe().get("path")
    if rank == 0:
        tag = (f"G={G} E={E} L={L} d={a.d_model} dff={a.d_ffn} B={a.batch} {a.dtype} path={path} "
               f"routed {res['routed_fraction_checked_step']:.3f} max rel err {res['max_rel_err_sampled']:.2e}")
        if res["parity"] == "ok":
            print(f"[mgpu-shape] {tag} OK", flush=True)
        else:
            print(f"[mgpu-shape] {tag} FAIL {res['failures']}", flush=True)
    dist.barrier()
    m.close()
    dist.destroy_process_group()
    sys.exit(0 if res["parity"] == "ok" else 1)


if __name__ == "__main__":
    main()
