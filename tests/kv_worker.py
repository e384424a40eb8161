"""torchrun worker (one process per GPU): per-step K/V append into every
rank's replica of the context cache over NVLink (CUDA-IPC peer pointers), then
coherent attention over the local replica. Rank r holds the tokens of the
sequences r + G*i (round-robin homes, proj/src/sim.cpp:111) in a shuffled
(dispatch) order. Every rank checks its local replica against the oracle
(oracle/attention.py) bit for bit and its attention outputs within 1e-2.
Launched by tests/test_multi_gpu.py::test_kv_append_replicated."""
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import attention as oatt  # noqa: E402
from paper_2401_08383_b200.attention import (close_replica, coherent_attention,  # noqa: E402
                                             export_replica, import_replica, kv_append)


def main():
    rank, G = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", rank)))
    dist.init_process_group("nccl", device_id=torch.device("cuda", torch.cuda.current_device()))
    B, H, Dh, Cap, steps = 6, 8, 64, 256, 3  # >1 MB caches: one allocator segment each
    S = G * B
    g = torch.Generator().manual_seed(11)
    k0 = torch.randn(S, H, Cap, Dh, generator=g).to(torch.bfloat16)
    v0 = torch.randn(S, H, Cap, Dh, generator=g).to(torch.bfloat16)
    ctx0 = torch.randint(0, Cap - steps, (S,), generator=g, dtype=torch.int32)
    ctx0[0] = Cap - 1  # fills up during the run -> overflow on the next steps
    k, v, ctx = k0.cuda(), v0.cuda(), ctx0.clone().cuda()
    shared = [export_replica(t) for t in (k, v, ctx)]
    everyone = [None] * G
    dist.all_gather_object(everyone, shared)
    # map the peers' buffers on this GPU (CUDA IPC, NVLink peer access)
    peers = [None if p == rank else
             [import_replica(h, off, t.shape, t.dtype) for (h, off), t in zip(everyone[p], (k, v, ctx))]
             for p in range(G)]
    order = [rank] + [p for p in range(G) if p != rank]  # replica 0 = local
    ks = [k if p == rank else peers[p][0] for p in order]
    vs = [v if p == rank else peers[p][1] for p in order]
    cs = [ctx if p == rank else peers[p][2] for p in order]
    ok, ov, oc = k0.float().numpy().copy(), v0.float().numpy().copy(), ctx0.numpy().copy()
    overflow = torch.zeros(1, dtype=torch.int32, device="cuda")
    want_over = 0
    for step in range(steps):
        gs = torch.Generator().manual_seed(100 + step)  # same on every rank
        kn_all = torch.randn(S, H, Dh, generator=gs).to(torch.bfloat16)
        vn_all = torch.randn(S, H, Dh, generator=gs).to(torch.bfloat16)
        q_all = torch.randn(S, H, Dh, generator=gs).to(torch.bfloat16)
        mine = torch.arange(rank, S, G)[torch.randperm(B, generator=gs)]
        seq = mine.to(torch.int32)
        kv_append(kn_all[mine].contiguous().cuda(), vn_all[mine].contiguous().cuda(),
                  seq.cuda(), ks, vs, cs, overflow)
        torch.cuda.synchronize()
        dist.barrier()
        # oracle: all ranks' tokens (one per sequence, so the order is free)
        want_over += oatt.kv_append(kn_all.float().numpy(), vn_all.float().numpy(),
                                    np.arange(S), ok, ov, oc)
        assert ctx.cpu().numpy().tolist() == oc.tolist(), (rank, step)
        assert np.array_equal(k.float().cpu().numpy(), ok), (rank, step)
        assert np.array_equal(v.float().cpu().numpy(), ov), (rank, step)
        out = coherent_attention(q_all[mine].contiguous().cuda(), seq.cuda(), ctx, k, v)
        torch.cuda.synchronize()
        ref = oatt.coherent_attention(q_all[mine].float().numpy(), seq.numpy(), oc, ok, ov,
                                      Dh ** -0.5)
        err = np.abs(out.float().cpu().numpy() - ref).max()
        assert err <= 1e-2 * max(np.abs(ref).max(), 1.0), (rank, step, err)
        dist.barrier()
    total_over = overflow.clone()
    dist.all_reduce(total_over)
    assert int(total_over.item()) == want_over, (int(total_over.item()), want_over)
    if rank == 0:
        print(f"kv_append replicated over {G} GPUs: OK (steps {steps}, overflow "
              f"{want_over})", flush=True)
    torch.cuda.synchronize()
    dist.barrier()
    for p in range(G):
        if peers[p] is not None:
            for t, (h, off) in zip(peers[p], everyone[p]):
                close_replica(t, off)
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
