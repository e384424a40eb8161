"""CPU (gloo, world_size 2) tests of the multi-rank host logic: IPC-handle
exchange, exact histogram reduction, and placement agreement (rank 0 solves
solve_staged on the summed counts, every rank receives the same table)."""
import os
import socket

import numpy as np
import pytest


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import oracle as orc
        from paper_2401_08383_b200 import dist as xd
        from paper_2401_08383_b200.affinity import Topology
        handles = xd.exchange_handles(bytes([rank]) * 64)
        # each rank counts the transitions of its own half of the tokens
        paths = orc.generate_markov_trace(16, 6, 4000, 0.9, 4, 3)
        mine = paths[rank::world]
        counts, _ = orc.count_transitions(mine, 16)
        total = xd.sum_counts(counts)
        assign = xd.agree_placement(total, Topology(1, 4))
        routes = np.full((8, 3), -1, np.int32)
        routes[rank::world] = rank + 1
        merged = xd.merge_routes(routes)
        mx = xd.max_over_ranks(float(rank * 10))
        q.put((rank, [h[0] for h in handles], total, assign, merged, mx))
    finally:
        dist.destroy_process_group()


def test_gloo_two_ranks_agree():
    import torch.multiprocessing as mp
    from oracle import oracle as orc
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted([q.get(timeout=240) for _ in procs], key=lambda r: r[0])
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    paths = orc.generate_markov_trace(16, 6, 4000, 0.9, 4, 3)
    want, _ = orc.count_transitions(paths, 16)
    for rank, handles, total, assign, merged, mx in res:
        assert handles == [0, 1]
        assert np.array_equal(total, want)            # exact integer all-reduce
        assert np.array_equal(assign, res[0][3])       # same table on every rank
        orc.validate_placement(assign, 4)
        assert (merged[0::2] == 1).all() and (merged[1::2] == 2).all()
        assert mx == 10.0
    # the agreed placement is never worse than the vanilla one on the full trace
    # (the planted groups here are the contiguous blocks, so both are optimal)
    from paper_2401_08383_b200 import placement as pl
    from paper_2401_08383_b200.affinity import Topology
    base = pl.objective_crossings(want, pl.contiguous_placement(16, 6, Topology(1, 4)))
    assert pl.objective_crossings(want, res[0][3]) <= base
