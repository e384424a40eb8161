"""The C++ mirror of the reference API (include/exflow/exflow.hpp), compiled
into a standalone caller (tests/cpp/test_mirror.cpp, built by build() into
build/test_mirror and linked against libexflow_b200.so) that runs the
reference's known-answer tests the way its own callers would: trace and
placement I/O, token_hops, the placement table, the solver, exception types
and messages (host group, CPU); count_transitions and simulate through the
GPU kernels (gpu group). Also exf_token_hops through the C-ABI."""
import os
import subprocess

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
EXE = os.path.join(ROOT, "build", "test_mirror")
GOLDEN = os.path.join(ROOT, "tests", "golden")


def _run(group):
    if not os.path.exists(EXE):
        subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "paper_2401_08383_b200", "csrc")],
                       check=True)
    r = subprocess.run([EXE, group, GOLDEN], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "0 failures" in r.stdout
    return r.stdout


def test_cpp_mirror_host_group():
    out = _run("host")
    assert int(out.split(":")[1].split()[0]) >= 50


@pytest.mark.gpu
def test_cpp_mirror_gpu_group():
    _run("gpu")


def test_token_hops_capi_matches_reference_kats():
    # proj/tests/test_sim.cpp:44-54 on the contiguous 1x4 placement
    from paper_2401_08383_b200 import affinity, _capi
    from paper_2401_08383_b200 import placement as pl
    t4 = affinity.Topology(1, 4)
    a = pl.contiguous_placement(8, 3, t4)
    tot = lambda path, home, mode: int(affinity.token_hops(path, home, a, mode, t4)[2].sum())
    assert tot([0, 4, 2], 1, affinity.VANILLA) == 4
    assert tot([0, 4, 2], 1, affinity.COHERENT) == 3
    assert tot([5, 5, 4], 3, affinity.VANILLA) == 6
    assert tot([5, 5, 4], 3, affinity.COHERENT) == 1
    crossed, tier, hops = affinity.token_hops([0, 4, 2], 1, a, affinity.COHERENT, t4)
    assert crossed.tolist() == [True, True, True] and tier.tolist() == [1, 1, 1]
    with pytest.raises(_capi.ExflowInvalidArgument, match="home gpu out of range"):
        affinity.token_hops([0, 4, 2], 4, a, affinity.VANILLA, t4)


def test_token_hops_sum_equals_oracle_replay(orc):
    # per-token semantics summed over a seeded trace == the oracle's simulate
    from paper_2401_08383_b200 import affinity
    from paper_2401_08383_b200 import placement as pl
    topo = affinity.Topology(2, 2)
    paths = orc.generate_markov_trace(8, 5, 300, 0.7, 2, 9)
    a = pl.random_placement(8, 5, topo, 4)
    for mode in (affinity.VANILLA, affinity.COHERENT):
        hops = sum(int(affinity.token_hops(paths[t], t % 4, a, mode, topo)[2].sum())
                   for t in range(paths.shape[0]))
        rep = orc.simulate(paths, a, 2, 2, orc.VANILLA if mode == affinity.VANILLA else orc.COHERENT)
        assert hops == rep.hops_intra_node + rep.hops_inter_node
