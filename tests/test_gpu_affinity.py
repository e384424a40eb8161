"""GPU parity: kernel (5) histogram and the routing replay vs the CPU oracle.

Bit-exact integer equality on the reference KATs (proj/tests/test_trace.cpp,
test_sim.cpp), on seeded synthetic traces, at BASELINE sizes (2^20 tokens),
and on edge cases (single token, single expert, gap = L-1, E = 64).
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def aff():
    from paper_2401_08383_b200 import _capi, affinity
    if _capi.load().exf_device_ok() != 1:
        pytest.fail("no sm_100 GPU visible to libexflow_b200.so")
    return affinity


def _eq(aff, orc, paths, E, gap):
    got = aff.count_transitions(paths, E, gap)
    want, tot = orc.count_transitions(paths, E, gap, threads=4)
    assert np.array_equal(got.matrices, want)
    assert np.array_equal(got.row_totals, tot)
    return got


def test_hand_count_kats(aff, orc):
    got = _eq(aff, orc, np.array([[0, 0], [0, 0], [0, 1], [1, 1]], np.int32), 2, 1)
    assert got.matrices[0].tolist() == [[2, 1], [0, 1]] and got.row_totals[0].tolist() == [3, 1]
    got = _eq(aff, orc, np.array([[0, 1, 0]], np.int32), 2, 2)
    assert got.matrices[0, 0, 0] == 1 and got.matrices.sum() == 1
    _eq(aff, orc, np.zeros((3, 2), np.int32), 1, 1)  # single expert


def test_acceptance_random_traces(aff, orc):
    # proj/tests/acceptance.cpp:343-369: 1,000 random traces, conservation + rows
    rng = orc.Rng(99)
    for _ in range(1000):
        experts = 1 + rng.below_int(6)
        layers = 2 + rng.below_int(4)
        tokens = 1 + rng.below_int(40)
        paths = np.array([rng.below_int(experts) for _ in range(layers * tokens)],
                         np.int32).reshape(tokens, layers)
        gap = 1 + rng.below_int(layers - 1)
        got = _eq(aff, orc, paths, experts, gap)
        assert (got.matrices.sum(axis=(1, 2)) == tokens).all()
        probs = aff.conditional_probabilities(got)
        assert np.allclose(probs.matrices.sum(axis=2), probs.seen.astype(float), atol=1e-9)


@pytest.mark.parametrize("E,L,T,gap", [(8, 4, 256, 1), (8, 24, 1 << 20, 1), (16, 24, 300001, 3),
                                       (32, 24, 1 << 18, 1), (64, 24, 1 << 20, 1),
                                       (64, 24, 70000, 23), (5, 7, 1, 6)])
def test_synthetic_sizes_bit_exact(aff, orc, E, L, T, gap):
    groups = 4 if E % 4 == 0 else 1
    paths = orc.generate_markov_trace(E, L, T, 0.8, groups, E * 1000 + L)
    got = _eq(aff, orc, paths, E, gap)
    assert (got.matrices.sum(axis=(1, 2)) == T).all()  # size-independent: conservation


def test_token_order_invariance(aff, orc):
    paths = orc.generate_markov_trace(16, 6, 50000, 0.7, 4, 3)
    perm = np.random.default_rng(0).permutation(50000)
    a = aff.count_transitions(paths, 16).matrices
    b = aff.count_transitions(paths[perm], 16).matrices
    assert np.array_equal(a, b)


def test_replay_demo_and_kats(aff, orc):
    demo = np.array([[0, 4, 2], [5, 5, 4]], np.int32)
    a = orc.contiguous_placement(8, 3, 4)
    topo = aff.Topology(1, 4)
    v = aff.simulate(demo, a, aff.SimConfig(mode=aff.VANILLA, topology=topo, homes=[1, 3]))
    assert v.total_crossings() == 10 and v.hops_inter_node == 0 and v.p == pytest.approx(5 / 6)
    c = aff.simulate(demo, a, aff.SimConfig(mode=aff.COHERENT, topology=topo, homes=[1, 3]))
    assert c.total_crossings() == 4 and c.p_star == pytest.approx(4 / 6)
    assert (c.alltoall_count, c.allgather_count, c.setup_allgather_count) == (3, 1, 1)
    assert (v.alltoall_count, v.allgather_count) == (6, 0)


@pytest.mark.parametrize("E,L,T,nodes,gpn", [(8, 4, 256, 1, 2), (8, 4, 256, 1, 4),
                                             (8, 4, 256, 1, 8), (64, 24, 1 << 20, 1, 8),
                                             (32, 12, 50000, 2, 4), (16, 24, 100003, 4, 2)])
def test_replay_matches_oracle(aff, orc, E, L, T, nodes, gpn):
    paths = orc.generate_markov_trace(E, L, T, 0.8, 4, 42 + E)
    for seed, assign in enumerate([orc.contiguous_placement(E, L, nodes * gpn),
                                   orc.random_placement(E, L, nodes * gpn, 5)]):
        for mode in (0, 1):
            got = aff.simulate(paths, assign, aff.SimConfig(
                mode=mode, topology=aff.Topology(nodes, gpn)))
            want = orc.simulate(paths, assign, nodes, gpn, mode, threads=4)
            for f in ("hops_intra_node", "hops_inter_node", "locality_gpu", "locality_node", "p",
                      "p_star", "alltoall_count", "allgather_count", "volume_units",
                      "estimated_latency"):
                assert getattr(got, f) == getattr(want, f), f


def test_replay_survey_probe(aff, orc):
    paths = orc.generate_markov_trace(8, 4, 256, 0.8, 4, 42)
    for g, pstar in ((2, 0.199219), (4, 0.282227), (8, 0.665039)):
        r = aff.simulate(paths, orc.contiguous_placement(8, 4, g),
                         aff.SimConfig(mode=aff.COHERENT, topology=aff.Topology(1, g)))
        assert round(r.p_star, 6) == pstar


def test_replay_rejects_bad_inputs(aff, orc):
    demo = np.array([[0, 4, 2], [5, 5, 4]], np.int32)
    a = orc.contiguous_placement(8, 3, 4)
    with pytest.raises(aff._capi.ExflowInvalidArgument):
        aff.simulate(demo, a, aff.SimConfig(topology=aff.Topology(1, 4), homes=[1]))
    with pytest.raises(aff._capi.ExflowInvalidArgument):
        aff.simulate(demo, a, aff.SimConfig(topology=aff.Topology(1, 4), homes=[1, 9]))
    with pytest.raises(aff._capi.ExflowInvalidArgument):
        aff.simulate(demo, a, aff.SimConfig(topology=aff.Topology(2, 4)))
