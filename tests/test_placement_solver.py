"""CPU tests of the host placement solver (csrc/host/solver.cpp, placement_table.cpp via the
C-ABI) against the oracle's brute force and the reference's KATs
(proj/tests/test_placement.cpp, proj/tests/acceptance.cpp criteria 4-7)."""
import numpy as np
import pytest

from paper_2401_08383_b200 import _capi
from paper_2401_08383_b200 import placement as pl
from paper_2401_08383_b200.affinity import Topology


def _random_counts(orc, experts, layers, tokens, seed):
    # proj/tests/test_placement.cpp:34-46 (Rng(seed), row-major below_int draws)
    rng = orc.Rng(seed)
    paths = np.array([rng.below_int(experts) for _ in range(tokens * layers)],
                     np.int32).reshape(tokens, layers)
    return orc.count_transitions(paths, experts)[0]


def test_dp_diagonal_and_antidiagonal():
    # test_placement.cpp:56-73
    a, r = pl.solve_exact_dp(np.array([[[10, 0], [0, 10]]], np.int64), 2)
    assert r.objective == 0.0 and a[0, 0] == a[1, 0] and a[0, 1] == a[1, 1]
    a, r = pl.solve_exact_dp(np.array([[[0, 10], [10, 0]]], np.int64), 2)
    assert r.objective == 0.0 and a[0, 0] == a[1, 1] and a[0, 1] == a[1, 0]


def test_dp_rejections_and_state_cap(orc):
    # :75-79, :103-112
    with pytest.raises(_capi.ExflowInvalidArgument):
        pl.solve_exact_dp(_random_counts(orc, 3, 2, 10, 1), 2)
    assert pl.balanced_assignment_count(8, 2) == 70
    assert pl.balanced_assignment_count(16, 2) == 10001
    assert pl.balanced_assignment_count(4, 4) == 24
    assert pl.balanced_assignment_count(4, 1) == 1
    with pytest.raises(_capi.ExflowInvalidArgument, match="local-search"):
        pl.solve_exact_dp(_random_counts(orc, 16, 2, 50, 2), 2)


def test_uniform_weights_cost_sixteen(orc):
    # :81-89
    counts = np.ones((2, 4, 4), np.int64)
    assert orc.brute_force_optimum(counts, 2) == 16.0
    assert pl.solve_exact_dp(counts, 2)[1].objective == 16.0


def test_dp_equals_brute_force(orc):
    # :91-101 and acceptance.cpp:187-212 (criterion 4, 20 instances Rng(4242))
    for rnd in range(8):
        e, l = (4 if rnd % 2 == 0 else 6), 2 + rnd % 2
        c = _random_counts(orc, e, l, 120, 100 + rnd)
        a, r = pl.solve_exact_dp(c, 2)
        assert r.objective == orc.brute_force_optimum(c, 2)
        assert r.objective == orc.objective_crossings(c, a)
        orc.validate_placement(a, 2)
    rng = orc.Rng(4242)
    for i in range(20):
        e, l = (4 if i % 2 == 0 else 6), 2 + (i // 2) % 2
        paths = np.array([rng.below_int(e) for _ in range(150 * l)], np.int32).reshape(150, l)
        c = orc.count_transitions(paths, e)[0]
        a, r = pl.solve_exact_dp(c, 2)
        assert r.objective == orc.brute_force_optimum(c, 2)
        # criterion 5: annealing within 2% of the exact optimum, never below
        _, ls = pl.solve_local_search(c, 2, pl.AnnealParams(seed=77 + i))
        assert dp_ok(ls.objective, r.objective)


def dp_ok(ls, dp):
    return dp - 1e-9 <= ls <= dp * 1.02 + 1e-9


def test_local_search_planted_and_singletons(orc):
    # :114-139
    paths = orc.generate_markov_trace(8, 4, 2000, 1.0, 4, 5)
    c = orc.count_transitions(paths, 8)[0]
    a, r = pl.solve_local_search(c, 4, pl.AnnealParams(seed=7))
    assert r.objective == 0.0 and orc.objective_crossings(c, a) == 0.0
    for seed in range(6):
        c = _random_counts(orc, 4, 3, 60, 300 + seed)
        assert (pl.solve_local_search(c, 4, pl.AnnealParams(seed=seed))[1].objective ==
                pl.solve_exact_dp(c, 4)[1].objective)
    for seed in range(6):  # :141-151 soundness
        c = _random_counts(orc, 6, 3, 80, 400 + seed)
        a, ls = pl.solve_local_search(c, 2, pl.AnnealParams(seed=seed))
        assert ls.objective >= pl.solve_exact_dp(c, 2)[1].objective - 1e-9
        orc.validate_placement(a, 2)


def test_degenerate_solves_and_param_validation():
    # :153-182
    a, r = pl.solve_local_search(np.zeros((1, 2, 2), np.int64), 2)
    assert r.objective == 0.0
    a, r = pl.solve_local_search(np.array([[[3, 1], [2, 4]]], np.int64), 1)
    assert r.objective == 0.0 and (a == 0).all()
    assert pl.solve_exact_dp(np.array([[[3, 1], [2, 4]]], np.int64), 1)[1].objective == 0.0
    w = np.array([[[1, 0], [0, 1]]], np.int64)
    with pytest.raises(_capi.ExflowInvalidArgument):
        pl.solve_local_search(w, 2, pl.AnnealParams(restarts=0))
    with pytest.raises(_capi.ExflowInvalidArgument):
        pl.solve_local_search(w, 2, pl.AnnealParams(cooling=0.0))


def test_staged_one_node_equals_single_level(orc):
    # :184-196
    c = _random_counts(orc, 8, 3, 150, 11)
    a1, r1 = pl.solve_staged(c, Topology(1, 4), pl.AnnealParams(seed=13))
    a2, r2 = pl.solve_exact_dp(c, 4)
    assert r1.objective == r2.objective and (a1 == a2).all()


def test_staged_planted_two_nodes(orc):
    # :198-216 and the diagonal chain case :218-229
    c = orc.count_transitions(orc.generate_markov_trace(8, 3, 3000, 1.0, 2, 21), 8)[0]
    a, r = pl.solve_staged(c, Topology(2, 2), pl.AnnealParams(seed=3))
    assert r.inter_node_crossings == 0.0
    w = np.zeros((2, 8, 8), np.int64)
    for m in w:
        np.fill_diagonal(m, 5)
    a, r = pl.solve_staged(w, Topology(2, 2))
    assert r.inter_node_crossings == 0.0 and r.intra_node_crossings == 0.0 and r.objective == 0.0


def _permuted_planted(orc, E, L, T, alpha, groups, seed, perm_seed):
    # acceptance.cpp:71-78
    paths = orc.generate_markov_trace(E, L, T, alpha, groups, seed)
    perm = list(range(E))
    orc.Rng(perm_seed).shuffle(perm)
    return orc.permute_experts(paths, E, np.array(perm, np.int32))


def test_acceptance_planted_recovery(orc):
    # acceptance.cpp:239-269 (criterion 6)
    paths = _permuted_planted(orc, 32, 12, 50000, 1.0, 8, 42, 4242)
    c = orc.count_transitions(paths, 32)[0]
    a, r = pl.solve_staged(c, Topology(2, 4), pl.AnnealParams(seed=7))
    assert r.objective == 0.0
    homes = a[0][paths[:, 0]]
    rep = orc.simulate(paths, a, 2, 4, orc.COHERENT, homes=homes)
    assert abs(rep.locality_gpu - orc.expected_planted_locality(1.0, 8)) <= 0.01


def test_acceptance_locality_gain_single_node(orc):
    # acceptance.cpp:276-309 (criterion 7) on the single-node 8-GPU box: the
    # GPU-level locality gain over contiguous placement must be >= 2x.
    for seed in range(3):
        paths = _permuted_planted(orc, 32, 8, 20000, 0.8, 8, 500 + seed, 9000 + seed)
        c = orc.count_transitions(paths, 32)[0]
        a, _ = pl.solve_staged(c, Topology(1, 8), pl.AnnealParams(seed=seed))
        aff = orc.simulate(paths, a, 1, 8, orc.COHERENT)
        base = orc.simulate(paths, orc.contiguous_placement(32, 8, 8), 1, 8, orc.COHERENT)
        assert aff.locality_gpu >= 2.0 * base.locality_gpu
        assert aff.p_star < base.p_star


def test_contiguous_random_json_roundtrip(orc):
    topo = Topology(1, 4)
    a = pl.contiguous_placement(8, 3, topo)
    assert (a == orc.contiguous_placement(8, 3, 4)).all()
    r = pl.random_placement(8, 4, Topology(2, 2), 77)
    assert (r == orc.random_placement(8, 4, 4, 77)).all()  # same xoshiro draw order
    back, t2 = pl.placement_from_json(pl.placement_to_json(r, Topology(2, 2)))
    assert (back == r).all() and t2.num_nodes == 2
    import os
    fx = os.path.join(os.path.dirname(__file__), "golden", "two_token_demo_placement.json")
    fa, ft = pl.placement_from_json(open(fx).read())
    assert (fa == a).all() and ft.gpus_per_node == 4
    bad = a.copy()
    bad[0, 0] = 3
    with pytest.raises(_capi.ExflowInvalidArgument, match="places"):
        pl.validate_placement(bad, topo)


def test_objective_crossings_matches_oracle(orc):
    c = _random_counts(orc, 8, 3, 200, 55)
    for seed in range(4):
        a = orc.random_placement(8, 3, 4, seed)
        for level, lv in ((pl.GPU, False), (pl.NODE, True)):
            assert pl.objective_crossings(c, a, Topology(2, 2), level) == \
                orc.objective_crossings(c, a, gpus_per_node=2, level_node=lv)


def test_synth_host_matches_oracle(orc):
    a = pl.generate_markov_trace(8, 4, 256, 0.8, 4, 42)
    assert (a == orc.generate_markov_trace(8, 4, 256, 0.8, 4, 42)).all()
    b = pl.generate_markov_trace(64, 24, 5000, 0.8, 8, 3)
    assert (b == orc.generate_markov_trace(64, 24, 5000, 0.8, 8, 3)).all()


def test_solver_matches_reference_restatement():
    """The redesigned solver (incremental swap ledger, restarts on host
    threads) reproduces, placement for placement, the outputs of a line-by-
    line restatement of proj/src/placement.cpp:87-821 (same xoshiro draw
    order) on 16 seeded histograms: exact DP, annealing (1-4 restarts, default
    and short schedules), one- and two-node staging
    (tests/golden/make_solver_golden.py)."""
    import json
    import os
    g = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "solver_golden.json")))
    assert len(g["cases"]) == 16
    for k, cs in enumerate(g["cases"]):
        counts = np.asarray(cs["counts"], np.int64)
        prm = pl.AnnealParams(restarts=cs["restarts"], max_iters=cs["max_iters"], seed=cs["seed"])
        if cs["method"] == "staged":
            a, r = pl.solve_staged(counts, Topology(cs["nodes"], cs["gpn"]), prm)
        else:
            a, r = pl.solve_local_search(counts, cs["nodes"] * cs["gpn"], prm)
        assert np.array_equal(a, np.asarray(cs["assign"])), f"case {k}: placement differs"
        assert r.objective == cs["objective"] and r.iterations == cs["iterations"], f"case {k}"
