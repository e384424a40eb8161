"""Generates tests/golden/solver_golden.json: placements and objectives of
solve_staged / solve_local_search on seeded random histograms, computed by
the round-1 host solver at commit f4d7c57, which restated
proj/src/placement.cpp:87-821 line by line (same loops, same xoshiro draw
order). The redesigned solver (csrc/host/solver.cpp: incremental swap
ledger, parallel restarts) must reproduce them exactly
(tests/test_placement_solver.py::test_solver_matches_reference_restatement).

Usage (in the build container, needs git + nvcc): python tests/golden/make_solver_golden.py
"""
import ctypes as C
import json
import os
import subprocess
import tempfile

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
COMMIT = "f4d7c57"


class AP(C.Structure):
    _fields_ = [("restarts", C.c_int32), ("max_iters", C.c_int64), ("initial_temperature", C.c_double),
                ("cooling", C.c_double), ("seed", C.c_uint64)]


class SR(C.Structure):
    _fields_ = [("solver", C.c_char * 32), ("objective", C.c_double), ("seed", C.c_uint64),
                ("iterations", C.c_int64), ("restarts", C.c_int32), ("has_optimality_gap", C.c_int32),
                ("optimality_gap", C.c_double), ("has_tiers", C.c_int32),
                ("inter_node_crossings", C.c_double), ("intra_node_crossings", C.c_double),
                ("weighted_cost", C.c_double)]


def build_old(tmp):
    subprocess.run(f"git -C {ROOT} archive {COMMIT} paper_2401_08383_b200/csrc include | tar -x -C {tmp}",
                   shell=True, check=True)
    mk = os.path.join(tmp, "paper_2401_08383_b200", "csrc")
    subprocess.run(["make", "-s", "-j8", "-C", mk, f"ROOT={tmp}", f"OUT={tmp}/libold.so",
                    f"BUILD={tmp}/build"], check=True)
    return C.CDLL(f"{tmp}/libold.so")


def cases():
    rng = np.random.default_rng(2024)
    out = []
    for k in range(16):
        E = [4, 8, 8, 16][k % 4]
        L = int(rng.integers(3, 6))
        gpn = [2, 4, 2, 4][k % 4]
        nodes = 2 if (k % 3 == 0 and E % (2 * gpn) == 0) else 1
        dense = k % 2 == 0
        c = rng.integers(0, 40, (L - 1, E, E)) if dense else \
            (rng.random((L - 1, E, E)) < 0.25) * rng.integers(0, 500, (L - 1, E, E))
        out.append(dict(E=E, L=L, nodes=nodes, gpn=gpn, seed=int(rng.integers(0, 1 << 40)),
                        restarts=int(rng.integers(1, 5)), max_iters=int([0, 800, 2500][k % 3]),
                        counts=c.astype(np.int64).tolist(),
                        method="staged" if k % 4 != 3 else "local_search"))
    return out


def main():
    with tempfile.TemporaryDirectory() as tmp:
        lib = build_old(tmp)
        res = []
        for cs in cases():
            counts = np.ascontiguousarray(cs["counts"], np.int64)
            a = np.zeros((cs["L"], cs["E"]), np.int32)
            r = SR()
            p = AP(cs["restarts"], cs["max_iters"], 0.0, 0.999, cs["seed"])
            if cs["method"] == "staged":
                rc = lib.exf_solve_staged(counts.ctypes.data_as(C.c_void_p), cs["L"], cs["E"], cs["nodes"],
                                          cs["gpn"], C.c_double(1.0), C.c_double(4.0), C.byref(p),
                                          C.c_int64(10000), a.ctypes.data_as(C.c_void_p), C.byref(r))
            else:
                rc = lib.exf_solve_local_search(counts.ctypes.data_as(C.c_void_p), cs["L"], cs["E"],
                                                cs["nodes"] * cs["gpn"], C.byref(p),
                                                a.ctypes.data_as(C.c_void_p), C.byref(r))
            assert rc == 0
            res.append(dict(cs, assign=a.tolist(), objective=r.objective, iterations=r.iterations))
    with open(os.path.join(ROOT, "tests", "golden", "solver_golden.json"), "w") as f:
        json.dump({"generator": f"round-1 restatement of proj/src/placement.cpp at {COMMIT}",
                   "cases": res}, f)


if __name__ == "__main__":
    main()
