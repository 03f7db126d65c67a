"""Pin the CPU oracle before trusting it (CPU only).

1. Golden fixtures: outputs of the reference itself (oracle/_ref, the
   unmodified reference headers + Eigen stand-in) stored by
   tests/golden/make_golden.py; the restatement must reproduce every array
   bit for bit.
2. Kernel-by-kernel: restatement vs reference build on seeded random inputs
   (bitwise), when oracle/_ref is available.
"""
import glob
import os

import numpy as np
import pytest

from paper_1610_03154_b200.types import (CandidateSet, SetupOptions, SolveOptions, SparseMatrix, StrengthConfig,
                                         StrengthMeasure, constant_candidates)
from tests.golden_cases import CASES
from tests.helpers import aniso2d, poisson1d, random_sparse, random_spd_sparse, tridiag

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def load_golden(name):
    z = np.load(os.path.join(GOLDEN, f"{name}.npz"))
    A = SparseMatrix(len(z["A_ro"]) - 1, len(z["A_ro"]) - 1, z["A_ro"], z["A_ci"], z["A_va"], int(z["A_bs"][0]))
    k = int(z["B_k"][0])
    B = CandidateSet(A.n_rows, k, z["B"])
    Bh = CandidateSet(A.n_rows, k, z["Bh"]) if "Bh" in z else None
    return z, A, B, Bh, z["b"]


def check_against_golden(z, h, x, rep, values_bitwise=True, tol=1e-10, solve_bitwise=None):
    solve_bitwise = values_bitwise if solve_bitwise is None else solve_bitwise
    assert h.n_levels() == int(z["levels"][0])
    assert int(h.stagnated) == int(z["stagnated"][0])
    for l in range(h.n_levels()):
        mats = [(0, "A")] + ([(1, "P"), (2, "R")] if l + 1 < h.n_levels() else [])
        for which, tag in mats:
            M = h.matrix(l, which)
            assert np.array_equal(M.row_offsets, z[f"L{l}_{tag}_ro"]), (l, tag)
            assert np.array_equal(M.col_indices, z[f"L{l}_{tag}_ci"]), (l, tag)
            want = z[f"L{l}_{tag}_va"]
            if values_bitwise:
                assert M.values.tobytes() == want.tobytes(), (l, tag)
            else:
                assert np.max(np.abs(M.values - want)) <= tol * max(np.max(np.abs(want)), 1e-300), (l, tag)
        got_b = h.candidates(l, 0).data
        if values_bitwise:
            assert got_b.tobytes() == z[f"L{l}_B"].tobytes(), l
        else:
            assert np.max(np.abs(got_b - z[f"L{l}_B"])) <= tol * max(np.max(np.abs(z[f"L{l}_B"])), 1e-300), l
        assert int(h.symmetric(l)) == int(z[f"L{l}_sym"][0])
    hist = np.array(rep.residual_history)
    assert rep.iterations == int(z["its"][0])
    assert int(rep.converged) == int(z["its"][1])
    if solve_bitwise:
        assert hist.tobytes() == z["hist"].tobytes()
        assert x.tobytes() == z["x"].tobytes()
    else:
        assert np.max(np.abs(hist - z["hist"])) <= tol * np.max(np.abs(z["hist"]))
        assert np.max(np.abs(x - z["x"])) <= tol * max(np.max(np.abs(z["x"])), 1e-300)


@pytest.mark.parametrize("name", sorted(CASES))
def test_port_matches_reference_golden(port, name):
    z, A, B, Bh, b = load_golden(name)
    _, _, _, _, so, vo = CASES[name]()
    h = port.setup(A, B, so, Bh)
    assert np.array_equal(h.ledger(), z["ledger"])  # WorkLedger after setup (work.hpp:38-67)
    x, rep = port.solve(h, b, None, vo)
    check_against_golden(z, h, x, rep)
    got_c = np.array([rep.chi_oc, rep.chi_cc, rep.work_units_solve, rep.work_units_setup])
    assert got_c.tobytes() == z["complexity"].tobytes()


def test_golden_inputs_reproducible():
    """the committed inputs are the generator's current output (generator pin)"""
    for name, make in CASES.items():
        z, A, B, Bh, b = load_golden(name)
        A2, B2, Bh2, b2, _, _ = make()
        assert A == A2 and B.data.tobytes() == B2.data.tobytes() and b.tobytes() == b2.tobytes(), name


# ---- restatement vs reference build, kernel by kernel -------------------------------
def test_sparse_kernels_bitwise(port, ref):
    rng = np.random.default_rng(42)
    for _ in range(100):  # test_sparse_core.cpp:70-96 shapes
        n, m, k = (int(v) for v in rng.integers(2, 65, size=3))
        A = random_sparse(n, m, 0.3, rng)
        B = random_sparse(m, k, 0.3, rng)
        x = rng.uniform(-1, 1, m)
        assert port.spmv(A, x).tobytes() == ref.spmv(A, x).tobytes()
        assert port.transpose(A) == ref.transpose(A)
        assert port.matmul(A, B) == ref.matmul(A, B)
        R = random_sparse(k, n, 0.3, rng)
        assert port.galerkin_product(R, A, B) == ref.galerkin_product(R, A, B)
    for _ in range(20):
        G = random_sparse(12, 12, 0.45, rng)
        for theta, kk in [(0.3, 2), (0.0, None), (None, 1), (0.1, None)]:
            assert port.filter_matrix(G, theta, kk) == ref.filter_matrix(G, theta, kk)
        assert port.is_symmetric(G) == ref.is_symmetric(G)


def test_strength_and_aggregation_bitwise(port, ref):
    mats = [poisson1d(16), aniso2d(10, 0.001), aniso2d(9, 1.0), tridiag(12, -1.0, 4.0, -2.0),
            random_spd_sparse(30, 0.2, np.random.default_rng(1))]
    for A in mats:
        for cfg in (StrengthConfig(StrengthMeasure.symmetric, 0.25), StrengthConfig(StrengthMeasure.classical, 0.25),
                    StrengthConfig(StrengthMeasure.evolution, 4.0),
                    StrengthConfig(StrengthMeasure.evolution, 4.0, 2, 1)):
            S1, o1 = port.strength(A, cfg, want_ops=True)
            S2, o2 = ref.strength(A, cfg, want_ops=True)
            assert S1 == S2 and o1 == o2
            N1 = port.normalize_strength(S1)
            assert N1 == ref.normalize_strength(S2)
            a1, a2 = port.greedy_aggregate(N1), ref.greedy_aggregate(N1)
            assert a1[0] == a2[0] and np.array_equal(a1[1], a2[1]) and np.array_equal(a1[2], a2[2])
        assert port.spectral_radius_estimate(A) == ref.spectral_radius_estimate(A)
    R = random_sparse(12, 12, 0.3, np.random.default_rng(29))
    for m in (1, 2, 3):
        assert port.amalgamate(R, m) == ref.amalgamate(R, m)


def test_relaxation_bitwise(port, ref):
    rng = np.random.default_rng(3)
    A = random_spd_sparse(20, 0.25, rng)
    b = rng.uniform(-1, 1, 20)
    x0 = rng.uniform(-1, 1, 20)
    for scheme, w, sw in ((0, 1.0, 3), (1, 0.0, 2), (2, 0.0, 2), (3, 0.0, 2), (0, 0.0, 1)):
        assert port.relax(A, scheme, w, sw, x0, b).tobytes() == ref.relax(A, scheme, w, sw, x0, b).tobytes()
    for A_ in (A, poisson1d(30), aniso2d(8, 0.1)):
        B = constant_candidates(A_.n_rows)
        for scheme, w in ((1, 0.0), (2, 0.0), (0, 0.6), (0, 0.0)):
            assert port.improve_candidates(A_, B, 4, scheme, w).data.tobytes() == \
                ref.improve_candidates(A_, B, 4, scheme, w).data.tobytes()


def test_interpolation_bitwise(port, ref):
    """line fixture (test_interpolation.cpp:37-49) through inject, enforce and energy-min"""
    for n, degree in ((8, 2), (16, 2), (24, 1)):
        A = poisson1d(n)
        S = port.normalize_strength(port.strength(A, StrengthConfig(StrengthMeasure.symmetric, 0.0)))
        na, own, roots = port.greedy_aggregate(S)
        Cm = SparseMatrix(n, na, np.arange(n + 1), own, np.ones(n))
        N = port.root_node_pattern(port.sparsity_pattern(S, Cm, degree), roots)
        assert N == ref.root_node_pattern(ref.sparsity_pattern(S, Cm, degree), roots)
        B = constant_candidates(n)
        T1, Bc1 = port.inject_tentative(own, roots, N, B, 1)
        T2, Bc2 = ref.inject_tentative(own, roots, N, B, 1)
        assert T1 == T2 and Bc1.data.tobytes() == Bc2.data.tobytes()
        for kry, its in ((0, 4), (0, 40), (1, 4)):
            P1 = port.energy_minimize(A, T1, B, Bc1, N, its, kry, roots)
            P2 = ref.energy_minimize(A, T2, B, Bc2, N, its, kry, roots)
            assert P1[0] == P2[0] and P1[1:] == P2[1:]
        E1 = port.enforce_constraints(T1, B, Bc1, N)
        assert E1 == ref.enforce_constraints(T1, B, Bc1, N)
