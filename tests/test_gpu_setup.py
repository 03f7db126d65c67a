"""GPU rn_setup + solve against the CPU oracle on small problems covering every
branch of the path: symmetric SOC + CG (C1-like), evolution SOC + prefilter
(C2-like), nonsymmetric GMRES with separate restriction (C3/C4-like), and
block elasticity with k = 3 > m = 2 (C5-like).

Parity classes: in the sequential-reduction context every
level's A, P, R, B, Bc must be bit-identical; in the default context the
structure (row offsets, column indices, aggregates) must be identical and the
values within 1e-10 relative.  Solve: residual histories within 1e-10
relative (the coarsest solve is a pseudo-inverse product on the GPU and a COD
solve on the CPU), iteration counts equal."""
import numpy as np
import pytest

import paper_1610_03154_b200.api as api
from paper_1610_03154_b200.types import (EvolutionWeighting, FilterRule, KrylovKind, RelaxConfig, RelaxScheme,
                                         SetupOptions,
                                         SolveMethod, SolveOptions, StrengthConfig, StrengthMeasure,
                                         constant_candidates, from_triplets)
from tests.helpers import aniso2d, poisson1d, rel_max_err, same_structure

pytestmark = pytest.mark.gpu

JAC = RelaxConfig(RelaxScheme.jacobi, 0.0, 1)


def _cases():
    cases = []
    # C1-like: 5-point Poisson, symmetric SOC 0.25, degree 2, 4 CG iterations
    cases.append(("poisson", lambda: api.generate_config(1, 24),
                  SetupOptions(strength=StrengthConfig(StrengthMeasure.symmetric, 0.25), pre_relax=JAC, post_relax=JAC,
                               max_size=30), SolveOptions(SolveMethod.pcg)))
    # C2-like: rotated anisotropic Q1, evolution SOC, prefilter 0.1, 6 CG iterations
    so = SetupOptions(pre_relax=JAC, post_relax=JAC, max_size=40)
    so.interp.prefilter = FilterRule(0.1, None)
    so.interp.energy_iters = 6
    cases.append(("rotated", lambda: api.generate_config(2, 25), so, SolveOptions(SolveMethod.pcg)))
    # C3-like: recirculating convection-diffusion, GMRES energy-min, FGMRES
    so = SetupOptions(pre_relax=JAC, post_relax=JAC, max_size=40)
    so.interp.krylov = KrylovKind.gmres
    so.interp.energy_iters = 4
    cases.append(("recirc", lambda: api.generate_config(3, 24), so, SolveOptions(SolveMethod.fgmres, max_iters=30)))
    # C4-like: upwind transport, degree 3, no candidate sweeps
    so = SetupOptions(pre_relax=JAC, post_relax=JAC, max_size=40, candidate_sweeps=0)
    so.interp.krylov = KrylovKind.gmres
    so.interp.degree = 3
    so.interp.energy_iters = 4
    cases.append(("transport", lambda: api.generate_config(4, 24), so, SolveOptions(SolveMethod.fgmres, max_iters=30)))
    # C5-like: Q1 plane strain, k = 3 rigid-body modes, block size 2
    so = SetupOptions(strength=StrengthConfig(StrengthMeasure.symmetric, 0.1), pre_relax=JAC, post_relax=JAC,
                      max_size=40)
    so.interp.energy_iters = 4
    cases.append(("elasticity", lambda: api.generate_config(5, 10), so, SolveOptions(SolveMethod.pcg)))
    return cases


CASES = _cases()


def compare(hg, ho, bitwise):
    assert hg.n_levels() == ho.n_levels()
    assert hg.stagnated == ho.stagnated
    L = hg.n_levels()
    for l in range(L):
        assert hg.symmetric(l) == ho.symmetric(l), l
        for which in ((0, 1, 2) if l < L - 1 else (0,)):
            a, b = hg.matrix(l, which), ho.matrix(l, which)
            assert same_structure(a, b), (l, which)
            if bitwise:
                assert a.values.tobytes() == b.values.tobytes(), (l, which)
            else:
                assert rel_max_err(a.values, b.values) <= 1e-10, (l, which)
        ca, cb = hg.candidates(l, 0), ho.candidates(l, 0)
        if bitwise:
            assert ca.data.tobytes() == cb.data.tobytes(), l
        else:
            assert rel_max_err(ca.data, cb.data) <= 1e-10, l


@pytest.mark.parametrize("name,gen,so,vo", CASES, ids=[c[0] for c in CASES])
def test_setup_bitwise_sequential(gpu_seq, port, name, gen, so, vo):
    A, B, Bh, b = gen()
    hg = api.setup(A, B, so, Bh, ctx=gpu_seq)
    ho = port.setup(A, B, so, Bh)
    compare(hg, ho, bitwise=True)
    for l in range(hg.n_levels() - 1):
        assert hg.relax_weights(l) == ho.relax_weights(l)
    xg, rg = api.solve(hg, b, None, vo)
    xo, ro = port.solve(ho, b, None, vo)
    assert rg.iterations == ro.iterations and rg.converged == ro.converged
    assert rel_max_err(rg.residual_history, ro.residual_history) <= 1e-10
    assert rel_max_err(xg, xo) <= 1e-10
    assert rg.chi_oc == ro.chi_oc and rg.chi_cc == ro.chi_cc


@pytest.mark.parametrize("name,gen,so,vo", CASES, ids=[c[0] for c in CASES])
def test_work_ledger_matches_reference(gpu_seq, port, name, gen, so, vo):
    """WorkLedger (work.hpp:38-67): every bucket's work units equal the reference's, after
    setup (evolution SOC counted on demand) and after a solve"""
    A, B, Bh, b = gen()
    hg = api.setup(A, B, so, Bh, ctx=gpu_seq)
    ho = port.setup(A, B, so, Bh)
    assert hg.ledger().tobytes() == ho.ledger().tobytes(), (hg.ledger(), ho.ledger())
    api.solve(hg, b, None, vo)
    port.solve(ho, b, None, vo)
    assert hg.ledger().tobytes() == ho.ledger().tobytes(), (hg.ledger(), ho.ledger())


def _postfilter_cases():
    cases = []
    so = SetupOptions(pre_relax=JAC, post_relax=JAC, max_size=40)
    so.interp.prefilter = FilterRule(0.1, None)
    so.interp.postfilter = FilterRule(0.1, None)
    so.interp.energy_iters = 6
    cases.append(("rotated-post", lambda: api.generate_config(2, 33), so, SolveOptions(SolveMethod.pcg)))
    so = SetupOptions(strength=StrengthConfig(StrengthMeasure.symmetric, 0.1), pre_relax=JAC, post_relax=JAC,
                      max_size=40)
    so.interp.postfilter = FilterRule(0.2, None)
    so.interp.energy_iters = 4
    cases.append(("elasticity-post", lambda: api.generate_config(5, 12), so, SolveOptions(SolveMethod.pcg)))
    so = SetupOptions(pre_relax=JAC, post_relax=JAC, max_size=40)
    so.interp.krylov = KrylovKind.gmres
    so.interp.energy_iters = 4
    so.interp.postfilter = FilterRule(None, 3)
    cases.append(("recirc-post-k3", lambda: api.generate_config(3, 24), so,
                  SolveOptions(SolveMethod.fgmres, max_iters=30)))
    return cases


@pytest.mark.parametrize("name,gen,so,vo", _postfilter_cases(), ids=[c[0] for c in _postfilter_cases()])
def test_postfilter_bitwise(gpu_seq, port, name, gen, so, vo):
    """post-filter pipeline (interpolation.hpp:648-659): filter, support floor with the
    span-rank test and the reference's std::sort tie order, constraints, one energy-min
    iteration -- every level bitwise, ledger equal"""
    A, B, Bh, b = gen()
    hg = api.setup(A, B, so, Bh, ctx=gpu_seq)
    ho = port.setup(A, B, so, Bh)
    compare(hg, ho, bitwise=True)
    assert hg.ledger().tobytes() == ho.ledger().tobytes()
    xg, rg = api.solve(hg, b, None, vo)
    xo, ro = port.solve(ho, b, None, vo)
    assert rg.iterations == ro.iterations


def test_work_ledger_options(gpu_seq, port):
    """ledger under the other count paths: symmetric SOC, Jacobi candidate improvement
    (its spectral estimate), l1-weighted evolution, degree 1"""
    A = aniso2d(30, 0.05)
    B = constant_candidates(A.n_rows)
    cases = [SetupOptions(strength=StrengthConfig(StrengthMeasure.symmetric, 0.25), pre_relax=JAC, post_relax=JAC,
                          max_size=40),
             SetupOptions(strength=StrengthConfig(StrengthMeasure.evolution, 4.0, 2, EvolutionWeighting.l1jacobi),
                          pre_relax=JAC, post_relax=JAC, max_size=40),
             SetupOptions(candidate_relax=RelaxConfig(RelaxScheme.jacobi, 0.0, 1), pre_relax=JAC, post_relax=JAC,
                          max_size=40)]
    cases[1].interp.degree = 1
    for so in cases:
        hg = api.setup(A, B, so, ctx=gpu_seq)
        ho = port.setup(A, B, so)
        assert hg.ledger().tobytes() == ho.ledger().tobytes(), (so, hg.ledger(), ho.ledger())


@pytest.mark.parametrize("name,gen,so,vo", CASES, ids=[c[0] for c in CASES])
def test_setup_parallel_reductions(gpu_tree, port, name, gen, so, vo):
    A, B, Bh, b = gen()
    hg = api.setup(A, B, so, Bh, ctx=gpu_tree)
    ho = port.setup(A, B, so, Bh)
    compare(hg, ho, bitwise=False)
    xg, rg = api.solve(hg, b, None, vo)
    xo, ro = port.solve(ho, b, None, vo)
    assert rg.iterations == ro.iterations
    assert rel_max_err(rg.residual_history, ro.residual_history) <= 1e-10


def test_line_hierarchy_known_answers(gpu):
    """test_hierarchy.cpp:23-34: 8-point line -> 3 coarse rows, R == P^T, A1 == RAP bitwise"""
    A = poisson1d(8)
    so = SetupOptions(strength=StrengthConfig(StrengthMeasure.symmetric, 0.0), max_size=2)
    h = api.setup(A, constant_candidates(8), so, ctx=gpu)
    assert h.n_levels() >= 2
    assert h.matrix(1, 0).n_rows == 3
    assert h.symmetric(0)
    P, R = h.matrix(0, 1), h.matrix(0, 2)
    assert R == api.transpose(P, ctx=gpu)
    assert h.matrix(1, 0) == api.galerkin_product(R, A, P, ctx=gpu)


def test_solve_zero_rhs(gpu):
    """test_cycle.cpp:44-54"""
    A = poisson1d(16)
    h = api.setup(A, constant_candidates(16), SetupOptions(max_size=4, pre_relax=JAC, post_relax=JAC), ctx=gpu)
    x, rep = api.solve(h, np.zeros(16))
    assert rep.converged and rep.iterations == 0 and not np.any(x)


def test_single_level_direct(gpu):
    """test_cycle.cpp:28-42"""
    A = poisson1d(12)
    h = api.setup(A, constant_candidates(12), SetupOptions(max_size=20), ctx=gpu)
    assert h.n_levels() == 1
    rng = np.random.default_rng(7)
    want = rng.uniform(-1, 1, 12)
    b = api.spmv(A, want, ctx=gpu)
    x, rep = api.solve(h, b)
    assert rep.converged and rep.iterations == 1
    assert np.max(np.abs(x - want)) < 1e-12


def test_stationary_vcycle_contracts(gpu):
    """test_cycle.cpp:75-88 with weighted Jacobi smoothing"""
    A = aniso2d(32, 1.0)
    h = api.setup(A, constant_candidates(A.n_rows), SetupOptions(pre_relax=JAC, post_relax=JAC), ctx=gpu)
    rng = np.random.default_rng(3)
    b = rng.uniform(-1, 1, A.n_rows)
    x, rep = api.solve(h, b, None, SolveOptions(tol=1e-10, max_iters=60))
    assert rep.converged


def test_errors_map_to_reference_exceptions(gpu):
    with pytest.raises(ValueError):
        api.setup(poisson1d(4), constant_candidates(5), SetupOptions(), ctx=gpu)
    from paper_1610_03154_b200.types import from_triplets
    Z = from_triplets(2, 2, [(0, 1, 1.0), (1, 1, 1.0)])
    with pytest.raises(RuntimeError, match="zero diagonal at row 0"):
        api.strength(Z, StrengthConfig(StrengthMeasure.symmetric, 0.1), ctx=gpu)


@pytest.mark.parametrize("config,size", [(2, 96), (5, 48), (4, 64)])
def test_fused_coarse_cycle_matches_per_kernel(gpu, monkeypatch, config, size):
    """The cooperative coarse V-cycle (levels 1.. in one launch) is bit-identical to the
    launch-per-kernel cycle: same x, same residual history."""
    A, B, Bh, b = api.generate_config(config, size)
    so, vo = api.config_options(config)
    h = api.setup(A, B, so, Bh, ctx=gpu)
    assert h.n_levels() >= 3
    x1, r1 = api.solve(h, b, None, vo)
    monkeypatch.setenv("AMGCU_FUSED_CYCLE", "0")
    x0, r0 = api.solve(h, b, None, vo)
    monkeypatch.delenv("AMGCU_FUSED_CYCLE")
    assert r1.iterations == r0.iterations
    assert np.asarray(x1).tobytes() == np.asarray(x0).tobytes()
    assert list(r1.residual_history) == list(r0.residual_history)


GSNE = RelaxConfig(RelaxScheme.gsne, 0.0, 1)
BSGS = RelaxConfig(RelaxScheme.block_sym_gauss_seidel, 0.0, 1)


@pytest.mark.parametrize("scheme", [RelaxScheme.gsne, RelaxScheme.block_sym_gauss_seidel],
                         ids=["gsne", "block_sgs"])
def test_relax_remaining_schemes(gpu_seq, port, scheme):
    """gsne (relaxation.hpp:128-142) and block symmetric Gauss-Seidel (143-167) against
    the reference sweeps, bit for bit: several sweeps, block sizes 1 and 2 (elasticity),
    non-symmetric rows, long rows"""
    rng = np.random.default_rng(53)
    mats = [aniso2d(20, 0.1), api.generate_config(5, 6)[0], api.generate_config(3, 16)[0]]
    for A in mats:
        n = A.n_rows
        b = rng.uniform(-1, 1, n)
        x0 = rng.uniform(-1, 1, n)
        for sweeps in (1, 3):
            got = api.relax(A, int(scheme), 0.0, sweeps, x0, b, ctx=gpu_seq)
            want = port.relax(A, int(scheme), 0.0, sweeps, x0, b)
            assert got.tobytes() == want.tobytes(), (n, A.block_size, sweeps)
        B = api.CandidateSet(n, 2, rng.uniform(0.5, 1.5, 2 * n))
        got = api.improve_candidates(A, B, 2, int(scheme), 0.0, ctx=gpu_seq)
        want = port.improve_candidates(A, B, 2, int(scheme), 0.0)
        assert got.data.tobytes() == want.data.tobytes(), n


@pytest.mark.parametrize("relax", [GSNE, BSGS], ids=["gsne", "block_sgs"])
def test_setup_solve_remaining_schemes(gpu_seq, port, relax):
    """rn_setup + solve with gsne / block symmetric GS as pre-, post- and candidate
    relaxation: hierarchy bitwise (parity mode), ledger equal, solves equal"""
    for gen, vo in ((lambda: api.generate_config(2, 17), SolveOptions(SolveMethod.stationary, max_iters=10)),
                    (lambda: api.generate_config(5, 6), SolveOptions(SolveMethod.fgmres, max_iters=8))):
        A, B, Bh, b = gen()
        so = SetupOptions(pre_relax=relax, post_relax=relax, candidate_relax=RelaxConfig(relax.scheme, 0.0, 1),
                          max_size=30)
        hg = api.setup(A, B, so, Bh, ctx=gpu_seq)
        ho = port.setup(A, B, so, Bh)
        compare(hg, ho, bitwise=True)
        assert hg.ledger().tobytes() == ho.ledger().tobytes()
        xg, rg = api.solve(hg, b, None, vo)
        xo, ro = port.solve(ho, b, None, vo)
        assert rg.iterations == ro.iterations and rg.converged == ro.converged
        assert rel_max_err(rg.residual_history, ro.residual_history) <= 1e-10
        assert rel_max_err(xg, xo) <= 1e-10
        assert hg.ledger().tobytes() == ho.ledger().tobytes()


@pytest.mark.parametrize("cfg,size,max_size", [(2, 96, 1600), (5, 96, 2200), (1, 64, 1000)], ids=["C2-96", "C5-96", "C1-64"])
def test_coarse_gauss_jordan(gpu, port, cfg, size, max_size):
    """coarsest level of 513..4096 rows: inverted by the Gauss-Jordan kernel (the CPU side
    by the reference's COD): hierarchy bitwise, solve to 1e-10 with the same iterations"""
    A, B, Bh, b = api.generate_config(cfg, size)
    so, vo = api.config_options(cfg)
    so.max_size = max_size
    hg = api.setup(A, B, so, Bh, ctx=gpu)
    ho = port.setup(A, B, so, Bh)
    n_coarse = hg.matrix(hg.n_levels() - 1, 0).n_rows
    assert 512 < n_coarse <= 4096, n_coarse
    assert hg.n_levels() == ho.n_levels()
    for l in range(hg.n_levels()):
        assert hg.matrix(l, 0) == ho.matrix(l, 0)
    xg, rg = api.solve(hg, b, None, vo)
    xo, ro = port.solve(ho, b, None, vo)
    assert rg.iterations == ro.iterations and rg.converged == ro.converged
    assert rel_max_err(rg.residual_history, ro.residual_history) <= 1e-10
    assert rel_max_err(xg, xo) <= 1e-10


def test_coarse_gauss_jordan_pivoting(gpu, port):
    """a coarsest operator whose partial pivoting must swap rows (non-symmetric, small
    diagonal): the Gauss-Jordan inverse against the CPU solve, 1e-10"""
    rng = np.random.default_rng(5)
    n = 700
    t = []
    for i in range(n):
        for j in range(max(0, i - 3), min(n, i + 4)):
            v = rng.uniform(-1.0, 1.0)
            if i == j:
                v *= 1e-3
            t.append((i, j, v))
    A = from_triplets(n, n, t)
    so = SetupOptions(max_size=1000)  # one level: the coarsest is A itself
    hg = api.setup(A, constant_candidates(n), so, ctx=gpu)
    ho = port.setup(A, constant_candidates(n), so)
    assert hg.n_levels() == 1
    b = rng.uniform(-1.0, 1.0, n)
    vo = SolveOptions(max_iters=1)
    xg, rg = api.solve(hg, b, None, vo)
    xo, ro = port.solve(ho, b, None, vo)
    assert rel_max_err(xg, xo) <= 1e-10
