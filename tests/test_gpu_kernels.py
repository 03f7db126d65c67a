"""GPU kernel parity: each libamgcu entry point against the CPU oracle on the
same inputs.  Integer structure and every fp64 value must be bit-identical
(the kernels keep the reference's per-entry operation order, --fmad=false);
reductions that the reference takes sequentially are bit-identical in the
sequential-reduction context (gpu_seq) and within 1e-12 otherwise."""
import numpy as np
import pytest

import paper_1610_03154_b200.api as api
from paper_1610_03154_b200.types import (CandidateSet, EvolutionWeighting, StrengthConfig, StrengthMeasure,
                                         constant_candidates,
                                         from_triplets, identity)
from tests.helpers import aniso2d, from_triplets, poisson1d, random_sparse, random_spd_sparse, rel_max_err, stencil9, tridiag

pytestmark = pytest.mark.gpu


def bitwise(a, b):
    return a == b


def test_spmv_bitwise(gpu, port):
    rng = np.random.default_rng(42)
    for _ in range(20):
        n, m = rng.integers(2, 80, size=2)
        A = random_sparse(int(n), int(m), 0.3, rng)
        x = rng.uniform(-1, 1, int(m))
        assert api.spmv(A, x, ctx=gpu).tobytes() == port.spmv(A, x).tobytes()


def test_transpose_bitwise(gpu, port):
    rng = np.random.default_rng(7)
    for _ in range(20):
        n, m = rng.integers(1, 90, size=2)
        A = random_sparse(int(n), int(m), 0.25, rng)
        assert bitwise(api.transpose(A, ctx=gpu), port.transpose(A))
    assert api.transpose(identity(4), ctx=gpu) == identity(4)


def test_matmul_bitwise_random(gpu, port):
    """test_sparse_core.cpp:70-96 shapes (100 random instances)"""
    rng = np.random.default_rng(42)
    for _ in range(100):
        n, m, k = (int(v) for v in rng.integers(2, 65, size=3))
        A = random_sparse(n, m, 0.3, rng)
        B = random_sparse(m, k, 0.3, rng)
        assert api.matmul(A, B, ctx=gpu) == port.matmul(A, B)
        R = random_sparse(k, n, 0.3, rng)
        assert api.galerkin_product(R, A, B, ctx=gpu) == port.galerkin_product(R, A, B)


def test_matmul_long_rows_and_cancellation(gpu, port):
    """rows above the shared-memory capacity and exact-zero drops (sparse.hpp:208)"""
    rng = np.random.default_rng(3)
    A = random_sparse(30, 400, 0.9, rng)
    B = random_sparse(400, 300, 0.5, rng)
    assert api.matmul(A, B, ctx=gpu) == port.matmul(A, B)
    # 512..2048 products per row (one warp per block, shared-memory hash), mixed with
    # shorter and longer rows
    for da, db in ((0.1, 0.2), (0.05, 0.5), (0.3, 0.1)):
        A = random_sparse(60, 200, da, rng)
        B = random_sparse(200, 300, db, rng)
        assert api.matmul(A, B, ctx=gpu) == port.matmul(A, B), (da, db)
    # more distinct columns than the shared-memory table of the block kernel holds:
    # those rows take the table in global scratch
    A = random_sparse(3, 1500, 0.9, rng)
    ii, jj = np.nonzero(rng.random((1500, 8000)) < 0.02)
    B = from_triplets(1500, 8000, list(zip(ii.tolist(), jj.tolist(), rng.uniform(0.5, 1.0, ii.size).tolist())))
    assert api.matmul(A, B, ctx=gpu) == port.matmul(A, B)
    # exact cancellation: (1, -1) . (x, x) = 0 is dropped
    A2 = from_triplets(2, 2, [(0, 0, 1.0), (0, 1, -1.0), (1, 1, 2.0)])
    B2 = from_triplets(2, 1, [(0, 0, 3.0), (1, 0, 3.0)])
    C = api.matmul(A2, B2, ctx=gpu)
    assert C == port.matmul(A2, B2)
    assert C.nnz() == 1


def test_matmul_hash_rows_collisions(gpu, port):
    """65..512 products per row (the hash-accumulation kernel): many products per output
    column and small-integer values, so exact cancellations to 0.0 are frequent"""
    rng = np.random.default_rng(11)
    for n, m, k, da, db in ((50, 40, 20, 0.5, 0.5), (20, 60, 8, 0.9, 0.9), (40, 30, 200, 0.6, 0.4)):
        ta, tb = [], []
        for i in range(n):
            for j in range(m):
                if rng.random() < da:
                    ta.append((i, j, float(rng.choice([-2.0, -1.0, 1.0, 2.0]))))
        for i in range(m):
            for j in range(k):
                if rng.random() < db:
                    tb.append((i, j, float(rng.choice([-1.0, 0.5, 1.0, 3.0]))))
        A, B = from_triplets(n, m, ta), from_triplets(m, k, tb)
        assert api.matmul(A, B, ctx=gpu) == port.matmul(A, B), (n, m, k)


def test_filter_matrix(gpu, port):
    rng = np.random.default_rng(17)
    for _ in range(20):
        G = random_sparse(12, 12, 0.45, rng)
        for theta, k in [(0.3, 2), (0.0, None), (None, 1), (0.1, None), (None, 3)]:
            assert api.filter_matrix(G, theta, k, ctx=gpu) == port.filter_matrix(G, theta, k)
        R = random_sparse(9, 5, 0.6, rng)
        assert api.filter_matrix(R, 0.4, 2, ctx=gpu) == port.filter_matrix(R, 0.4, 2)


def test_is_symmetric(gpu, port):
    rng = np.random.default_rng(5)
    A = random_spd_sparse(24, 0.3, rng)
    assert api.is_symmetric(A, ctx=gpu) and port.is_symmetric(A)
    B = random_sparse(20, 20, 0.3, rng)
    assert api.is_symmetric(B, ctx=gpu) == port.is_symmetric(B)
    U = from_triplets(3, 3, [(0, 0, 1.0), (0, 1, 1e-20), (1, 1, 1.0), (2, 2, 1.0)])
    assert api.is_symmetric(U, ctx=gpu) == port.is_symmetric(U)


def test_spectral_radius(gpu_seq, gpu_tree, port):
    for A in (poisson1d(32), aniso2d(12, 0.1), aniso2d(20, 1.0), aniso2d(300, 0.01)):
        want = port.spectral_radius_estimate(A)
        assert api.spectral_radius_estimate(A, ctx=gpu_seq) == want
        assert abs(api.spectral_radius_estimate(A, ctx=gpu_tree) - want) <= 1e-12 * want


def test_spectral_radius_cooperative_matches_steps(gpu_tree, monkeypatch):
    """The one-launch cooperative Arnoldi reproduces the launch-per-step path bit for bit
    (same reduction trees), at sizes that use one and several virtual blocks per block."""
    for A in (poisson1d(5), aniso2d(30, 0.1), aniso2d(150, 1.0), aniso2d(800, 0.01)):
        coop = api.spectral_radius_estimate(A, ctx=gpu_tree)
        monkeypatch.setenv("AMGCU_ARNOLDI_STEPS", "1")
        steps = api.spectral_radius_estimate(A, ctx=gpu_tree)
        monkeypatch.delenv("AMGCU_ARNOLDI_STEPS")
        assert coop == steps, (A.n_rows, coop, steps)


@pytest.mark.parametrize("measure,tol", [(StrengthMeasure.symmetric, 0.25), (StrengthMeasure.symmetric, 0.0),
                                         (StrengthMeasure.classical, 0.25), (StrengthMeasure.evolution, 4.0)])
def test_strength(gpu_seq, port, measure, tol):
    for A in (poisson1d(16), aniso2d(10, 0.001), aniso2d(9, 1.0), tridiag(12, -1.0, 4.0, -2.0)):
        cfg = StrengthConfig(measure, tol)
        S = api.strength(A, cfg, ctx=gpu_seq)
        assert S == port.strength(A, cfg)
        N = api.normalize_strength(S, ctx=gpu_seq)
        assert N == port.normalize_strength(S)
        n, own, roots = api.greedy_aggregate(N, ctx=gpu_seq)
        n2, own2, roots2 = port.greedy_aggregate(N)
        assert n == n2 and np.array_equal(own, own2) and np.array_equal(roots, roots2)


def _dense(D):
    return from_triplets(D.shape[0], D.shape[1],
                         [(i, j, float(D[i, j])) for i in range(D.shape[0]) for j in range(D.shape[1]) if D[i, j] != 0.0])


def _evolution_cases(rng):
    cases = []
    # non-symmetric pattern with a full diagonal
    R = random_sparse(60, 60, 0.08, rng)
    D = R.to_dense() + np.diag(rng.uniform(2.0, 3.0, 60))
    cases.append(_dense(D))
    # one-sided (upwind, lower bidiagonal) operator: mass lands on column neighbours only
    U = np.diag(np.full(40, 2.0)) + np.diag(np.full(39, -1.0), -1)
    cases.append(_dense(U))
    # a dense row and column (> 64 entries: the generic neighbourhood kernel)
    n = 90
    H = np.diag(np.full(n, 4.0)) + np.diag(np.full(n - 1, -1.0), 1) + np.diag(np.full(n - 1, -1.0), -1)
    H[0, :] = -0.5
    H[:, 0] = -0.25
    H[0, 0] = 50.0
    cases.append(_dense(H))
    # a row without a stored diagonal
    M = aniso2d(6, 0.5).to_dense()
    M[7, 7] = 0.0
    cases.append(_dense(M))
    return cases


@pytest.mark.parametrize("steps", [1, 2, 3])
@pytest.mark.parametrize("weighting", [EvolutionWeighting.spectral, EvolutionWeighting.l1jacobi])
def test_evolution_variants(gpu_seq, port, steps, weighting):
    """Evolution SOC on patterns the structured configs do not exercise: non-symmetric,
    one-sided, rows beyond the two-step kernel's capacity, a missing diagonal."""
    rng = np.random.default_rng(41)
    for A in _evolution_cases(rng):
        cfg = StrengthConfig(StrengthMeasure.evolution, 4.0, steps, weighting)
        try:
            want = port.strength(A, cfg)
        except RuntimeError as e:  # zero diagonal under spectral weighting
            with pytest.raises(RuntimeError, match=str(e).split(" at row")[0]):
                api.strength(A, cfg, ctx=gpu_seq)
            continue
        assert api.strength(A, cfg, ctx=gpu_seq) == want, (A.n_rows, steps, weighting)


def test_amalgamate(gpu, port):
    rng = np.random.default_rng(29)
    R = random_sparse(12, 12, 0.3, rng)
    for m in (1, 2, 3):
        assert api.amalgamate(R, m, ctx=gpu) == port.amalgamate(R, m)
    # node rows on both sides of the warp kernel's shared-memory capacity (640 entries),
    # with explicit zeros (blocks whose max |s| is 0 are dropped)
    t = [(i, j, 0.0 if rng.uniform() < 0.2 else rng.uniform(-1.0, 1.0))
         for i in range(240) for j in range(480) if rng.uniform() < (0.75 if i < 40 else 0.08)]
    t.append((239, 479, 0.0))
    Z = from_triplets(240, 480, t)
    for m in (2, 3, 4):
        assert api.amalgamate(Z, m, ctx=gpu) == port.amalgamate(Z, m), m


def test_aggregation_known_answers(gpu):
    """test_aggregation.cpp:18-49"""
    def path(n):
        return api.normalize_strength(api.strength(poisson1d(n), StrengthConfig(StrengthMeasure.symmetric, 0.0),
                                                   ctx=gpu), ctx=gpu)
    n, own, roots = api.greedy_aggregate(path(8), ctx=gpu)
    assert n == 3 and list(roots) == [0, 3, 6] and list(own) == [0, 0, 1, 1, 1, 2, 2, 2]
    n, own, roots = api.greedy_aggregate(path(5), ctx=gpu)
    assert n == 2 and list(roots) == [0, 3] and list(own) == [0, 0, 1, 1, 1]
    n, own, roots = api.greedy_aggregate(identity(5), ctx=gpu)
    assert n == 5 and list(roots) == list(range(5))
    n, own, roots = api.greedy_aggregate(path(3), ctx=gpu)
    assert n == 1 and list(roots) == [0] and list(own) == [0, 0, 0]


def test_aggregation_grids(gpu, port):
    """Pass 1 (the sync-free wavefront) on grids of 20k-36k nodes, with long-range
    couplings and with two-row reach, against the sequential pass."""
    rng = np.random.default_rng(47)
    for A_ in (stencil9(200, 150, rng), stencil9(300, 120, rng, cross=True, extra=0.02, reach=20000),
               stencil9(130, 260, rng, ry=2, cross=True)):
        R = A_.copy() if hasattr(A_, "copy") else A_
        R.values = np.abs(R.values)
        S = port.normalize_strength(R)
        a = api.greedy_aggregate(S, ctx=gpu)
        b = port.greedy_aggregate(S)
        assert a[0] == b[0] and np.array_equal(a[1], b[1]) and np.array_equal(a[2], b[2]), A_.n_rows


def test_aggregation_random(gpu, port):
    rng = np.random.default_rng(31)
    for _ in range(10):
        R = random_sparse(200, 200, 0.02, rng)
        R.values = np.abs(R.values)
        S = port.normalize_strength(R)
        a = api.greedy_aggregate(S, ctx=gpu)
        b = port.greedy_aggregate(S)
        assert a[0] == b[0] and np.array_equal(a[1], b[1]) and np.array_equal(a[2], b[2])


def test_improve_candidates(gpu_seq, port):
    rng = np.random.default_rng(19)
    A = random_spd_sparse(40, 0.2, rng)
    for A_ in (A, poisson1d(30), aniso2d(8, 0.1)):
        B = constant_candidates(A_.n_rows)
        for scheme, w in ((1, 0.0), (2, 0.0), (0, 0.6), (0, 0.0)):
            got = api.improve_candidates(A_, B, 4, scheme, w, ctx=gpu_seq)
            want = port.improve_candidates(A_, B, 4, scheme, w)
            assert got.data.tobytes() == want.data.tobytes(), (scheme, w)


def wide_stencil(nx, ny, r, rng, interleave=1):
    """(2r+1)^2-point couplings on an nx x ny grid (rows of up to (2r+1)^2 entries),
    diagonally dominant, interleave > 1 repeats every node as that many coupled DOFs"""
    t = []
    m = interleave
    for y in range(ny):
        for x in range(nx):
            for d in range(m):
                row = (y * nx + x) * m + d
                off = 0.0
                for dy in range(-r, r + 1):
                    for dx in range(-r, r + 1):
                        xx, yy = x + dx, y + dy
                        if 0 <= xx < nx and 0 <= yy < ny:
                            for e in range(m):
                                col = (yy * nx + xx) * m + e
                                if col != row:
                                    v = -rng.uniform(0.1, 1.0)
                                    off += -v
                                    t.append((row, col, v))
                t.append((row, row, off + 1.0))
    return from_triplets(nx * ny * m, nx * ny * m, t)


@pytest.mark.parametrize("k", [1, 3])
def test_gauss_seidel_segment_warps(gpu_seq, port, k, monkeypatch):
    """Warp-per-segment kernel: long segments (grid rows) of rows longer than 32 entries
    (7x7 couplings, and 5x5 with 2 interleaved DOFs per node), several sweeps, bitwise
    (the single-CTA kernel, which would take these small cases, is switched off)"""
    monkeypatch.setenv("AMGCU_GS_CTA", "0")
    rng = np.random.default_rng(7)
    for A_ in (wide_stencil(40, 12, 3, rng), wide_stencil(24, 10, 2, rng, interleave=2)):
        assert max(np.diff(A_.row_offsets)) > 32
        B = CandidateSet(A_.n_rows, k, rng.uniform(0.5, 1.5, A_.n_rows * k))
        for sweeps in (1, 4):
            got = api.improve_candidates(A_, B, sweeps, 1, 0.0, ctx=gpu_seq)
            want = port.improve_candidates(A_, B, sweeps, 1, 0.0)
            assert got.data.tobytes() == want.data.tobytes(), (A_.n_rows, k, sweeps)


@pytest.mark.parametrize("k", [1, 3])
def test_gauss_seidel_cta(gpu_seq, port, k):
    """Single-CTA shared-memory kernel (small levels): forward and symmetric sweeps, wide
    rows, interleaved DOFs, bitwise"""
    rng = np.random.default_rng(11)
    for A_ in (wide_stencil(12, 9, 3, rng), wide_stencil(8, 7, 2, rng, interleave=2), random_spd_sparse(40, 0.2, rng)):
        B = CandidateSet(A_.n_rows, k, rng.uniform(0.5, 1.5, A_.n_rows * k))
        for scheme in (1, 2):
            for sweeps in (1, 4):
                got = api.improve_candidates(A_, B, sweeps, scheme, 0.0, ctx=gpu_seq)
                want = port.improve_candidates(A_, B, sweeps, scheme, 0.0)
                assert got.data.tobytes() == want.data.tobytes(), (A_.n_rows, k, scheme, sweeps)


def test_gauss_seidel_long_segments(gpu_seq, port):
    """Segments of many 32-row blocks (the solver / prefetcher / poller hand-offs
    across blocks), forward, symmetric and multi-column sweeps."""
    for A_ in (poisson1d(1000), aniso2d(70, 0.1), aniso2d(33, 1.0)):
        for k in (1, 3):
            rng = np.random.default_rng(k)
            B = CandidateSet(A_.n_rows, k, rng.uniform(0.5, 1.5, A_.n_rows * k))
            for scheme in (1, 2):
                got = api.improve_candidates(A_, B, 3, scheme, 0.0, ctx=gpu_seq)
                want = port.improve_candidates(A_, B, 3, scheme, 0.0)
                assert got.data.tobytes() == want.data.tobytes(), (A_.n_rows, k, scheme)


@pytest.mark.parametrize("lanes", ["1", "0"])
def test_gauss_seidel_lane_segments(gpu_seq, port, monkeypatch, lanes):
    """Lane-per-segment kernel (gs_lanes.cuh) against the reference sweep: 9-point
    grids over several CTAs (cross-CTA poll slots), long-range couplings (sibling
    rings, evicted ring slots, rows past the record), 1..4 sweeps, zero and non-zero
    right-hand sides; lanes=0 runs the same cases through the 3-warp segment kernel."""
    monkeypatch.setenv("AMGCU_GS_LANES", lanes)
    rng = np.random.default_rng(41)
    cases = [stencil9(64, 100, rng), stencil9(200, 40, rng), stencil9(48, 70, rng, cross=True, extra=0.3),
             stencil9(40, 90, rng, cross=True, extra=0.2, reach=300),
             stencil9(40, 90, rng, cross=True, extra=0.5, reach=2000), stencil9(50, 80, rng, ry=2, cross=True),
             stencil9(36, 75, rng, ry=2, cross=True, extra=0.3, reach=200),
             # wide rows (10..21 entries: the T = 20 records, halo of two segments)
             stencil9(50, 80, rng, ry=2), stencil9(36, 110, rng, ry=2, extra=0.2, reach=300),
             stencil9(64, 70, rng, rx=3, ry=1, extra=0.1)]
    for A_ in cases:
        n = A_.n_rows
        for sweeps in (1, 4):
            B = CandidateSet(n, 1, rng.uniform(0.5, 1.5, n))
            got = api.improve_candidates(A_, B, sweeps, 1, 0.0, ctx=gpu_seq)
            want = port.improve_candidates(A_, B, sweeps, 1, 0.0)
            assert got.data.tobytes() == want.data.tobytes(), (n, sweeps)
        b = rng.uniform(-1, 1, n)
        x0 = rng.uniform(-1, 1, n)
        got = api.relax(A_, 1, 0.0, 3, x0, b, ctx=gpu_seq)
        want = port.relax(A_, 1, 0.0, 3, x0, b)
        assert got.tobytes() == want.tobytes(), n
    # interleaved vector unknowns (block size 2, chains of stride 2), three candidate
    # columns relaxed one launch each
    A_, B_, _, _ = api.generate_config(5, 24)
    got = api.improve_candidates(A_, B_, 4, 1, 0.0, ctx=gpu_seq)
    want = port.improve_candidates(A_, B_, 4, 1, 0.0)
    assert got.data.tobytes() == want.data.tobytes()


def test_relax(gpu_seq, port):
    rng = np.random.default_rng(3)
    A = random_spd_sparse(20, 0.25, rng)
    b = rng.uniform(-1, 1, 20)
    x0 = rng.uniform(-1, 1, 20)
    for scheme, w, sw in ((0, 1.0, 3), (1, 0.0, 2), (2, 0.0, 2), (0, 0.0, 1)):
        got = api.relax(A, scheme, w, sw, x0, b, ctx=gpu_seq)
        want = port.relax(A, scheme, w, sw, x0, b)
        assert got.tobytes() == want.tobytes(), (scheme, w, sw)
