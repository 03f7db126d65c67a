"""Test fixtures restated from the reference's tests/helpers.hpp:14-62."""
import numpy as np

from paper_1610_03154_b200.types import SparseMatrix, from_triplets


def tridiag(n, lo, di, up):
    t = []
    for i in range(n):
        if i > 0:
            t.append((i, i - 1, lo))
        t.append((i, i, di))
        if i + 1 < n:
            t.append((i, i + 1, up))
    return from_triplets(n, n, t)


def poisson1d(n):
    return tridiag(n, -1.0, 2.0, -1.0)


def aniso2d(n, eps):
    """u_xx + eps u_yy on an n x n interior grid (helpers.hpp:27-40)"""
    t = []
    for j in range(n):
        for i in range(n):
            r = j * n + i
            t.append((r, r, 2.0 + 2.0 * eps))
            if i > 0:
                t.append((r, r - 1, -1.0))
            if i + 1 < n:
                t.append((r, r + 1, -1.0))
            if j > 0:
                t.append((r, r - n, -eps))
            if j + 1 < n:
                t.append((r, r + n, -eps))
    return from_triplets(n * n, n * n, t)


def random_sparse(rows, cols, density, rng):
    """seeded random sparse matrix (numpy generator; shapes as helpers.hpp:42-55)"""
    t = []
    for i in range(rows):
        for j in range(cols):
            if rng.uniform() < density:
                v = rng.uniform(-1.0, 1.0)
                if v == 0.0:
                    v = 0.5
                t.append((i, j, v))
    return from_triplets(rows, cols, t)


def random_spd_sparse(n, density, rng):
    M = random_sparse(n, n, density, rng).to_dense()
    D = M.T @ M + n * 0.5 * np.eye(n)
    t = [(i, j, D[i, j]) for i in range(n) for j in range(n) if D[i, j] != 0.0]
    return from_triplets(n, n, t)


def rel_max_err(got, want):
    got, want = np.asarray(got), np.asarray(want)
    scale = max(np.max(np.abs(want)) if want.size else 0.0, 1e-300)
    return float(np.max(np.abs(got - want)) / scale) if want.size else 0.0


def same_structure(a: SparseMatrix, b: SparseMatrix):
    return (a.n_rows == b.n_rows and a.n_cols == b.n_cols and np.array_equal(a.row_offsets, b.row_offsets)
            and np.array_equal(a.col_indices, b.col_indices))


def stencil9(nx, ny, rng, extra=0.0, reach=None, rx=1, ry=1, cross=False):
    """nx x ny grid, (2 rx + 1) x (2 ry + 1)-point coupling (9-point by default) with
    seeded random off-diagonal values and a dominant diagonal; `extra` = fraction of
    rows given one more coupling to a random row within `reach` (long-range hand-offs
    for the Gauss-Seidel kernels); cross=True keeps only the axis neighbours (5-point)."""
    t = []
    n = nx * ny
    for j in range(ny):
        for i in range(nx):
            r = j * nx + i
            t.append((r, r, 4.0 * (2 * rx + 1) * (2 * ry + 1) + rng.uniform()))
            for dj in range(-ry, ry + 1):
                for di in range(-rx, rx + 1):
                    if cross and di and dj:
                        continue
                    if (di or dj) and 0 <= i + di < nx and 0 <= j + dj < ny:
                        t.append((r, r + dj * nx + di, -rng.uniform(0.1, 1.0)))
    if extra:
        reach = reach or n
        for r in range(n):
            if rng.uniform() < extra:
                c = int(np.clip(r + rng.integers(-reach, reach + 1), 0, n - 1))
                if abs(c - r) > nx + 1:
                    t.append((r, c, -rng.uniform(0.01, 0.1)))
    return from_triplets(n, n, t)
