"""The exact-order reduction kernel (csrc/seqsum.cu) through the C ABI (amgcu_dot):
dot and norm2 must equal the reference's sequential loop (sparse.hpp:309-315) bit for
bit, from one term to several groups of tiles (> 2^20 terms), on the sequence kinds
the BLAS-1 of the setup and solve produce and on adversarial ones."""
import numpy as np
import pytest

import paper_1610_03154_b200.api as api

pytestmark = pytest.mark.gpu


def seq(t):
    return float(np.add.accumulate(t)[-1]) if t.size else 0.0


def kinds(n, rng):
    u = rng.uniform(-1.0, 1.0, n)
    x = 1.0 + 0.5 * rng.uniform(-1.0, 1.0, n)
    y = u - (np.dot(x, u) / np.dot(x, x)) * x  # orthogonalised: the sum ends near 0
    z = np.zeros(n)
    z[::2] = u[::2]
    z[1::2] = -u[::2][: n // 2]  # exact cancellations
    lead = u.copy()
    lead[: n // 2] = 0.0  # a long run of zero terms first
    big = u * np.ldexp(1.0, rng.integers(-80, 80, n))
    return {"walk": (u, np.ones(n)), "ortho": (x, y), "square": (u, u), "cancel": (z, np.ones(n)),
            "leading_zeros": (lead, u), "range": (big, u), "const": (np.full(n, 0.1), np.ones(n))}


@pytest.mark.parametrize("n", [0, 1, 2, 17, 4095, 4096, 4097, 100_003, 1_048_576 + 12_345, 3_000_000])
def test_dot_matches_sequential_loop(gpu_seq, n):
    rng = np.random.default_rng(n + 1)
    for name, (a, b) in kinds(n, rng).items():
        got = api.dot(a, b, ctx=gpu_seq)
        want = seq(a * b)
        assert np.float64(got).tobytes() == np.float64(want).tobytes(), (name, n, got, want)
    a = rng.uniform(-1.0, 1.0, n)
    got = api.norm2(a, ctx=gpu_seq)
    want = float(np.sqrt(seq(a * a)))
    assert np.float64(got).tobytes() == np.float64(want).tobytes(), (n, got, want)


def test_dot_specials(gpu_seq):
    t = np.array([1.0, np.inf, -1.0])
    assert np.isinf(api.dot(t, np.ones(3), ctx=gpu_seq))
    t = np.array([1.0, np.nan, 2.0] * 3000)
    assert np.isnan(api.dot(t, np.ones(t.size), ctx=gpu_seq))
    t = np.array([-0.0] * 5000)
    assert np.float64(api.dot(t, np.ones(t.size), ctx=gpu_seq)).tobytes() == np.float64(0.0).tobytes()


def test_dot_repeated_calls_reuse_workspace(gpu_seq):
    """the workspace's tickets and look-back flags are reset by every launch"""
    rng = np.random.default_rng(5)
    for n in (5_000_000, 10, 70_000, 5_000_000, 1):
        a, b = rng.uniform(-1, 1, n), rng.uniform(-1, 1, n)
        assert api.dot(a, b, ctx=gpu_seq) == seq(a * b)
