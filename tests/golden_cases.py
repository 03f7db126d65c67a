"""Small seeded cases shared by the golden-fixture generator and the tests.
Every case returns (A, B, Bhat, b, SetupOptions, SolveOptions)."""
import numpy as np

from paper_1610_03154_b200.types import (FilterRule, RelaxConfig, RelaxScheme, SetupOptions, SolveMethod,
                                         SolveOptions, StrengthConfig, StrengthMeasure, constant_candidates)
from tests.helpers import aniso2d, poisson1d


def _config(cfg, size, max_size):
    import paper_1610_03154_b200.api as api  # host-only calls (generator, options): no GPU needed
    A, B, Bh, b = api.generate_config(cfg, size)
    so, vo = api.config_options(cfg)
    so.max_size = max_size
    return A, B, Bh, b, so, vo


def _rhs(n, seed):
    return np.random.default_rng(seed).uniform(-1.0, 1.0, n)


def c1_poisson():
    return _config(1, 24, 30)


def c2_rotated():
    return _config(2, 25, 40)


def c3_recirc():
    return _config(3, 24, 40)


def c4_transport():
    return _config(4, 24, 40)


def c5_elasticity():
    return _config(5, 10, 40)


def default_aniso():
    """reference defaults (evolution SOC, symmetric Gauss-Seidel smoothing), stationary V(1,1)"""
    A = aniso2d(12, 0.1)
    return A, constant_candidates(A.n_rows), None, _rhs(A.n_rows, 3), SetupOptions(max_size=10), SolveOptions()


def line8():
    """test_hierarchy.cpp:13-34 line options"""
    A = poisson1d(8)
    so = SetupOptions(strength=StrengthConfig(StrengthMeasure.symmetric, 0.0), max_size=2)
    return A, constant_candidates(8), None, _rhs(8, 5), so, SolveOptions()


def jacobi_pcg_aniso():
    A = aniso2d(20, 0.05)
    jac = RelaxConfig(RelaxScheme.jacobi, 0.0, 1)
    so = SetupOptions(pre_relax=jac, post_relax=jac, max_size=8)
    return A, constant_candidates(A.n_rows), None, _rhs(A.n_rows, 23), so, SolveOptions(SolveMethod.pcg, tol=1e-10)


def postfilter_aniso():
    """test_hierarchy.cpp:56-78 (post-filter 0.1); oracle pin only (not on the GPU path yet)"""
    A = aniso2d(10, 0.01)
    so = SetupOptions(max_size=8)
    so.interp.postfilter = FilterRule(0.1, None)
    return A, constant_candidates(A.n_rows), None, _rhs(A.n_rows, 11), so, SolveOptions()


CASES = {
    "c1_poisson": c1_poisson, "c2_rotated": c2_rotated, "c3_recirc": c3_recirc, "c4_transport": c4_transport,
    "c5_elasticity": c5_elasticity, "default_aniso": default_aniso, "line8": line8,
    "jacobi_pcg_aniso": jacobi_pcg_aniso, "postfilter_aniso": postfilter_aniso,
}
GPU_CASES = [k for k in CASES if k not in ("postfilter_aniso",)]
