"""Gauss-Seidel per-row cost on a single long chain (1D Poisson: one segment, no
cross-segment dependency) vs a 2D grid: isolates the solver's own row step."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_1610_03154_b200.api as api
from paper_1610_03154_b200.types import CandidateSet
from tests.helpers import poisson1d, aniso2d
ctx = api.Context(0)
for name, A in (("1d-200k", poisson1d(200000)), ("2d-512", aniso2d(512, 0.1))):
    B = CandidateSet(A.n_rows, 1, np.ones(A.n_rows))
    for sweeps in (1, 4):
        api.improve_candidates(A, B, sweeps, 1, 0.0, ctx=ctx)
        ctx.set_profiling(True)
        api.improve_candidates(A, B, sweeps, 1, 0.0, ctx=ctx)
        ms = ctx.profile()["gauss_seidel_wavefront"][1]
        ctx.set_profiling(False)
        print(f"{name} n {A.n_rows} sweeps {sweeps}: {ms:.3f} ms = {ms * 1e6 / (A.n_rows * sweeps):.1f} ns/row-sweep", flush=True)
