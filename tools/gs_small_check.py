"""Small Gauss-Seidel parity check through the C ABI (improve_candidates): quick triage
of the GS kernels on the box.  Usage: gs_small_check.py [case] [scheme] [sweeps]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_1610_03154_b200.api as api
from oracle.pyoracle import Oracle
from paper_1610_03154_b200.types import constant_candidates
from tests.helpers import poisson1d, aniso2d, random_spd_sparse
ctx = api.Context(0)
port = Oracle("port")
rng = np.random.default_rng(19)
cases = {"spd40": random_spd_sparse(40, 0.2, rng), "p1d30": poisson1d(30), "p1d3": poisson1d(3),
         "aniso8": aniso2d(8, 0.1)}
names = [sys.argv[1]] if len(sys.argv) > 1 else list(cases)
schemes = [int(sys.argv[2])] if len(sys.argv) > 2 else [1, 2]
sweeps = int(sys.argv[3]) if len(sys.argv) > 3 else 4
for name in names:
    A_ = cases[name]
    B = constant_candidates(A_.n_rows)
    for scheme in schemes:
        got = api.improve_candidates(A_, B, sweeps, scheme, 0.0, ctx=ctx)
        want = port.improve_candidates(A_, B, sweeps, scheme, 0.0)
        print(name, scheme, sweeps, got.data.tobytes() == want.data.tobytes(), flush=True)
