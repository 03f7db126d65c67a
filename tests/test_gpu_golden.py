"""GPU path against the reference's own outputs (tests/golden/*.npz, written by
tests/golden/make_golden.py from the unmodified reference build).  In parity mode
(sequential reductions) every level's A / P / R, the candidates and the WorkLedger
are bit-identical to the reference's; the solve takes the same iteration count with
residual history and x within 1e-10 (the coarsest-level pseudo-inverse is
factorised differently), and the complexities (chi_oc, chi_cc, setup work units)
are bit-identical.  Covers the five config families, the defaults, the 8-point line
hierarchy and the post-filter pipeline (interpolation.hpp:648-659)."""
import numpy as np
import pytest

from paper_1610_03154_b200 import api
from tests.golden_cases import CASES
from tests.test_oracle_pin import check_against_golden, load_golden


@pytest.mark.gpu
@pytest.mark.parametrize("name", sorted(CASES))
def test_gpu_matches_reference_golden(gpu_seq, name):
    z, A, B, Bh, b = load_golden(name)
    _, _, _, _, so, vo = CASES[name]()
    h = api.setup(A, B, so, Bh, ctx=gpu_seq)
    assert np.array_equal(h.ledger(), z["ledger"])
    x, rep = api.solve(h, b, None, vo)
    check_against_golden(z, h, x, rep, values_bitwise=True, tol=1e-10, solve_bitwise=False)
    got_c = np.array([rep.chi_oc, rep.chi_cc, rep.work_units_setup])
    assert got_c.tobytes() == z["complexity"][[0, 1, 3]].tobytes()
    # solve-phase work units: same iteration count, same per-cycle count
    assert rep.work_units_solve == z["complexity"][2]
