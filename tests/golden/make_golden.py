"""Generate golden fixtures from the REFERENCE implementation itself.

Runs oracle/_ref/libamgref.so (the unmodified reference headers under
/root/reference/proj/include compiled against oracle/eigen_shim) on small
seeded problems and stores every hierarchy array and the solve history in
tests/golden/*.npz.  tests/test_oracle_pin.py checks the CPU restatement
(oracle/rnamg_port.cpp) and tests/test_gpu_*.py check the GPU path against
these files, so the pin survives on machines without /root/reference.

Usage: python tests/golden/make_golden.py   (needs oracle/_ref built)
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

from oracle.pyoracle import Oracle  # noqa: E402
from tests.golden_cases import CASES  # noqa: E402


def dump(name, A, B, Bh, b, so, vo, ref):
    h = ref.setup(A, B, so, Bh)
    out = {"A_ro": A.row_offsets, "A_ci": A.col_indices, "A_va": A.values, "A_bs": np.array([A.block_size]),
           "B": B.data, "B_k": np.array([B.k]), "b": b, "levels": np.array([h.n_levels()]),
           "stagnated": np.array([int(h.stagnated)]), "ledger": h.ledger()}
    if Bh is not None:
        out["Bh"] = Bh.data
    for l in range(h.n_levels()):
        mats = [(0, "A")] + ([(1, "P"), (2, "R")] if l + 1 < h.n_levels() else [])
        for which, tag in mats:
            M = h.matrix(l, which)
            out[f"L{l}_{tag}_ro"] = M.row_offsets
            out[f"L{l}_{tag}_ci"] = M.col_indices
            out[f"L{l}_{tag}_va"] = M.values
            out[f"L{l}_{tag}_shape"] = np.array([M.n_rows, M.n_cols, M.block_size])
        out[f"L{l}_B"] = h.candidates(l, 0).data
        if l + 1 < h.n_levels():
            out[f"L{l}_Bc"] = h.candidates(l, 1).data
            out[f"L{l}_w"] = np.array(h.relax_weights(l))
        out[f"L{l}_sym"] = np.array([int(h.symmetric(l))])
    x, rep = ref.solve(h, b, None, vo)
    out["x"] = x
    out["hist"] = np.array(rep.residual_history)
    out["its"] = np.array([rep.iterations, int(rep.converged), int(rep.diverged)])
    out["complexity"] = np.array([rep.chi_oc, rep.chi_cc, rep.work_units_solve, rep.work_units_setup])
    np.savez_compressed(os.path.join(HERE, f"{name}.npz"), **out)
    print(name, "levels", h.n_levels(), "its", rep.iterations)


def main():
    ref = Oracle("ref")
    for name, make in CASES.items():
        A, B, Bh, b, so, vo = make()
        dump(name, A, B, Bh, b, so, vo, ref)


if __name__ == "__main__":
    main()
