"""The drop-in boundary (CPU): libamgcu.so loads without a GPU and exports every
entry point include/amgcu.h declares; ctypes structs match the header; host-only
entry points (generators, option presets) work; compute calls fail loudly
without a device instead of falling back to the CPU."""
import ctypes as C
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_functions():
    src = open(os.path.join(ROOT, "include", "amgcu.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    names = re.findall(r"\b(amgcu_[a-z0-9_]+)\s*\(", src)
    return sorted(set(names))


def test_library_exports_every_declared_symbol():
    import paper_1610_03154_b200.api as api
    names = declared_functions()
    assert len(names) > 40
    missing = [n for n in names if not hasattr(api.lib, n)]
    assert not missing, missing


def test_struct_layouts_match_header():
    from paper_1610_03154_b200._abi import CsrC, SetupOptionsC, SolveOptionsC, SolveReportC, StrengthConfigC
    # field lists mirror the header declarations one to one
    src = open(os.path.join(ROOT, "include", "amgcu.h")).read()
    for struct, cls in (("amgcu_setup_options", SetupOptionsC), ("amgcu_solve_options", SolveOptionsC),
                        ("amgcu_solve_report", SolveReportC), ("amgcu_strength_config", StrengthConfigC),
                        ("amgcu_csr", CsrC)):
        body = re.search(r"typedef struct \{([^{}]*)\}\s*" + struct + ";", src).group(1)
        body = re.sub(r"/\*.*?\*/", "", body, flags=re.S)
        fields = re.findall(r"\b(\w+)\s*;", body)
        assert fields == [f[0] for f in cls._fields_], struct


def test_generators_and_presets_without_gpu():
    import paper_1610_03154_b200.api as api
    A, B, Bh, b = api.generate_config(1, 8)
    assert A.n_rows == 64 and A.nnz() == 64 * 5 - 4 * 8 and B.k == 1 and Bh is None
    so, vo = api.config_options(5)
    assert so.strength.drop_tol == 0.1 and so.interp.energy_iters == 4 and vo.method == 1
    with pytest.raises(ValueError):
        api.generate_config(9, 8)


def test_compute_fails_loudly_without_device():
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is visible")
    import paper_1610_03154_b200.api as api
    with pytest.raises(RuntimeError, match="no CUDA device"):
        api.Context(0)
