"""The C++ drop-in header (include/amg_b200.hpp) compiles against the
reference-shaped caller tests/cpp/run_single.cpp and links with libamgcu.so
(CPU); on a GPU the program runs and matches the oracle's iteration count."""
import json
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIBDIR = os.path.join(ROOT, "paper_1610_03154_b200", "_lib")


@pytest.fixture(scope="module")
def binary(tmp_path_factory):
    out = str(tmp_path_factory.mktemp("cpp") / "run_single")
    cmd = ["g++", "-std=c++20", "-O2", "-I", os.path.join(ROOT, "include"), os.path.join(ROOT, "tests", "cpp",
           "run_single.cpp"), "-L", LIBDIR, "-lamgcu", f"-Wl,-rpath,{LIBDIR}", "-o", out]
    r = subprocess.run(cmd, capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    return out


def test_dropin_compiles_and_links(binary):
    assert os.path.exists(binary)


def test_dropin_complexity_on_hand_built_hierarchy(tmp_path):
    """complexity.hpp's measures read only the host mirror (test_complexity.cpp's use)"""
    out = str(tmp_path / "complexity_check")
    cmd = ["g++", "-std=c++20", "-O2", "-I", os.path.join(ROOT, "include"),
           os.path.join(ROOT, "tests", "cpp", "complexity_check.cpp"), "-L", LIBDIR, "-lamgcu",
           f"-Wl,-rpath,{LIBDIR}", "-o", out]
    r = subprocess.run(cmd, capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    got = json.loads(subprocess.run([out], capture_output=True, text=True, check=True).stdout)
    assert got["oc"] == pytest.approx(180 / 120, rel=1e-15)
    assert got["cc"] == pytest.approx((3 * 120 + 90 + 3 * 48 + 30) / 120, rel=1e-15)
    assert got["cc20"] == got["cc"]
    assert got["cc00"] == pytest.approx((120 + 90 + 48 + 30) / 120, rel=1e-15)
    assert got["finest"] == 30 and got["coarsest"] == 4


@pytest.mark.gpu
def test_dropin_runs_like_the_reference_caller(binary, port):
    import paper_1610_03154_b200.api as api
    r = subprocess.run([binary, "2", "65", "report"], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr
    got = json.loads(r.stdout)
    A, B, Bh, b = api.generate_config(2, 65)
    so, vo = api.config_options(2)
    h = port.setup(A, B, so, Bh)
    _, rep = port.solve(h, b, None, vo)
    # run_single's record (amg_main.cpp:249-282) through Hierarchy's fields
    assert got["levels"] == h.n_levels() and got["iterations"] == rep.iterations and got["converged"] == 1
    assert got["nnz_P0"] == h.matrix(0, 1).nnz()
    assert got["coarse_rows"] == h.matrix(h.n_levels() - 1, 0).n_rows
    assert got["wu"][:4] == list(h.ledger()[:4]) and got["sc"] == sum(h.ledger()[:4])
    # acceptance.cpp:107-112 on h.levels: P Bc = B
    assert got["interp_err"] <= 1e-12
    # complexity.hpp from the host mirror, and cycle() counting exactly cycle_complexity
    oc, cc = h.complexity()
    assert got["operator_complexity"] == oc and got["cycle_complexity"] == cc
    assert got["cycle_wu"] == pytest.approx(cc, rel=1e-14)
    assert got["cycle_complexity_2_1"] > cc and got["coeff_ok"] == 1
    # setup_report (complexity.hpp:39-66) through the header: per-level sizes, complexities, work units
    err = r.stderr
    rep_json = json.loads(err[:err.index("level,rows")])
    assert [lv["rows"] for lv in rep_json["levels"]] == [h.matrix(l, 0).n_rows for l in range(h.n_levels())]
    assert rep_json["operator_complexity"] == oc and rep_json["cycle_complexity"] == cc
    assert rep_json["work_units"]["setup_total"] == sum(h.ledger()[:4])
