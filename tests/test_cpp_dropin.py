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
    assert got["levels"] == h.n_levels() and got["iterations"] == rep.iterations
    assert got["nnz_P0"] == h.matrix(0, 1).nnz()
    # the ledger through the drop-in header (setup buckets; the solve bucket after one solve)
    assert got["wu"][:4] == list(h.ledger()[:4])
    # setup_report (complexity.hpp:39-66) through the header: per-level sizes, complexities, work units
    rep_json = json.loads(r.stderr.splitlines()[0])
    oc, cc = h.complexity()
    assert [lv["rows"] for lv in rep_json["levels"]] == [h.matrix(l, 0).n_rows for l in range(h.n_levels())]
    assert rep_json["operator_complexity"] == oc and rep_json["cycle_complexity"] == cc
    assert rep_json["work_units"]["setup_total"] == sum(h.ledger()[:4])
