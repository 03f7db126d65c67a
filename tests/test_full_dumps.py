"""The committed full-size oracle dumps (tests/golden/full, written by
tests/golden/make_full_dumps.py): the GPU's config-scale test compares against the
restatement's (port) dumps, and the reference build's dumps pin those at the BASELINE
sizes -- every hierarchy array bit-identical, the same iteration count and residual
history.  CPU only: reads the files, runs nothing."""
import os

import numpy as np
import pytest

from tests.golden.make_full_dumps import FULL, OUT
from tests.helpers import rel_max_err


def _load(name, kind):
    path = os.path.join(OUT, f"{name.lower()}_{kind}.npz")
    return np.load(path) if os.path.exists(path) else None


@pytest.mark.parametrize("name", list(FULL))
def test_port_dump_present(name):
    d = _load(name, "port")
    assert d is not None, f"missing port dump for {name}: run tests/golden/make_full_dumps.py {name}"
    assert len(d["keys"]) == len(d["values"]) > 0
    assert d["hist"].size > 0 and d["x_sample"].size > 0


REF = [n for n in FULL if _load(n, "ref") is not None]


@pytest.mark.parametrize("name", REF)
def test_reference_pins_port_at_full_size(name):
    p, r = _load(name, "port"), _load(name, "ref")
    assert str(p["problem"]) == str(r["problem"])
    assert list(p["levels"]) == list(r["levels"])
    pk = dict(zip(p["keys"].tolist(), p["values"].tolist()))
    rk = dict(zip(r["keys"].tolist(), r["values"].tolist()))
    assert sorted(pk) == sorted(rk)
    bad = [k for k in rk if pk[k] != rk[k]]
    assert not bad, bad[:8]
    assert list(p["its"]) == list(r["its"])
    assert rel_max_err(p["hist"], r["hist"]) <= 1e-10
    assert rel_max_err(p["x_sample"], r["x_sample"]) <= 1e-10
