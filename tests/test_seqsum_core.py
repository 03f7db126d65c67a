"""The exact sequential-order summation core (csrc/seqsum.cuh), emulated on the host
with the kernel's geometry and with small geometries that exercise every merge level,
must reproduce the reference's loop `s = 0.0; for i: s += t[i]` (sparse.hpp:309-313)
bit for bit on adversarial sequences: random walks, monotone sums, orthogonalised
products, exact cancellations, rounding ties, huge dynamic range, signed zeros and
specials, constant terms, and corrupted starting approximations (fallback paths)."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def fuzz_bin(tmp_path_factory):
    out = str(tmp_path_factory.mktemp("ss") / "seqsum_fuzz")
    subprocess.run(["g++", "-O2", "-std=c++20", "-ffp-contract=off", "-o", out,
                    os.path.join(ROOT, "tests", "cpp", "seqsum_fuzz.cpp")], check=True)
    return out


@pytest.mark.parametrize("seed", [1, 7, 2024])
def test_seqsum_emulation_bitwise(fuzz_bin, seed):
    r = subprocess.run([fuzz_bin, "1500", str(seed)], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout + r.stderr
    assert r.stdout.startswith("ok 1500"), r.stdout
