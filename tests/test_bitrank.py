"""The mask-pair records of the band-staged masked product (csrc/masked_band.cuh): the
match of two sorted column lists is stored as two bit masks, and a slot finds its partner
with a popcount and an n-th-set-bit search (csrc/bitrank.h, shared by the kernels).
tests/cpp/bitrank_check.cpp checks both against plain loops on the host."""
import os
import subprocess

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_bitrank_helpers_match_plain_loops(tmp_path):
    exe = str(tmp_path / "bitrank_check")
    subprocess.run(["g++", "-O2", "-std=c++20", "-I", os.path.join(ROOT, "paper_1610_03154_b200", "csrc"),
                    os.path.join(ROOT, "tests", "cpp", "bitrank_check.cpp"), "-o", exe], check=True)
    r = subprocess.run([exe], capture_output=True, text=True, timeout=120)
    bad, total = (int(v) for v in r.stdout.split())
    assert total > 1000000 and bad == 0
