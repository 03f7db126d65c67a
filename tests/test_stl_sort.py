"""The device replica of libstdc++'s std::sort (csrc/stl_sort.cuh) orders ties exactly
as std::sort does (ensure_min_support's unstable magnitude sort, interpolation.hpp:631-632):
tests/cpp/stl_sort_check.cpp compares the permutations on 5400 tie-heavy arrays."""
import os
import subprocess

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_stl_sort_replica_matches_std_sort(tmp_path):
    exe = str(tmp_path / "stl_sort_check")
    subprocess.run(["g++", "-O2", "-std=c++20", "-I", os.path.join(ROOT, "paper_1610_03154_b200", "csrc"),
                    os.path.join(ROOT, "tests", "cpp", "stl_sort_check.cpp"), "-o", exe], check=True)
    r = subprocess.run([exe], capture_output=True, text=True, timeout=120)
    bad, total = (int(v) for v in r.stdout.split())
    assert total == 5400 and bad == 0
