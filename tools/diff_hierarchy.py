"""Diagnostic: GPU hierarchy vs the CPU oracle for one config, level by level
(first structural mismatch, max relative value error per array)."""
import argparse
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1610_03154_b200.api as api  # noqa: E402
from oracle.pyoracle import Oracle  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=5)
ap.add_argument("--size", type=int, default=1024)
ap.add_argument("--seq", type=int, default=1)
ap.add_argument("--solve", type=int, default=1)
a = ap.parse_args()
A, B, Bh, b = api.generate_config(a.config, a.size)
so, vo = api.config_options(a.config)
ctx = api.Context(0, sequential_reductions=bool(a.seq))
t = time.perf_counter()
hg = api.setup(A, B, so, Bh, ctx=ctx)
print(f"gpu setup {time.perf_counter() - t:.2f}s levels {hg.n_levels()}", flush=True)
t = time.perf_counter()
ho = Oracle("port").setup(A, B, so, Bh)
print(f"cpu setup {time.perf_counter() - t:.2f}s levels {ho.n_levels()}", flush=True)
for l in range(min(hg.n_levels(), ho.n_levels())):
    last = l + 1 == min(hg.n_levels(), ho.n_levels())
    for which, tag in ((0, "A"), (1, "P"), (2, "R")):
        if which and (l + 1 >= hg.n_levels() or l + 1 >= ho.n_levels()):
            continue
        g, o = hg.matrix(l, which), ho.matrix(l, which)
        same = (g.n_rows == o.n_rows and g.n_cols == o.n_cols and np.array_equal(g.row_offsets, o.row_offsets)
                and np.array_equal(g.col_indices, o.col_indices))
        err = float(np.max(np.abs(g.values - o.values)) / max(np.max(np.abs(o.values)), 1e-300)) if same else None
        bit = same and g.values.tobytes() == o.values.tobytes()
        print(f"L{l} {tag}: shape g{g.n_rows}x{g.n_cols} o{o.n_rows}x{o.n_cols} nnz g{g.nnz()} o{o.nnz()} "
              f"struct={'same' if same else 'DIFF'} bitwise={bit} relerr={err}", flush=True)
        if not same and g.n_rows == o.n_rows:
            d = np.nonzero(np.diff(g.row_offsets) != np.diff(o.row_offsets))[0]
            print(f"   first differing rows: {d[:10]}", flush=True)
    cg, co = hg.candidates(l, 0), ho.candidates(l, 0)
    if cg.data.shape == co.data.shape:
        print(f"L{l} B relerr={np.max(np.abs(cg.data - co.data)) / max(np.max(np.abs(co.data)), 1e-300)} "
              f"bitwise={cg.data.tobytes() == co.data.tobytes()}", flush=True)
    print(f"L{l} symmetric g={hg.symmetric(l)} o={ho.symmetric(l)}")
if a.solve:
    xg, rg = api.solve(hg, b, None, vo)
    xo, ro = Oracle("port").solve(ho, b, None, vo)
    print("its", rg.iterations, ro.iterations, "conv", rg.converged, ro.converged)
