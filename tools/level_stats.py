"""Rows, nnz and row-length statistics of A, P, R on every level of a config's hierarchy."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_1610_03154_b200.api as api
cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 2
size = int(sys.argv[2]) if len(sys.argv) > 2 else 1024
A, B, Bh, b = api.generate_config(cfg, size)
so, vo = api.config_options(cfg)
h = api.setup(A, B, so, Bh, ctx=api.Context(0))
for l in range(h.n_levels()):
    for w, name in ((0, "A"), (1, "P"), (2, "R")):
        if w and l == h.n_levels() - 1:
            continue
        M = h.matrix(l, w)
        rl = np.diff(M.row_offsets)
        print(f"L{l} {name}: {M.n_rows:8d} x {M.n_cols:8d} nnz {len(M.col_indices):9d} row len mean {rl.mean():6.1f} "
              f"max {rl.max():5d}")
