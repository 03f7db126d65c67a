"""Gauss-Seidel device time per hierarchy level (improve_candidates with the
config's sweeps on each level's A, profiled by the library's CUDA events)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_1610_03154_b200.api as api
from paper_1610_03154_b200.types import CandidateSet
cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 2
size = int(sys.argv[2]) if len(sys.argv) > 2 else 1024
A, B, Bh, b = api.generate_config(cfg, size)
so, vo = api.config_options(cfg)
ctx = api.Context(0)
h = api.setup(A, B, so, Bh, ctx=ctx)
for l in range(h.n_levels() - 1):
    M = h.matrix(l, 0)
    k = h.candidates(l, 0).k
    Bl = CandidateSet(M.n_rows, k, np.ones(M.n_rows * k))
    api.improve_candidates(M, Bl, so.candidate_sweeps, 1, 0.0, ctx=ctx)
    ctx.set_profiling(True)
    api.improve_candidates(M, Bl, so.candidate_sweeps, 1, 0.0, ctx=ctx)
    ms = ctx.profile()["gauss_seidel_wavefront"][1]
    ctx.set_profiling(False)
    rl = np.diff(M.row_offsets)
    bw = int(np.max(np.abs(M.col_indices - np.repeat(np.arange(M.n_rows), rl)))) if M.nnz() else 0
    print(f"L{l} k {k} n {M.n_rows} bs {M.block_size} longest row {int(rl.max())} bandwidth {bw}: {ms:.3f} ms", flush=True)
