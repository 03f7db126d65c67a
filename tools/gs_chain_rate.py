"""Row rate of the warp-per-segment Gauss-Seidel kernel without cross-segment waits: one
1-D chain (a single segment, one warp, every value from the ring) of n rows, k columns,
and a 2-D 9-point grid for comparison.  Prints ns per row step."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ["AMGCU_GS_LANES"] = "0"
os.environ["AMGCU_GS_CTA"] = "0"
import numpy as np
import paper_1610_03154_b200.api as api
from paper_1610_03154_b200.types import CandidateSet, SparseMatrix

def chain(n, half_width):
    rows, cols, vals = [], [], []
    idx = np.arange(n)
    offs = list(range(-half_width, half_width + 1))
    ro = [0]
    ci = []; va = []
    for d in offs:
        pass
    # banded matrix, diagonal 2*half_width, off-diagonals -1
    cnt = np.zeros(n, dtype=np.int64)
    cl = []
    for d in offs:
        j = idx + d
        ok = (j >= 0) & (j < n)
        cl.append((idx[ok], j[ok], np.where(d == 0, 2.0 * half_width + 1, -1.0) * np.ones(ok.sum())))
    r = np.concatenate([c[0] for c in cl]); cc = np.concatenate([c[1] for c in cl]); v = np.concatenate([c[2] for c in cl])
    o = np.lexsort((cc, r))
    r, cc, v = r[o], cc[o], v[o]
    rp = np.zeros(n + 1, dtype=np.int32); np.add.at(rp, r + 1, 1); rp = np.cumsum(rp).astype(np.int32)
    return SparseMatrix(n, n, rp, cc.astype(np.int32), v)

ctx = api.Context(0)
for n, hw, k, sweeps in [(100000, 1, 1, 1), (100000, 1, 3, 1), (100000, 4, 1, 1), (100000, 4, 3, 1), (100000, 9, 3, 1), (100000, 9, 3, 4)]:
    A = chain(n, hw)
    B = CandidateSet(n, k, np.ones(n * k))
    api.improve_candidates(A, B, sweeps, 1, 0.0, ctx=ctx)
    ctx.set_profiling(True)
    api.improve_candidates(A, B, sweeps, 1, 0.0, ctx=ctx)
    ms = ctx.profile()["gauss_seidel_wavefront"][1]
    ctx.set_profiling(False)
    print(f"chain n {n} entries/row {2 * hw + 1} k {k} sweeps {sweeps}: {ms:.3f} ms, {ms * 1e6 / (n * sweeps):.0f} ns per row step", flush=True)
