"""Timeline of the wavefront Gauss-Seidel kernel: runs improve_candidates on a
BASELINE config's finest matrix with AMGCU_GS_TRACE set and summarises the
per-(sweep, 32-row block) globaltimer stamps: phase-A and phase-B durations,
the per-segment start lag and the sweep span."""
import argparse
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=2)
ap.add_argument("--size", type=int, default=1024)
ap.add_argument("--sweeps", type=int, default=4)
ap.add_argument("--out", default="gpurun_out/gs_trace.bin")
ap.add_argument("--level", type=int, default=0, help="relax the hierarchy's level-L matrix (setup first)")
ap.add_argument("--p1d", type=int, default=0, help="relax a 1D Poisson chain of this length instead")
a = ap.parse_args()
if os.path.exists(a.out):
    os.remove(a.out)
os.environ["AMGCU_GS_TRACE"] = a.out
import paper_1610_03154_b200.api as api  # noqa: E402

A, B, Bh, b = api.generate_config(a.config, a.size)
ctx = api.Context(0)
if a.p1d:
    from tests.helpers import poisson1d
    A = poisson1d(a.p1d)
    B = api.CandidateSet(A.n_rows, 1, np.ones(A.n_rows))
if a.level > 0:
    os.environ.pop("AMGCU_GS_TRACE")
    so, _ = api.config_options(a.config)
    h = api.setup(A, B, so, Bh, ctx=ctx)
    A = h.matrix(a.level, 0)
    B = api.CandidateSet(A.n_rows, 1, np.ones(A.n_rows))
    os.environ["AMGCU_GS_TRACE"] = a.out
rl = np.diff(A.row_offsets)
print(f"rows {A.n_rows} nnz/row mean {rl.mean():.1f} max {rl.max()} >16: {(rl > 16).mean() * 100:.1f}%")
api.improve_candidates(A, B, a.sweeps, 1, 0.0, ctx=ctx)  # warm
os.remove(a.out)
api.improve_candidates(A, B, a.sweeps, 1, 0.0, ctx=ctx)
raw = open(a.out, "rb").read()
n, nsw, nf = np.frombuffer(raw[:12], np.int32)
segs = np.frombuffer(raw[12:12 + 4 * (nf + 1)], np.int32)
tr = np.frombuffer(raw[12 + 4 * (nf + 1):], np.uint64).reshape(nsw, n, 4).astype(np.int64)
t0 = tr[tr > 0].min()
print(f"n {n} sweeps {nsw} segments {nf} (mean len {n / nf:.1f})")
allb = tr[:, :, 2][tr[:, :, 0] > 0]
print(f"launch span {(allb.max() - t0) / 1e3:.1f} us (first block start to last block end, all sweeps)")
for s in range(nsw):
    m = tr[s, :, 0] > 0
    blk = tr[s][m] - t0
    pa = blk[:, 1] - blk[:, 0]
    pb = blk[:, 2] - blk[:, 1]
    starts = tr[s, segs[:-1], 0] - t0
    ends = np.array([tr[s, max(segs[g], segs[g + 1] - 1) // 32 * 32 if False else 0, 2] for g in range(0)])
    seg_end = []
    for g in range(nf):
        q0, q1 = segs[g], segs[g + 1]
        last = q0 + ((q1 - 1 - q0) // 32) * 32
        seg_end.append(tr[s, last, 2] - t0)
    seg_end = np.array(seg_end)
    busy = seg_end - starts
    print(f"sweep {s}: span {(blk[:, 2].max() - blk[:, 0].min()) / 1e3:.1f} us  blocks {m.sum()}  "
          f"phaseA med {np.median(pa):.0f} ns p90 {np.percentile(pa, 90):.0f}  phaseB med {np.median(pb):.0f} ns "
          f"p90 {np.percentile(pb, 90):.0f}  seg start lag med {np.median(np.diff(starts)):.0f} ns  "
          f"seg end lag med {np.median(np.diff(seg_end)):.0f} ns  seg busy med {np.median(busy) / 1e3:.1f} us")
    if s == 0 and nf > 3:
        # row publish times: wait on the previous segment vs the own chain
        pub = tr[s, :, 3] - t0
        g = nf // 2
        q0, q1 = segs[g], segs[g + 1]
        L = q1 - q0
        p0 = pub[segs[g - 1]:segs[g - 1] + L]
        p1 = pub[q0:q1]
        d_chain = np.diff(p1)
        d_dep = p1[:-1] - p0[1:] if len(p0) == L else np.zeros(1)
        print(f"  row step (own chain) med {np.median(d_chain):.0f} ns p10 {np.percentile(d_chain, 10):.0f} "
              f"p90 {np.percentile(d_chain, 90):.0f}; row - prev-seg row+1 med {np.median(d_dep):.0f} ns "
              f"p10 {np.percentile(d_dep, 10):.0f} p90 {np.percentile(d_dep, 90):.0f}")
        print("  first 40 row steps:", d_chain[:40].tolist())
        print("  dep lags 40..80:", d_dep[40:80].tolist())
        g = nf // 2
        q0, q1 = segs[g], segs[g + 1]
        rows = tr[s, q0:q1:32] - t0
    if s == 0:
        g = nf // 2
        q0, q1 = segs[g], segs[g + 1]
        rows = tr[s, q0:q1:32] - t0
        wa = (rows[:, 1] - rows[:, 0]) / 1e3
        pb = (rows[:, 2] - rows[:, 1]) / 1e3
        print(f"  segment {g}: {len(rows)} blocks; wait-for-records med {np.median(wa):.2f} us, serial phase med {np.median(pb):.2f} us")
        print("  mid segment blocks (A start, A dur, B dur) us:",
              [(round(r[0] / 1e3, 1), round((r[1] - r[0]) / 1e3, 2), round((r[2] - r[1]) / 1e3, 2)) for r in rows[:8]])
