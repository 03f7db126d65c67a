"""Repeated forward-GS candidate sweeps on a config's fine operator (k candidate columns),
device time per call: checks run-to-run stability of the GS kernels."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_1610_03154_b200.api as api
cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 5
size = int(sys.argv[2]) if len(sys.argv) > 2 else 1024
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 5
A, B, Bh, b = api.generate_config(cfg, size)
so, vo = api.config_options(cfg)
ctx = api.Context(0)
out = []
for r in range(reps):
    ctx.set_profiling(True)
    t0 = time.perf_counter()
    Bo = api.improve_candidates(A, B, so.candidate_sweeps, 1, 0.0, ctx=ctx)
    wall = time.perf_counter() - t0
    ms = ctx.profile()["gauss_seidel_wavefront"][1]
    ctx.set_profiling(False)
    out.append(Bo.data.tobytes())
    print(f"rep {r}: GS {ms:.2f} ms wall {wall*1e3:.1f} ms same_as_first {out[-1] == out[0]}", flush=True)
