"""One warm-up and one measured RN-AMG setup + solve of a BASELINE config on
cuda:0 through the C ABI (the bench step without the harness) -- the command
profiled by ncu for the launch list and the per-kernel captures."""
import argparse
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import paper_1610_03154_b200.api as api  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=2)
ap.add_argument("--size", type=int, default=1024)
ap.add_argument("--reps", type=int, default=2)
ap.add_argument("--max-restarts", type=int, default=20)
ap.add_argument("--no-cand-overlap", action="store_true")
a = ap.parse_args()
A, B, Bh, b = api.generate_config(a.config, a.size)
so, vo = api.config_options(a.config)
ctx = api.Context(0)
if a.no_cand_overlap:
    ctx.set_candidate_overlap(False)
for r in range(a.reps):
    t0 = time.perf_counter()
    h = api.setup(A, B, so, Bh, ctx=ctx)
    ctx.synchronize()
    ts = time.perf_counter() - t0
    x, rep = api.solve(h, b, None, vo)
    restarts = 0
    while vo.method == 2 and not rep.converged and not rep.diverged and restarts < a.max_restarts:
        x, rep = api.solve(h, b, x, vo)
        restarts += 1
    print(f"rep {r}: levels {h.n_levels()} its {rep.iterations} conv {rep.converged} "
          f"wall {time.perf_counter() - t0:.3f}s (setup {ts:.3f}s) launches {ctx.launch_count()}", flush=True)
    del h
