"""Wall time of one RN-AMG setup + solve (after a warm-up) in both reduction modes:
the reference-exact mode (every global sum in the reference's index order) and the
tree mode -- plus the per-family device time of the exact-mode step."""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import paper_1610_03154_b200.api as api  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=2)
ap.add_argument("--size", type=int, default=0)
ap.add_argument("--modes", default="seq,tree")
ap.add_argument("--reps", type=int, default=2)
ap.add_argument("--max-restarts", type=int, default=3)
a = ap.parse_args()
size = a.size or {1: 256, 2: 1024, 3: 2048, 4: 2048, 5: 1024}[a.config]
A, B, Bh, b = api.generate_config(a.config, size)
so, vo = api.config_options(a.config)
out = {"config": a.config, "size": size}
for mode in a.modes.split(","):
    ctx = api.Context(0, sequential_reductions=(mode == "seq"))
    for r in range(a.reps):
        last = r == a.reps - 1
        if last:
            ctx.set_profiling(True)
        ctx.synchronize()
        t0 = time.perf_counter()
        h = api.setup(A, B, so, Bh, ctx=ctx)
        ctx.synchronize()
        t1 = time.perf_counter()
        x, rep = api.solve(h, b, None, vo)
        its = rep.iterations
        k = 0
        while vo.method == 2 and not rep.converged and not rep.diverged and k < a.max_restarts:
            x, rep = api.solve(h, b, x, vo)
            its += rep.iterations
            k += 1
        ctx.synchronize()
        t2 = time.perf_counter()
        if last:
            prof = ctx.profile()
            ctx.set_profiling(False)
            out[mode] = {"setup_s": t1 - t0, "solve_s": t2 - t1, "levels": h.n_levels(), "iterations": its,
                         "converged": bool(rep.converged),
                         "families_ms": {k_: round(v[1], 3) for k_, v in sorted(prof.items(), key=lambda kv: -kv[1][1])}}
        print(f"{mode} rep {r}: setup {t1 - t0:.3f}s solve {t2 - t1:.3f}s levels {h.n_levels()} its {its}", flush=True)
        del h
    ctx.close()
print(json.dumps(out), flush=True)
