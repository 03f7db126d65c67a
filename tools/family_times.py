"""Per-kernel-family device time of one RN-AMG setup + solve (after one warm-up)
through the library's CUDA-event profiler -- the quick A/B tool for kernel work."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import paper_1610_03154_b200.api as api  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=2)
ap.add_argument("--size", type=int, default=1024)
ap.add_argument("--reps", type=int, default=2)
ap.add_argument("--tag", default="")
a = ap.parse_args()
A, B, Bh, b = api.generate_config(a.config, a.size)
so, vo = api.config_options(a.config)
ctx = api.Context(0)
for r in range(a.reps):
    s0, l0 = ctx.sync_count(), ctx.launch_count()
    ctx.set_profiling(True)
    h = api.setup(A, B, so, Bh, ctx=ctx)
    x, rep = api.solve(h, b, None, vo)
    prof = ctx.profile()
    syncs, launches = ctx.sync_count() - s0, ctx.launch_count() - l0
    ctx.set_profiling(False)
    del h
tot = sum(v[1] for v in prof.values())
fams = " ".join(f"{k}={v[1]:.2f}({v[2] / v[1] / 1e6:.0f}GB/s)" for k, v in sorted(prof.items(), key=lambda kv: -kv[1][1]))
print(f"[{a.tag}] C{a.config}/{a.size} its {rep.iterations} total {tot:.1f} ms syncs {syncs} launches {launches} :: {fams}",
      flush=True)
