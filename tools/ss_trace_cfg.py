"""Exact-order reductions on a config's real solve vectors: setup, then `calls` solves of
`its` iterations each (restarts continue from x) with AMGCU_SS_TRACE=1 set by the caller;
the [seqsum] lines on stderr give the per-phase times, the list lengths and the terms
re-read by the element-by-element path."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1610_03154_b200.api as api
from paper_1610_03154_b200.types import SolveOptions
cfg = int(sys.argv[1]); size = int(sys.argv[2]); its = int(sys.argv[3]) if len(sys.argv) > 3 else 12
calls = int(sys.argv[4]) if len(sys.argv) > 4 else 1
A, B, Bh, b = api.generate_config(cfg, size)
so, vo = api.config_options(cfg)
ctx = api.Context(0)
h = api.setup(A, B, so, Bh, ctx=ctx)
x = None
for cnum in range(calls):
    print(f"=== solve {cnum}", flush=True, file=sys.stderr)
    t0 = time.perf_counter()
    x, rep = api.solve(h, b, x, SolveOptions(vo.method, vo.cycle, vo.tol, its))
    print(cnum, rep.iterations, rep.converged, f"{time.perf_counter() - t0:.3f}s", rep.residual_history[-1], flush=True)
