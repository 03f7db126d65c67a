"""C5 setup, then a few PCG iterations with AMGCU_SS_TRACE=1 set by the caller: the
exact-order reductions' phase times on the solve's real vectors."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1610_03154_b200.api as api
from paper_1610_03154_b200.types import SolveOptions
A, B, Bh, b = api.generate_config(5, int(sys.argv[1]) if len(sys.argv) > 1 else 1024)
so, vo = api.config_options(5)
ctx = api.Context(0)
h = api.setup(A, B, so, Bh, ctx=ctx)
print("=== solve", flush=True)
sys.stderr.flush()
x, rep = api.solve(h, b, None, SolveOptions(vo.method, vo.cycle, vo.tol, 3))
print(rep.iterations, flush=True)
