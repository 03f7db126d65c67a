"""Device time per exact-order dot (csrc/seqsum.cu) against the tree dot, for a range of
lengths, on device-resident operands (CUDA events on the library stream via the
context timer)."""
import ctypes as C
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1610_03154_b200.api as api  # noqa: E402

# bring the SM clock up from idle before timing short kernels (~0.3 s of GEMMs)
_w = torch.randn(4096, 4096, device="cuda")
for _ in range(60):
    _w = (_w @ _w).clamp_(-1, 1)
torch.cuda.synchronize()

lib = api.lib
rows = []
for mode in os.environ.get("SS_MODES", "seq,tree").split(","):
    ctx = api.Context(0, sequential_reductions=(mode == "seq"))
    for n in [int(v) for v in os.environ.get('SS_SIZES', '1000,30000,174421,1046529,4194304,30000000').split(',')]:
        g = torch.Generator(device="cuda").manual_seed(n)
        x = torch.rand(n, dtype=torch.float64, device="cuda", generator=g) * 2 - 1
        y = torch.rand(n, dtype=torch.float64, device="cuda", generator=g) * 2 - 1
        out = torch.zeros(1, dtype=torch.float64, device="cuda")
        for _ in range(3):
            lib.amgcu_dot_device(ctx.handle, C.c_void_p(x.data_ptr()), C.c_void_p(y.data_ptr()), n, 0,
                                 C.c_void_p(out.data_ptr()))
        ctx.synchronize()
        reps = 50 if n <= 4_194_304 else 10
        lib.amgcu_ctx_timer_start(ctx.handle)
        for _ in range(reps):
            lib.amgcu_dot_device(ctx.handle, C.c_void_p(x.data_ptr()), C.c_void_p(y.data_ptr()), n, 0,
                                 C.c_void_p(out.data_ptr()))
        ms = C.c_double()
        lib.amgcu_ctx_timer_stop(ctx.handle, C.byref(ms))
        us = ms.value * 1e3 / reps
        want = float(np.add.accumulate(x.cpu().numpy() * y.cpu().numpy())[-1]) if mode == "seq" else None
        ok = (out.item() == want) if want is not None else None
        rows.append((mode, n, us, 16.0 * n / (us * 1e-6) / 1e9, ok))
        print(f"{mode:5s} n={n:>10d} {us:9.1f} us  {16.0 * n / (us * 1e-6) / 1e9:8.1f} GB/s  bitwise={ok}", flush=True)
    ctx.close()
