"""A few exact-order dots of length n on device-resident operands (the command
profiled by ncu for the seqsum kernel)."""
import ctypes as C
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1610_03154_b200.api as api  # noqa: E402

# bring the SM clock up from idle before timing short kernels (~0.3 s of GEMMs)
_w = torch.randn(4096, 4096, device="cuda")
for _ in range(60):
    _w = (_w @ _w).clamp_(-1, 1)
torch.cuda.synchronize()

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1_046_529
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
ctx = api.Context(0)
x = torch.rand(n, dtype=torch.float64, device="cuda") * 2 - 1
y = torch.rand(n, dtype=torch.float64, device="cuda") * 2 - 1
out = torch.zeros(1, dtype=torch.float64, device="cuda")
for _ in range(reps):
    api.lib.amgcu_dot_device(ctx.handle, C.c_void_p(x.data_ptr()), C.c_void_p(y.data_ptr()), n, 0,
                             C.c_void_p(out.data_ptr()))
ctx.synchronize()
print(n, out.item())
