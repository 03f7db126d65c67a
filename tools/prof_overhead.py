"""Device time of one C5 setup+solve under different profiling masks and candidate-overlap
settings (does event timing of a family perturb the step?)."""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1610_03154_b200.api as api  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 5
size = int(sys.argv[2]) if len(sys.argv) > 2 else 1024
A, B, Bh, b = api.generate_config(cfg, size)
so, vo = api.config_options(cfg)
lib = api.lib
lib.amgcu_profile_family_name.restype = C.c_char_p
names = [lib.amgcu_profile_family_name(f).decode() for f in range(lib.amgcu_profile_family_count())]
ctx = api.Context(0)


def step():
    lib.amgcu_ctx_timer_start(ctx.handle)
    h = api.setup(A, B, so, Bh, ctx=ctx)
    x, rep = api.solve(h, b, None, vo)
    ms = C.c_double()
    lib.amgcu_ctx_timer_stop(ctx.handle, C.byref(ms))
    del h
    return ms.value


for _ in range(2):
    step()
for overlap in (True, False):
    ctx.set_candidate_overlap(overlap)
    for mask_name in (None, "gauss_seidel_wavefront", "spgemm", "all"):
        if mask_name is None:
            lib.amgcu_ctx_set_profiling(ctx.handle, 0)
        else:
            lib.amgcu_ctx_set_profiling(ctx.handle, 1)
            m = 0xffffffff if mask_name == "all" else (1 << names.index(mask_name))
            lib.amgcu_ctx_set_profile_mask(ctx.handle, C.c_uint32(m))
        t = [step() for _ in range(3)]
        print(f"overlap {overlap} profile {mask_name}: {' '.join(f'{v:.1f}' for v in t)} ms", flush=True)
        lib.amgcu_ctx_profile_reset(ctx.handle)
lib.amgcu_ctx_set_profiling(ctx.handle, 0)
