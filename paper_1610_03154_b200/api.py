"""Python binding of libamgcu (include/amgcu.h) mirroring the reference API.

Every compute call goes through the C ABI into the sm_100a kernels; there is
no CPU fallback.  If libamgcu.so is missing this module fails to import, and
if no CUDA device is visible the first call raises.
"""
from __future__ import annotations

import ctypes as C
import os
import threading

import numpy as np

from ._abi import (CsrC, SetupOptionsC, SolveOptionsC, SolveReportC, StrengthConfigC, as_f64, as_i32, f64p, i32p,
                   ptr_f64, ptr_i32)
from .types import (CandidateSet, Level, SetupOptions, SolveOptions, SolveReport, SparseMatrix, StrengthConfig,
                    raise_for)

_LIB_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), "_lib", "libamgcu.so")
if not os.path.exists(_LIB_PATH):
    raise ImportError(f"libamgcu.so not built at {_LIB_PATH}; run __graft_entry__.build()")
lib = C.CDLL(_LIB_PATH)

lib.amgcu_last_error.restype = C.c_char_p
lib.amgcu_last_error.argtypes = [C.c_void_p]
for _name in ("amgcu_ctx_create", "amgcu_ctx_destroy", "amgcu_ctx_set_sequential_reductions",
              "amgcu_ctx_set_candidate_overlap", "amgcu_ctx_set_masked_band", "amgcu_ctx_masked_band_stats", "amgcu_ctx_synchronize",
              "amgcu_ctx_launch_count", "amgcu_ctx_sync_count", "amgcu_setup", "amgcu_setup_device", "amgcu_hier_destroy",
              "amgcu_hier_levels", "amgcu_hier_get_matrix", "amgcu_hier_get_candidates", "amgcu_hier_level_symmetric",
              "amgcu_hier_relax_weights", "amgcu_hier_complexity", "amgcu_hier_ledger", "amgcu_solve", "amgcu_solve_device", "amgcu_cycle",
              "amgcu_spmv", "amgcu_transpose", "amgcu_matmul", "amgcu_galerkin_product", "amgcu_filter_matrix",
              "amgcu_is_symmetric", "amgcu_spectral_radius", "amgcu_strength", "amgcu_normalize_strength",
              "amgcu_amalgamate", "amgcu_greedy_aggregate", "amgcu_sparsity_pattern", "amgcu_improve_candidates",
              "amgcu_relax", "amgcu_generate", "amgcu_config_options", "amgcu_dot", "amgcu_dot_device"):
    getattr(lib, _name).restype = C.c_int
lib.amgcu_ctx_create.argtypes = [C.c_int, C.POINTER(C.c_void_p)]
lib.amgcu_ctx_destroy.argtypes = [C.c_void_p]
lib.amgcu_ctx_set_sequential_reductions.argtypes = [C.c_void_p, C.c_int]
lib.amgcu_ctx_set_candidate_overlap.argtypes = [C.c_void_p, C.c_int]
lib.amgcu_ctx_set_masked_band.argtypes = [C.c_void_p, C.c_int32]
lib.amgcu_ctx_masked_band_stats.argtypes = [C.c_void_p, C.POINTER(C.c_int64), C.POINTER(C.c_int64), C.POINTER(C.c_int32)]
lib.amgcu_ctx_synchronize.argtypes = [C.c_void_p]
lib.amgcu_ctx_launch_count.argtypes = [C.c_void_p, C.POINTER(C.c_int64)]
lib.amgcu_ctx_sync_count.argtypes = [C.c_void_p, C.POINTER(C.c_int64)]
lib.amgcu_setup.argtypes = [C.c_void_p, C.POINTER(CsrC), C.c_int32, f64p, f64p, C.POINTER(SetupOptionsC),
                            C.POINTER(C.c_void_p)]
lib.amgcu_setup_device.argtypes = [C.c_void_p, C.POINTER(CsrC), C.c_int32, C.c_void_p, C.c_void_p,
                                   C.POINTER(SetupOptionsC), C.POINTER(C.c_void_p)]
lib.amgcu_hier_destroy.argtypes = [C.c_void_p]
lib.amgcu_hier_levels.argtypes = [C.c_void_p, C.POINTER(C.c_int32), C.POINTER(C.c_int32)]
lib.amgcu_hier_get_matrix.argtypes = [C.c_void_p, C.c_int32, C.c_int32, C.POINTER(CsrC)]
lib.amgcu_hier_get_candidates.argtypes = [C.c_void_p, C.c_int32, C.c_int32, C.POINTER(C.c_int32),
                                          C.POINTER(C.c_int32), C.POINTER(f64p)]
lib.amgcu_hier_level_symmetric.argtypes = [C.c_void_p, C.c_int32, C.POINTER(C.c_int32)]
lib.amgcu_hier_relax_weights.argtypes = [C.c_void_p, C.c_int32, C.POINTER(C.c_double), C.POINTER(C.c_double)]
lib.amgcu_hier_complexity.argtypes = [C.c_void_p, C.POINTER(C.c_double), C.POINTER(C.c_double)]
lib.amgcu_hier_ledger.argtypes = [C.c_void_p, f64p]
lib.amgcu_solve.argtypes = [C.c_void_p, f64p, f64p, C.POINTER(SolveOptionsC), C.POINTER(SolveReportC), f64p, C.c_int32]
lib.amgcu_solve_device.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.POINTER(SolveOptionsC),
                                   C.POINTER(SolveReportC), f64p, C.c_int32]
lib.amgcu_cycle.argtypes = [C.c_void_p, f64p, f64p, C.c_int32]
lib.amgcu_spmv.argtypes = [C.c_void_p, C.POINTER(CsrC), f64p, f64p]
lib.amgcu_dot.argtypes = [C.c_void_p, f64p, f64p, C.c_int64, C.c_int32, C.POINTER(C.c_double)]
lib.amgcu_dot_device.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int64, C.c_int32, C.c_void_p]
lib.amgcu_transpose.argtypes = [C.c_void_p, C.POINTER(CsrC), C.POINTER(CsrC)]
lib.amgcu_matmul.argtypes = [C.c_void_p, C.POINTER(CsrC), C.POINTER(CsrC), C.POINTER(CsrC)]
lib.amgcu_galerkin_product.argtypes = [C.c_void_p, C.POINTER(CsrC), C.POINTER(CsrC), C.POINTER(CsrC), C.POINTER(CsrC)]
lib.amgcu_filter_matrix.argtypes = [C.c_void_p, C.POINTER(CsrC), C.c_int32, C.c_double, C.c_int32, C.POINTER(CsrC)]
lib.amgcu_is_symmetric.argtypes = [C.c_void_p, C.POINTER(CsrC), C.c_double, C.POINTER(C.c_int32)]
lib.amgcu_spectral_radius.argtypes = [C.c_void_p, C.POINTER(CsrC), C.c_int32, C.POINTER(C.c_double)]
lib.amgcu_strength.argtypes = [C.c_void_p, C.POINTER(CsrC), C.POINTER(StrengthConfigC), C.POINTER(CsrC)]
lib.amgcu_normalize_strength.argtypes = [C.c_void_p, C.POINTER(CsrC), C.POINTER(CsrC)]
lib.amgcu_amalgamate.argtypes = [C.c_void_p, C.POINTER(CsrC), C.c_int32, C.POINTER(CsrC)]
lib.amgcu_greedy_aggregate.argtypes = [C.c_void_p, C.POINTER(CsrC), C.POINTER(C.c_int32), i32p, i32p]
lib.amgcu_sparsity_pattern.argtypes = [C.c_void_p, C.POINTER(CsrC), C.POINTER(CsrC), C.c_int32, C.POINTER(CsrC)]
lib.amgcu_improve_candidates.argtypes = [C.c_void_p, C.POINTER(CsrC), C.c_int32, f64p, C.c_int32, C.c_int32,
                                         C.c_double, f64p]
lib.amgcu_relax.argtypes = [C.c_void_p, C.POINTER(CsrC), C.c_int32, C.c_double, C.c_int32, f64p, f64p]
lib.amgcu_generate.argtypes = [C.c_int32, C.c_int32, C.POINTER(CsrC), C.POINTER(C.c_int32), C.POINTER(f64p),
                               C.POINTER(C.c_int32), C.POINTER(f64p), C.POINTER(f64p)]
lib.amgcu_config_options.argtypes = [C.c_int32, C.POINTER(SetupOptionsC), C.POINTER(SolveOptionsC)]
lib.amgcu_default_setup_options.argtypes = [C.POINTER(SetupOptionsC)]
lib.amgcu_default_solve_options.argtypes = [C.POINTER(SolveOptionsC)]
lib.amgcu_free.argtypes = [C.c_void_p]
lib.amgcu_csr_free.argtypes = [C.POINTER(CsrC)]


class Context:
    """One CUDA device + stream.  sequential_reductions=True (the default) takes every
    global sum in the reference's left-to-right order, bit for bit (csrc/seqsum.cu);
    False selects deterministic tree reductions (reproducible, not the reference's bits)."""

    def __init__(self, device: int = 0, sequential_reductions: bool = True):
        h = C.c_void_p()
        code = lib.amgcu_ctx_create(device, C.byref(h))
        if code != 0:
            raise_for(code if code in (1, 2, 3) else 2, lib.amgcu_last_error(None).decode())
        self.handle = h.value
        self.set_sequential_reductions(sequential_reductions)

    def close(self):
        if getattr(self, "handle", None):
            lib.amgcu_ctx_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def set_sequential_reductions(self, on: bool):
        self._chk(lib.amgcu_ctx_set_sequential_reductions(self.handle, 1 if on else 0))

    def set_candidate_overlap(self, on: bool):
        """forward-GS candidate improvement on a second stream beside the aggregation (default on)"""
        self._chk(lib.amgcu_ctx_set_candidate_overlap(self.handle, 1 if on else 0))

    def set_masked_band(self, min_rows: int):
        """levels of at least min_rows rows run the band-staged (TMA) masked product; < 0: never"""
        self._chk(lib.amgcu_ctx_set_masked_band(self.handle, int(min_rows)))

    def masked_band_stats(self):
        """(plans accepted, plans refused, reason bits of the last refusal)"""
        a, r, f = C.c_int64(0), C.c_int64(0), C.c_int32(0)
        self._chk(lib.amgcu_ctx_masked_band_stats(self.handle, C.byref(a), C.byref(r), C.byref(f)))
        return a.value, r.value, f.value

    def synchronize(self):
        self._chk(lib.amgcu_ctx_synchronize(self.handle))

    def sync_count(self) -> int:
        v = C.c_int64()
        self._chk(lib.amgcu_ctx_sync_count(self.handle, C.byref(v)))
        return v.value

    def launch_count(self) -> int:
        v = C.c_int64()
        self._chk(lib.amgcu_ctx_launch_count(self.handle, C.byref(v)))
        return v.value

    def set_profiling(self, on: bool, mask: int = 0xFFFFFFFF):
        """Per-kernel-family CUDA-event timing (two events per launch of a masked family)."""
        self._chk(lib.amgcu_ctx_set_profiling(self.handle, 1 if on else 0))
        self._chk(lib.amgcu_ctx_set_profile_mask(self.handle, C.c_uint32(mask)))
        if on:
            self._chk(lib.amgcu_ctx_profile_reset(self.handle))

    def profile(self) -> dict:
        """{family: (launches, ms, algorithmic_bytes)} since the last reset."""
        lib.amgcu_profile_family_name.restype = C.c_char_p
        out = {}
        for f in range(lib.amgcu_profile_family_count()):
            n, ms, by = C.c_int64(), C.c_double(), C.c_double()
            self._chk(lib.amgcu_ctx_profile_query(self.handle, f, C.byref(n), C.byref(ms), C.byref(by)))
            if n.value:
                out[lib.amgcu_profile_family_name(f).decode()] = (n.value, ms.value, by.value)
        return out

    def _chk(self, code):
        if code != 0:
            raise_for(code if code in (1, 2, 3) else 2, lib.amgcu_last_error(self.handle).decode())

    def _csr(self, fn, *args):
        out = CsrC()
        self._chk(fn(self.handle, *args, C.byref(out)))
        m = SparseMatrix.from_c(out)
        lib.amgcu_csr_free(C.byref(out))
        return m


_default = None
_default_lock = threading.Lock()


def default_context() -> Context:
    global _default
    with _default_lock:
        if _default is None:
            _default = Context(0)
        return _default


def _ctx(ctx):
    return ctx if ctx is not None else default_context()


class Hierarchy:
    """Device-resident hierarchy (hierarchy.hpp:80-91).  Level data stays in
    HBM; `levels` downloads host mirrors on demand."""

    def __init__(self, ctx: Context, handle):
        self.ctx = ctx
        self.handle = handle

    def __del__(self):
        try:
            if self.handle:
                lib.amgcu_hier_destroy(self.handle)
                self.handle = None
        except Exception:
            pass

    def n_levels(self) -> int:
        n, s = C.c_int32(), C.c_int32()
        self.ctx._chk(lib.amgcu_hier_levels(self.handle, C.byref(n), C.byref(s)))
        return n.value

    @property
    def stagnated(self) -> bool:
        n, s = C.c_int32(), C.c_int32()
        self.ctx._chk(lib.amgcu_hier_levels(self.handle, C.byref(n), C.byref(s)))
        return bool(s.value)

    def matrix(self, level: int, which: int) -> SparseMatrix:
        out = CsrC()
        self.ctx._chk(lib.amgcu_hier_get_matrix(self.handle, level, which, C.byref(out)))
        m = SparseMatrix.from_c(out)
        lib.amgcu_csr_free(C.byref(out))
        return m

    def candidates(self, level: int, which: int) -> CandidateSet:
        n, k, d = C.c_int32(), C.c_int32(), f64p()
        self.ctx._chk(lib.amgcu_hier_get_candidates(self.handle, level, which, C.byref(n), C.byref(k), C.byref(d)))
        arr = np.ctypeslib.as_array(d, shape=(max(1, n.value * k.value),))[:n.value * k.value].copy()
        lib.amgcu_free(d)
        return CandidateSet(n.value, k.value, arr)

    def symmetric(self, level: int) -> bool:
        s = C.c_int32()
        self.ctx._chk(lib.amgcu_hier_level_symmetric(self.handle, level, C.byref(s)))
        return bool(s.value)

    def relax_weights(self, level: int):
        a, b = C.c_double(), C.c_double()
        self.ctx._chk(lib.amgcu_hier_relax_weights(self.handle, level, C.byref(a), C.byref(b)))
        return a.value, b.value

    def ledger(self) -> np.ndarray:
        """WorkLedger work units {aggregation, candidates, interpolation, RAP, solve}."""
        out = np.zeros(5)
        self.ctx._chk(lib.amgcu_hier_ledger(self.handle, ptr_f64(out)))
        return out

    def setup_report(self) -> dict:
        """The reference's setup_report (complexity.hpp:39-66) as a dict."""
        L = self.n_levels()
        levels = []
        for l in range(L):
            A = self.matrix(l, 0)
            row = {"level": l, "rows": A.n_rows, "nnz": A.nnz(),
                   "nnz_per_row": A.nnz() / A.n_rows if A.n_rows else 0.0, "symmetric": self.symmetric(l)}
            if l + 1 < L:
                row["nnz_P"] = self.matrix(l, 1).nnz()
                row["nnz_R"] = self.matrix(l, 2).nnz()
            levels.append(row)
        oc, cc = self.complexity()
        w = self.ledger()
        return {"levels": levels, "operator_complexity": oc, "cycle_complexity": cc,
                "work_units": {"aggregation": w[0], "candidates": w[1], "interp": w[2], "rap": w[3],
                               "solve_other": w[4], "setup_total": w[0] + w[1] + w[2] + w[3]}}

    def complexity(self):
        a, b = C.c_double(), C.c_double()
        self.ctx._chk(lib.amgcu_hier_complexity(self.handle, C.byref(a), C.byref(b)))
        return a.value, b.value

    @property
    def levels(self):
        out = []
        L = self.n_levels()
        for l in range(L):
            last = l == L - 1
            out.append(Level(self.matrix(l, 0), None if last else self.matrix(l, 1),
                             None if last else self.matrix(l, 2), self.candidates(l, 0),
                             None if last else self.candidates(l, 1), self.symmetric(l)))
        return out

    def finest(self):
        return self.matrix(0, 0)


# ---- the drop-in path ----------------------------------------------------------------------
def setup(A: SparseMatrix, B: CandidateSet, opts: SetupOptions = None, left: CandidateSet = None,
          ctx: Context = None) -> Hierarchy:
    """amg::setup / amg::rn_setup (hierarchy.hpp:252-287, 551-559) on the GPU."""
    ctx = _ctx(ctx)
    opts = opts or SetupOptions()
    if B.n != A.n_rows:
        raise ValueError("rn_setup: candidate size mismatch")
    if left is not None and (left.n != B.n or left.k != B.k):
        raise ValueError("rn_setup: left candidate shape mismatch")
    h = C.c_void_p()
    o = opts.to_c()
    ctx._chk(lib.amgcu_setup(ctx.handle, C.byref(A.to_c()), B.k, ptr_f64(B.data),
                             ptr_f64(left.data) if left is not None else None, C.byref(o), C.byref(h)))
    return Hierarchy(ctx, h.value)


rn_setup = setup


def solve(h: Hierarchy, b, x=None, opts: SolveOptions = None, history_cap: int = 100000):
    """amg::solve (cycle.hpp:114-271).  Returns (x, SolveReport)."""
    b = as_f64(b)
    n = b.shape[0]
    if x is None or len(x) == 0:
        x = np.zeros(n)
    else:
        x = as_f64(x).copy()
        if x.shape[0] != n:
            raise ValueError("solve: guess size mismatch")
    opts = opts or SolveOptions()
    rep = SolveReportC()
    hist = np.zeros(history_cap)
    o = opts.to_c()
    h.ctx._chk(lib.amgcu_solve(h.handle, ptr_f64(b), ptr_f64(x), C.byref(o), C.byref(rep), ptr_f64(hist),
                               history_cap))
    return x, SolveReport.from_c(rep, hist)


def cycle(h: Hierarchy, x, b, kind=0):
    """amg::cycle (cycle.hpp:100-107); returns the updated x."""
    x = as_f64(x).copy()
    b = as_f64(b)
    h.ctx._chk(lib.amgcu_cycle(h.handle, ptr_f64(x), ptr_f64(b), int(kind)))
    return x


# ---- kernel-level functions (one reference routine each) ----------------------------------
def spmv(A: SparseMatrix, x, ctx=None):
    ctx = _ctx(ctx)
    x = as_f64(x)
    y = np.zeros(A.n_rows)
    ctx._chk(lib.amgcu_spmv(ctx.handle, C.byref(A.to_c()), ptr_f64(x), ptr_f64(y)))
    return y


def dot(x, y, ctx=None):
    """sparse.hpp:309-313: sum of x[i] * y[i] from 0.0, left to right"""
    ctx = _ctx(ctx)
    x, y = as_f64(x), as_f64(y)
    if x.shape != y.shape:
        raise ValueError("dot: size mismatch")
    out = C.c_double()
    ctx._chk(lib.amgcu_dot(ctx.handle, ptr_f64(x), ptr_f64(y), x.size, 0, C.byref(out)))
    return out.value


def norm2(x, ctx=None):
    """sparse.hpp:315: sqrt(dot(x, x))"""
    ctx = _ctx(ctx)
    x = as_f64(x)
    out = C.c_double()
    ctx._chk(lib.amgcu_dot(ctx.handle, ptr_f64(x), ptr_f64(x), x.size, 1, C.byref(out)))
    return out.value


def transpose(A: SparseMatrix, ctx=None):
    return _ctx(ctx)._csr(lib.amgcu_transpose, C.byref(A.to_c()))


def matmul(A: SparseMatrix, B: SparseMatrix, ctx=None):
    return _ctx(ctx)._csr(lib.amgcu_matmul, C.byref(A.to_c()), C.byref(B.to_c()))


def galerkin_product(R, A, P, ctx=None):
    return _ctx(ctx)._csr(lib.amgcu_galerkin_product, C.byref(R.to_c()), C.byref(A.to_c()), C.byref(P.to_c()))


def filter_matrix(G, theta=None, k=None, ctx=None):
    return _ctx(ctx)._csr(lib.amgcu_filter_matrix, C.byref(G.to_c()), 1 if theta is not None else 0,
                          float(theta or 0.0), int(k or 0))


def is_symmetric(A, tol=1e-12, ctx=None):
    ctx = _ctx(ctx)
    s = C.c_int32()
    ctx._chk(lib.amgcu_is_symmetric(ctx.handle, C.byref(A.to_c()), tol, C.byref(s)))
    return bool(s.value)


def spectral_radius_estimate(A, steps=15, ctx=None):
    ctx = _ctx(ctx)
    r = C.c_double()
    ctx._chk(lib.amgcu_spectral_radius(ctx.handle, C.byref(A.to_c()), steps, C.byref(r)))
    return r.value


def strength(A, cfg: StrengthConfig, ctx=None):
    c = cfg.to_c()
    return _ctx(ctx)._csr(lib.amgcu_strength, C.byref(A.to_c()), C.byref(c))


def normalize_strength(S, ctx=None):
    return _ctx(ctx)._csr(lib.amgcu_normalize_strength, C.byref(S.to_c()))


def amalgamate(S, m, ctx=None):
    return _ctx(ctx)._csr(lib.amgcu_amalgamate, C.byref(S.to_c()), int(m))


def greedy_aggregate(S, ctx=None):
    """aggregation.hpp:29-98 -> (n_agg, node_to_agg, roots)"""
    ctx = _ctx(ctx)
    n = S.n_rows
    na = C.c_int32()
    n2a = np.zeros(max(n, 1), np.int32)
    roots = np.zeros(max(n, 1), np.int32)
    ctx._chk(lib.amgcu_greedy_aggregate(ctx.handle, C.byref(S.to_c()), C.byref(na), ptr_i32(n2a), ptr_i32(roots)))
    return na.value, n2a[:n], roots[:na.value]


def sparsity_pattern(S, Cm, degree, ctx=None):
    return _ctx(ctx)._csr(lib.amgcu_sparsity_pattern, C.byref(S.to_c()), C.byref(Cm.to_c()), int(degree))


def improve_candidates(A, B: CandidateSet, sweeps, scheme=1, weight=0.0, ctx=None):
    ctx = _ctx(ctx)
    out = np.zeros(B.n * B.k)
    ctx._chk(lib.amgcu_improve_candidates(ctx.handle, C.byref(A.to_c()), B.k, ptr_f64(B.data), int(sweeps),
                                          int(scheme), float(weight), ptr_f64(out)))
    return CandidateSet(B.n, B.k, out)


def relax(A, scheme, weight, sweeps, x, b, ctx=None):
    ctx = _ctx(ctx)
    x = as_f64(x).copy()
    b = as_f64(b)
    ctx._chk(lib.amgcu_relax(ctx.handle, C.byref(A.to_c()), int(scheme), float(weight), int(sweeps), ptr_f64(x),
                             ptr_f64(b)))
    return x


# ---- harness: BASELINE config generators (host) --------------------------------------------
def generate_config(config: int, n: int):
    """Returns (A, B, Bhat or None, b) for BASELINE config 1..5 at size n."""
    A = CsrC()
    k, hl = C.c_int32(), C.c_int32()
    B, Bh, b = f64p(), f64p(), f64p()
    code = lib.amgcu_generate(config, n, C.byref(A), C.byref(k), C.byref(B), C.byref(hl), C.byref(Bh), C.byref(b))
    if code != 0:
        raise_for(code, lib.amgcu_last_error(None).decode())
    M = SparseMatrix.from_c(A)
    lib.amgcu_csr_free(C.byref(A))
    nn = M.n_rows
    Bd = np.ctypeslib.as_array(B, shape=(nn * k.value,)).copy()
    lib.amgcu_free(B)
    Bhd = None
    if hl.value:
        Bhd = np.ctypeslib.as_array(Bh, shape=(nn * k.value,)).copy()
        lib.amgcu_free(Bh)
    bd = np.ctypeslib.as_array(b, shape=(nn,)).copy()
    lib.amgcu_free(b)
    return M, CandidateSet(nn, k.value, Bd), (CandidateSet(nn, k.value, Bhd) if Bhd is not None else None), bd


def config_options(config: int):
    so, vo = SetupOptionsC(), SolveOptionsC()
    code = lib.amgcu_config_options(config, C.byref(so), C.byref(vo))
    if code != 0:
        raise_for(code, lib.amgcu_last_error(None).decode())
    return SetupOptions.from_c(so), SolveOptions(vo.method, vo.cycle, vo.tol, vo.max_iters)
