"""ORACLE TEST INFRASTRUCTURE -- not part of the product.

ctypes wrapper of oracle/oracle_abi.h.  Two implementations share the ABI:
  Oracle("port") -> oracle/build/liboracle_port.so  (own restatement, rnamg_port.cpp)
  Oracle("ref")  -> oracle/_ref/libamgref.so        (reference headers + Eigen stand-in)
Only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline leg use this.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

from paper_1610_03154_b200._abi import (CsrC, SetupOptionsC, SolveOptionsC, SolveReportC, f64p, i32p, as_f64, as_i32,
                                        ptr_f64, ptr_i32)
from paper_1610_03154_b200.types import (CandidateSet, Level, SetupOptions, SolveOptions, SolveReport, SparseMatrix,
                                         StrengthConfig, raise_for)

HERE = os.path.dirname(os.path.abspath(__file__))
LIBS = {
    "port": os.path.join(HERE, "build", "liboracle_port.so"),
    "ref": os.path.join(HERE, "_ref", "libamgref.so"),
}

_cache = {}
GEN_LIB = os.path.join(HERE, "build", "libconfiggen.so")


def _gen():
    if GEN_LIB not in _cache:
        if not os.path.exists(GEN_LIB):
            raise FileNotFoundError(f"{GEN_LIB} not built (run __graft_entry__.build())")
        lib = C.CDLL(GEN_LIB)
        lib.gen_last_error.restype = C.c_char_p
        lib.gen_generate_config.argtypes = [C.c_int32, C.c_int32, C.POINTER(CsrC), C.POINTER(C.c_int32),
                                            C.POINTER(f64p), C.POINTER(C.c_int32), C.POINTER(f64p), C.POINTER(f64p)]
        lib.gen_config_options.argtypes = [C.c_int32, C.POINTER(SetupOptionsC), C.POINTER(SolveOptionsC)]
        lib.gen_free.argtypes = [C.c_void_p]
        _cache[GEN_LIB] = lib
    return _cache[GEN_LIB]


def generate_config(config: int, n: int):
    """BASELINE config `config` at size n from oracle/build/libconfiggen.so (the product's
    generators compiled for the CPU alone): (A, B, Bhat or None, b), the same bytes as
    paper_1610_03154_b200.api.generate_config without loading libamgcu.so."""
    lib = _gen()
    A = CsrC()
    k, hl = C.c_int32(), C.c_int32()
    B, Bh, b = f64p(), f64p(), f64p()
    code = lib.gen_generate_config(config, n, C.byref(A), C.byref(k), C.byref(B), C.byref(hl), C.byref(Bh), C.byref(b))
    if code != 0:
        raise_for(code, lib.gen_last_error().decode())
    M = SparseMatrix.from_c(A)
    for p in (A.row_offsets, A.col_indices, A.values):
        lib.gen_free(C.cast(p, C.c_void_p))
    nn = M.n_rows

    def take(p, count):
        a = np.ctypeslib.as_array(p, shape=(count,)).copy()
        lib.gen_free(C.cast(p, C.c_void_p))
        return a

    Bd = take(B, nn * k.value)
    Bhd = take(Bh, nn * k.value) if hl.value else None
    bd = take(b, nn)
    return M, CandidateSet(nn, k.value, Bd), (CandidateSet(nn, k.value, Bhd) if Bhd is not None else None), bd


def config_options(config: int):
    """(SetupOptions, SolveOptions) of BASELINE config `config` (libconfiggen.so)"""
    so, vo = SetupOptionsC(), SolveOptionsC()
    lib = _gen()
    code = lib.gen_config_options(config, C.byref(so), C.byref(vo))
    if code != 0:
        raise_for(code, lib.gen_last_error().decode())
    return SetupOptions.from_c(so), SolveOptions(vo.method, vo.cycle, vo.tol, vo.max_iters)


def available(kind: str) -> bool:
    return os.path.exists(LIBS[kind])


class Hierarchy:
    def __init__(self, orc, handle):
        self._orc = orc
        self.handle = handle

    def __del__(self):
        try:
            if self.handle:
                self._orc.lib.orc_hier_free(self.handle)
                self.handle = None
        except Exception:
            pass

    def n_levels(self):
        n, s = C.c_int32(), C.c_int32()
        self._orc._chk(self._orc.lib.orc_hier_levels(self.handle, C.byref(n), C.byref(s)))
        return n.value

    @property
    def stagnated(self):
        n, s = C.c_int32(), C.c_int32()
        self._orc._chk(self._orc.lib.orc_hier_levels(self.handle, C.byref(n), C.byref(s)))
        return bool(s.value)

    def matrix(self, level, which):
        return self._orc._csr_call(self._orc.lib.orc_hier_get_matrix, self.handle, level, which)

    def candidates(self, level, which):
        n, k, d = C.c_int32(), C.c_int32(), f64p()
        self._orc._chk(self._orc.lib.orc_hier_get_candidates(self.handle, level, which, C.byref(n), C.byref(k),
                                                             C.byref(d)))
        arr = np.ctypeslib.as_array(d, shape=(max(1, n.value * k.value),))[:n.value * k.value].copy()
        self._orc.lib.orc_free(d)
        return CandidateSet(n.value, k.value, arr)

    def symmetric(self, level):
        s = C.c_int32()
        self._orc._chk(self._orc.lib.orc_hier_level_symmetric(self.handle, level, C.byref(s)))
        return bool(s.value)

    def relax_weights(self, level):
        a, b = C.c_double(), C.c_double()
        self._orc._chk(self._orc.lib.orc_hier_relax_weights(self.handle, level, C.byref(a), C.byref(b)))
        return a.value, b.value

    def ledger(self):
        w = np.zeros(5)
        self._orc._chk(self._orc.lib.orc_hier_ledger(self.handle, ptr_f64(w)))
        return w

    def complexity(self):
        a, b = C.c_double(), C.c_double()
        self._orc._chk(self._orc.lib.orc_hier_complexity(self.handle, C.byref(a), C.byref(b)))
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


class Oracle:
    def __init__(self, kind="port"):
        path = LIBS[kind]
        if not os.path.exists(path):
            raise FileNotFoundError(f"oracle library {path} not built (run __graft_entry__.build())")
        if path not in _cache:
            _cache[path] = C.CDLL(path)
        self.lib = _cache[path]
        self.kind = kind
        lib = self.lib
        lib.orc_last_error.restype = C.c_char_p
        for name in ("orc_hier_levels", "orc_hier_get_matrix", "orc_hier_get_candidates", "orc_hier_level_symmetric",
                     "orc_hier_relax_weights", "orc_hier_ledger", "orc_hier_complexity", "orc_hier_free",
                     "orc_solve", "orc_cycle"):
            getattr(lib, name).argtypes = None
        lib.orc_hier_levels.argtypes = [C.c_void_p, C.POINTER(C.c_int32), C.POINTER(C.c_int32)]
        lib.orc_hier_get_matrix.argtypes = [C.c_void_p, C.c_int32, C.c_int32, C.POINTER(CsrC)]
        lib.orc_hier_get_candidates.argtypes = [C.c_void_p, C.c_int32, C.c_int32, C.POINTER(C.c_int32),
                                                C.POINTER(C.c_int32), C.POINTER(f64p)]
        lib.orc_hier_level_symmetric.argtypes = [C.c_void_p, C.c_int32, C.POINTER(C.c_int32)]
        lib.orc_hier_relax_weights.argtypes = [C.c_void_p, C.c_int32, C.POINTER(C.c_double), C.POINTER(C.c_double)]
        lib.orc_hier_ledger.argtypes = [C.c_void_p, f64p]
        lib.orc_hier_complexity.argtypes = [C.c_void_p, C.POINTER(C.c_double), C.POINTER(C.c_double)]
        lib.orc_hier_free.argtypes = [C.c_void_p]
        lib.orc_solve.argtypes = [C.c_void_p, f64p, f64p, C.c_void_p, C.POINTER(SolveReportC), f64p, C.c_int32]
        lib.orc_cycle.argtypes = [C.c_void_p, f64p, f64p, C.c_int32]

    # -- helpers -----------------------------------------------------------
    def _chk(self, code):
        if code != 0:
            raise_for(code, self.lib.orc_last_error().decode())

    def _csr_call(self, fn, *args):
        out = CsrC()
        self._chk(fn(*args, C.byref(out)))
        m = SparseMatrix.from_c(out)
        self.lib.orc_csr_free(C.byref(out))
        return m

    # -- sparse core ---------------------------------------------------------
    def spmv(self, A: SparseMatrix, x):
        x = as_f64(x)
        y = np.zeros(A.n_rows)
        self._chk(self.lib.orc_spmv(C.byref(A.to_c()), ptr_f64(x), ptr_f64(y)))
        return y

    def transpose(self, A):
        return self._csr_call(self.lib.orc_transpose, C.byref(A.to_c()))

    def matmul(self, A, B, want_ops=False):
        ops = C.c_double()
        out = CsrC()
        self._chk(self.lib.orc_matmul(C.byref(A.to_c()), C.byref(B.to_c()), C.byref(out), C.byref(ops)))
        m = SparseMatrix.from_c(out)
        self.lib.orc_csr_free(C.byref(out))
        return (m, ops.value) if want_ops else m

    def galerkin_product(self, R, A, P):
        return self._csr_call(self.lib.orc_galerkin_product, C.byref(R.to_c()), C.byref(A.to_c()),
                              C.byref(P.to_c()))

    def filter_matrix(self, G, theta=None, k=None):
        return self._csr_call(self.lib.orc_filter_matrix, C.byref(G.to_c()), C.c_int32(theta is not None),
                              C.c_double(theta or 0.0), C.c_int32(k or 0))

    def is_symmetric(self, A, tol=1e-12):
        s = C.c_int32()
        self._chk(self.lib.orc_is_symmetric(C.byref(A.to_c()), C.c_double(tol), C.byref(s)))
        return bool(s.value)

    def spectral_radius_estimate(self, A, steps=15):
        r = C.c_double()
        self._chk(self.lib.orc_spectral_radius(C.byref(A.to_c()), C.c_int32(steps), C.byref(r)))
        return r.value

    # -- strength / aggregation ---------------------------------------------
    def strength(self, A, cfg: StrengthConfig, want_ops=False):
        ops = C.c_double()
        out = CsrC()
        c = cfg.to_c()
        self._chk(self.lib.orc_strength(C.byref(A.to_c()), C.byref(c), C.byref(out), C.byref(ops)))
        m = SparseMatrix.from_c(out)
        self.lib.orc_csr_free(C.byref(out))
        return (m, ops.value) if want_ops else m

    def normalize_strength(self, S):
        return self._csr_call(self.lib.orc_normalize_strength, C.byref(S.to_c()))

    def amalgamate(self, S, m):
        return self._csr_call(self.lib.orc_amalgamate, C.byref(S.to_c()), C.c_int32(m))

    def greedy_aggregate(self, S):
        n = S.n_rows
        na = C.c_int32()
        n2a = np.zeros(max(n, 1), np.int32)
        roots = np.zeros(max(n, 1), np.int32)
        self._chk(self.lib.orc_greedy_aggregate(C.byref(S.to_c()), C.byref(na), ptr_i32(n2a), ptr_i32(roots)))
        return na.value, n2a[:n], roots[:na.value]

    def sparsity_pattern(self, S, Cm, degree):
        return self._csr_call(self.lib.orc_sparsity_pattern, C.byref(S.to_c()), C.byref(Cm.to_c()),
                              C.c_int32(degree))

    def root_node_pattern(self, N, roots):
        r = as_i32(roots)
        return self._csr_call(self.lib.orc_root_node_pattern, C.byref(N.to_c()), C.c_int32(len(r)), ptr_i32(r))

    def improve_candidates(self, A, B: CandidateSet, sweeps, scheme=1, weight=0.0):
        out = np.zeros(B.n * B.k)
        self._chk(self.lib.orc_improve_candidates(C.byref(A.to_c()), C.c_int32(B.k), ptr_f64(B.data),
                                                  C.c_int32(sweeps), C.c_int32(int(scheme)), C.c_double(weight),
                                                  ptr_f64(out)))
        return CandidateSet(B.n, B.k, out)

    def relax(self, A, scheme, weight, sweeps, x, b):
        x = as_f64(x).copy()
        b = as_f64(b)
        self._chk(self.lib.orc_relax(C.byref(A.to_c()), C.c_int32(int(scheme)), C.c_double(weight),
                                     C.c_int32(sweeps), ptr_f64(x), ptr_f64(b)))
        return x

    def relax_weight(self, A, scheme=0, weight=0.0):
        w = C.c_double()
        self._chk(self.lib.orc_relax_weight(C.byref(A.to_c()), C.c_int32(int(scheme)), C.c_double(weight),
                                            C.byref(w)))
        return w.value

    def inject_tentative(self, node_to_agg, roots, N, B: CandidateSet, m):
        n2a, r = as_i32(node_to_agg), as_i32(roots)
        out = CsrC()
        bc = f64p()
        self._chk(self.lib.orc_inject_tentative(C.c_int32(len(n2a)), C.c_int32(len(r)), ptr_i32(n2a), ptr_i32(r),
                                                C.byref(N.to_c()), C.c_int32(B.k), ptr_f64(B.data), C.c_int32(m),
                                                C.byref(out), C.byref(bc)))
        T = SparseMatrix.from_c(out)
        self.lib.orc_csr_free(C.byref(out))
        nc = len(r) * m
        Bc = np.ctypeslib.as_array(bc, shape=(max(1, nc * B.k),))[:nc * B.k].copy()
        self.lib.orc_free(bc)
        return T, CandidateSet(nc, B.k, Bc)

    def enforce_constraints(self, P, B: CandidateSet, Bc: CandidateSet, allowed=None):
        return self._csr_call(self.lib.orc_enforce_constraints, C.byref(P.to_c()), C.c_int32(B.k),
                              ptr_f64(B.data), ptr_f64(Bc.data),
                              C.byref(allowed.to_c()) if allowed is not None else None)

    def energy_minimize(self, A, T, B, Bc, N, energy_iters, krylov, roots):
        r = as_i32(roots)
        out = CsrC()
        its, bd = C.c_int32(), C.c_int32()
        self._chk(self.lib.orc_energy_minimize(C.byref(A.to_c()), C.byref(T.to_c()), C.c_int32(B.k),
                                               ptr_f64(B.data), ptr_f64(Bc.data), C.byref(N.to_c()),
                                               C.c_int32(energy_iters), C.c_int32(int(krylov)), C.c_int32(len(r)),
                                               ptr_i32(r), C.byref(out), C.byref(its), C.byref(bd)))
        P = SparseMatrix.from_c(out)
        self.lib.orc_csr_free(C.byref(out))
        return P, its.value, bool(bd.value)

    # -- hierarchy / solve ---------------------------------------------------
    def setup(self, A, B: CandidateSet, opts: SetupOptions, left: CandidateSet = None):
        h = C.c_void_p()
        o = opts.to_c()
        self._chk(self.lib.orc_setup(C.byref(A.to_c()), C.c_int32(B.k), ptr_f64(B.data),
                                     ptr_f64(left.data) if left is not None else None, C.byref(o), C.byref(h)))
        return Hierarchy(self, h.value)

    def solve(self, h: Hierarchy, b, x=None, opts: SolveOptions = None, history_cap=100000):
        b = as_f64(b)
        n = b.shape[0]
        x = np.zeros(n) if x is None or len(x) == 0 else as_f64(x).copy()
        opts = opts or SolveOptions()
        rep = SolveReportC()
        hist = np.zeros(history_cap)
        o = opts.to_c()
        self._chk(self.lib.orc_solve(h.handle, ptr_f64(b), ptr_f64(x), C.byref(o), C.byref(rep), ptr_f64(hist),
                                     C.c_int32(history_cap)))
        return x, SolveReport.from_c(rep, hist)

    def cycle(self, h: Hierarchy, x, b, kind=0):
        x = as_f64(x).copy()
        b = as_f64(b)
        self._chk(self.lib.orc_cycle(h.handle, ptr_f64(x), ptr_f64(b), C.c_int32(int(kind))))
        return x

    def generate_reference(self, kind, n, ny=0, eps=1.0, psi=0.0, nu=0.3, young=1.0, flow=0, material=1):
        A = CsrC()
        k, hl = C.c_int32(), C.c_int32()
        B, Bh, rhs = f64p(), f64p(), f64p()
        self._chk(self.lib.orc_generate_reference(kind, n, ny, C.c_double(eps), C.c_double(psi), C.c_double(nu),
                                                  C.c_double(young), flow, material, C.byref(A), C.byref(k),
                                                  C.byref(B), C.byref(hl), C.byref(Bh), C.byref(rhs)))
        M = SparseMatrix.from_c(A)
        self.lib.orc_csr_free(C.byref(A))
        nn = M.n_rows
        Bd = np.ctypeslib.as_array(B, shape=(nn * k.value,)).copy()
        self.lib.orc_free(B)
        Bhd = None
        if hl.value:
            Bhd = np.ctypeslib.as_array(Bh, shape=(nn * k.value,)).copy()
            self.lib.orc_free(Bh)
        r = np.ctypeslib.as_array(rhs, shape=(nn,)).copy()
        self.lib.orc_free(rhs)
        return M, CandidateSet(nn, k.value, Bd), (CandidateSet(nn, k.value, Bhd) if Bhd is not None else None), r
