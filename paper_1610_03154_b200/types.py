"""Host-side mirror of the reference's public types (namespace amg).

Same names, fields and defaults as the reference headers so code written
against the reference reads the same here:
  SparseMatrix        core/sparse.hpp:25-62
  CandidateSet        core/dense.hpp:15-32
  StrengthConfig      strength.hpp:15-25
  FilterRule / InterpConfig   interpolation.hpp:19-32
  RelaxConfig         relaxation.hpp:18-24
  SetupOptions        hierarchy.hpp:24-36
  SolveOptions / SolveReport  cycle.hpp:17-36
These are plain containers; the compute lives in libamgcu.so (CUDA, sm_100a).
"""
from __future__ import annotations

import ctypes as C
import enum
from dataclasses import dataclass, field
from typing import List, Optional

import numpy as np

from ._abi import CsrC, SetupOptionsC, SolveOptionsC, StrengthConfigC, as_f64, as_i32, ptr_f64, ptr_i32


class StrengthMeasure(enum.IntEnum):
    classical = 0
    symmetric = 1
    evolution = 2


class EvolutionWeighting(enum.IntEnum):
    spectral = 0
    l1jacobi = 1


class KrylovKind(enum.IntEnum):
    cg = 0
    gmres = 1


class RelaxScheme(enum.IntEnum):
    jacobi = 0
    gauss_seidel = 1
    sym_gauss_seidel = 2
    gsne = 3
    block_sym_gauss_seidel = 4


class SetupMethod(enum.IntEnum):
    rn = 0
    sa = 1
    cf = 2


class SolveMethod(enum.IntEnum):
    stationary = 0
    pcg = 1
    fgmres = 2


class CycleKind(enum.IntEnum):
    V = 0
    W = 1


class SparseMatrix:
    """Canonical CSR: sorted columns, no duplicates, no stored zeros (sparse.hpp:21-24)."""

    __slots__ = ("n_rows", "n_cols", "block_size", "row_offsets", "col_indices", "values")

    def __init__(self, n_rows=0, n_cols=0, row_offsets=None, col_indices=None, values=None, block_size=1):
        self.n_rows = int(n_rows)
        self.n_cols = int(n_cols)
        self.block_size = int(block_size)
        self.row_offsets = as_i32(np.zeros(self.n_rows + 1) if row_offsets is None else row_offsets)
        self.col_indices = as_i32(np.zeros(0) if col_indices is None else col_indices)
        self.values = as_f64(np.zeros(0) if values is None else values)

    def nnz(self) -> int:
        return int(self.col_indices.shape[0])

    def row_nnz(self, i) -> int:
        return int(self.row_offsets[i + 1] - self.row_offsets[i])

    def row_cols(self, i):
        return self.col_indices[self.row_offsets[i]:self.row_offsets[i + 1]]

    def row_vals(self, i):
        return self.values[self.row_offsets[i]:self.row_offsets[i + 1]]

    def coeff(self, i, j) -> float:
        cols = self.row_cols(i)
        p = int(np.searchsorted(cols, j))
        if p < cols.shape[0] and cols[p] == j:
            return float(self.values[self.row_offsets[i] + p])
        return 0.0

    def __eq__(self, o) -> bool:  # bitwise, as SparseMatrix::operator== (sparse.hpp:58-61)
        return (self.n_rows == o.n_rows and self.n_cols == o.n_cols
                and np.array_equal(self.row_offsets, o.row_offsets)
                and np.array_equal(self.col_indices, o.col_indices)
                and self.values.tobytes() == o.values.tobytes())

    def to_dense(self) -> np.ndarray:
        d = np.zeros((self.n_rows, self.n_cols))
        rows = np.repeat(np.arange(self.n_rows), np.diff(self.row_offsets))
        d[rows, self.col_indices] = self.values
        return d

    def to_c(self) -> CsrC:
        c = CsrC(self.n_rows, self.n_cols, self.nnz(), self.block_size, ptr_i32(self.row_offsets),
                 ptr_i32(self.col_indices), ptr_f64(self.values))
        c._keep = (self.row_offsets, self.col_indices, self.values)
        return c

    @staticmethod
    def from_c(c: CsrC) -> "SparseMatrix":
        n, nnz = c.n_rows, c.nnz
        ro = np.ctypeslib.as_array(c.row_offsets, shape=(n + 1,)).copy()
        ci = np.ctypeslib.as_array(c.col_indices, shape=(nnz,)).copy() if nnz else np.zeros(0, np.int32)
        va = np.ctypeslib.as_array(c.values, shape=(nnz,)).copy() if nnz else np.zeros(0)
        return SparseMatrix(n, c.n_cols, ro, ci, va, c.block_size)

    def __repr__(self):
        return f"SparseMatrix({self.n_rows}x{self.n_cols}, nnz={self.nnz()}, block_size={self.block_size})"


def from_triplets(n_rows, n_cols, triplets) -> SparseMatrix:
    """sparse.hpp:72-100 for small test fixtures: sums duplicates (stable order),
    drops exact zeros.  Large generators live in libamgcu (amgcu_generate)."""
    rows = {}
    for (i, j, v) in triplets:
        if not (0 <= i < n_rows and 0 <= j < n_cols):
            raise ValueError("from_triplets: entry out of range")
        rows.setdefault(i, {})
        rows[i][j] = rows[i].get(j, 0.0) + v
    ro = [0]
    ci, va = [], []
    for i in range(n_rows):
        for j in sorted(rows.get(i, {})):
            v = rows[i][j]
            if v != 0.0:
                ci.append(j)
                va.append(v)
        ro.append(len(ci))
    return SparseMatrix(n_rows, n_cols, ro, ci, va)


def identity(n) -> SparseMatrix:
    return SparseMatrix(n, n, np.arange(n + 1), np.arange(n), np.ones(n))


class CandidateSet:
    """n x k column-major candidate block (dense.hpp:15-32)."""

    __slots__ = ("n", "k", "data")

    def __init__(self, n, k, data=None):
        if n < 0 or k < 1:
            raise ValueError("CandidateSet: need n >= 0, k >= 1")
        self.n, self.k = int(n), int(k)
        self.data = as_f64(np.zeros(self.n * self.k) if data is None else np.asarray(data).reshape(-1))

    def at(self, i, j):
        return float(self.data[j * self.n + i])

    def col(self, j):
        return self.data[j * self.n:(j + 1) * self.n]

    def as_columns(self) -> np.ndarray:
        return self.data.reshape(self.k, self.n).T


def constant_candidates(n) -> CandidateSet:
    return CandidateSet(n, 1, np.ones(n))


@dataclass
class StrengthConfig:
    measure: StrengthMeasure = StrengthMeasure.evolution
    drop_tol: float = 4.0
    evolution_steps: int = 2
    weighting: EvolutionWeighting = EvolutionWeighting.spectral

    def to_c(self):
        return StrengthConfigC(int(self.measure), float(self.drop_tol), int(self.evolution_steps),
                               int(self.weighting))


@dataclass
class FilterRule:
    theta: Optional[float] = None
    k: Optional[int] = None


@dataclass
class InterpConfig:
    degree: int = 2
    prefilter: Optional[FilterRule] = None
    postfilter: Optional[FilterRule] = None
    energy_iters: int = 0
    krylov: KrylovKind = KrylovKind.cg


@dataclass
class RelaxConfig:
    scheme: RelaxScheme = RelaxScheme.sym_gauss_seidel
    weight: float = 0.0
    sweeps: int = 1


@dataclass
class SetupOptions:
    method: SetupMethod = SetupMethod.rn
    strength: StrengthConfig = field(default_factory=StrengthConfig)
    interp: InterpConfig = field(default_factory=InterpConfig)
    pre_relax: RelaxConfig = field(default_factory=lambda: RelaxConfig(RelaxScheme.sym_gauss_seidel, 0.0, 1))
    post_relax: RelaxConfig = field(default_factory=lambda: RelaxConfig(RelaxScheme.sym_gauss_seidel, 0.0, 1))
    max_size: int = 20
    max_levels: int = 25
    candidate_sweeps: int = 4
    candidate_relax: RelaxConfig = field(default_factory=lambda: RelaxConfig(RelaxScheme.gauss_seidel, 0.0, 1))

    def to_c(self) -> SetupOptionsC:
        o = SetupOptionsC()
        o.method = int(self.method)
        o.strength_measure = int(self.strength.measure)
        o.drop_tol = float(self.strength.drop_tol)
        o.evolution_steps = int(self.strength.evolution_steps)
        o.weighting = int(self.strength.weighting)
        o.degree = int(self.interp.degree)
        for name, rule in (("prefilter", self.interp.prefilter), ("postfilter", self.interp.postfilter)):
            setattr(o, name + "_set", 1 if rule is not None else 0)
            setattr(o, name + "_theta_set", 1 if (rule is not None and rule.theta is not None) else 0)
            setattr(o, name + "_theta", float(rule.theta) if (rule is not None and rule.theta is not None) else 0.0)
            setattr(o, name + "_k", int(rule.k) if (rule is not None and rule.k is not None) else 0)
        o.energy_iters = int(self.interp.energy_iters)
        o.krylov = int(self.interp.krylov)
        o.pre_scheme, o.pre_weight, o.pre_sweeps = int(self.pre_relax.scheme), float(self.pre_relax.weight), int(self.pre_relax.sweeps)
        o.post_scheme, o.post_weight, o.post_sweeps = int(self.post_relax.scheme), float(self.post_relax.weight), int(self.post_relax.sweeps)
        o.max_size, o.max_levels, o.candidate_sweeps = int(self.max_size), int(self.max_levels), int(self.candidate_sweeps)
        o.cand_scheme, o.cand_weight, o.cand_sweeps = (int(self.candidate_relax.scheme), float(self.candidate_relax.weight),
                                                       int(self.candidate_relax.sweeps))
        return o

    @staticmethod
    def from_c(o: SetupOptionsC) -> "SetupOptions":
        def rule(prefix):
            if not getattr(o, prefix + "_set"):
                return None
            return FilterRule(getattr(o, prefix + "_theta") if getattr(o, prefix + "_theta_set") else None,
                              getattr(o, prefix + "_k") if getattr(o, prefix + "_k") > 0 else None)
        return SetupOptions(
            SetupMethod(o.method),
            StrengthConfig(StrengthMeasure(o.strength_measure), o.drop_tol, o.evolution_steps,
                           EvolutionWeighting(o.weighting)),
            InterpConfig(o.degree, rule("prefilter"), rule("postfilter"), o.energy_iters, KrylovKind(o.krylov)),
            RelaxConfig(RelaxScheme(o.pre_scheme), o.pre_weight, o.pre_sweeps),
            RelaxConfig(RelaxScheme(o.post_scheme), o.post_weight, o.post_sweeps),
            o.max_size, o.max_levels, o.candidate_sweeps,
            RelaxConfig(RelaxScheme(o.cand_scheme), o.cand_weight, o.cand_sweeps))


@dataclass
class SolveOptions:
    method: SolveMethod = SolveMethod.stationary
    cycle: CycleKind = CycleKind.V
    tol: float = 1e-8
    max_iters: int = 100

    def to_c(self) -> SolveOptionsC:
        return SolveOptionsC(int(self.method), int(self.cycle), float(self.tol), int(self.max_iters))


@dataclass
class SolveReport:
    residual_history: List[float] = field(default_factory=list)
    iterations: int = 0
    converged: bool = False
    diverged: bool = False
    rho: float = 0.0
    chi_oc: float = 0.0
    chi_cc: float = 0.0
    work_units_solve: float = 0.0
    work_units_setup: float = 0.0

    @staticmethod
    def from_c(r, hist) -> "SolveReport":
        return SolveReport(list(hist[:min(r.history_len, len(hist))]), r.iterations, bool(r.converged),
                           bool(r.diverged), r.rho, r.chi_oc, r.chi_cc, r.work_units_solve, r.work_units_setup)


@dataclass
class Level:
    A: SparseMatrix
    P: Optional[SparseMatrix]
    R: Optional[SparseMatrix]
    B: CandidateSet
    Bc: Optional[CandidateSet]
    symmetric: bool


class AmgError(Exception):
    pass


_EXC = {1: ValueError, 2: RuntimeError, 3: AmgError}


def raise_for(code: int, msg: str):
    """Map status codes to the reference exception classes
    (invalid_argument -> ValueError, runtime_error -> RuntimeError)."""
    if code == 0:
        return
    exc = _EXC.get(code, RuntimeError)
    raise exc(msg)
