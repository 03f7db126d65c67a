"""ctypes mirror of include/amgcu.h (structs shared by the product C ABI and the
oracle ABI in oracle/oracle_abi.h)."""
import ctypes as C

import numpy as np

i32p = C.POINTER(C.c_int32)
f64p = C.POINTER(C.c_double)


class CsrC(C.Structure):
    _fields_ = [
        ("n_rows", C.c_int32),
        ("n_cols", C.c_int32),
        ("nnz", C.c_int32),
        ("block_size", C.c_int32),
        ("row_offsets", i32p),
        ("col_indices", i32p),
        ("values", f64p),
    ]


class SetupOptionsC(C.Structure):
    _fields_ = [
        ("method", C.c_int32),
        ("strength_measure", C.c_int32),
        ("drop_tol", C.c_double),
        ("evolution_steps", C.c_int32),
        ("weighting", C.c_int32),
        ("degree", C.c_int32),
        ("prefilter_set", C.c_int32),
        ("prefilter_theta_set", C.c_int32),
        ("prefilter_theta", C.c_double),
        ("prefilter_k", C.c_int32),
        ("postfilter_set", C.c_int32),
        ("postfilter_theta_set", C.c_int32),
        ("postfilter_theta", C.c_double),
        ("postfilter_k", C.c_int32),
        ("energy_iters", C.c_int32),
        ("krylov", C.c_int32),
        ("pre_scheme", C.c_int32),
        ("pre_weight", C.c_double),
        ("pre_sweeps", C.c_int32),
        ("post_scheme", C.c_int32),
        ("post_weight", C.c_double),
        ("post_sweeps", C.c_int32),
        ("max_size", C.c_int32),
        ("max_levels", C.c_int32),
        ("candidate_sweeps", C.c_int32),
        ("cand_scheme", C.c_int32),
        ("cand_weight", C.c_double),
        ("cand_sweeps", C.c_int32),
    ]


class SolveOptionsC(C.Structure):
    _fields_ = [("method", C.c_int32), ("cycle", C.c_int32), ("tol", C.c_double), ("max_iters", C.c_int32)]


class SolveReportC(C.Structure):
    _fields_ = [
        ("iterations", C.c_int32),
        ("converged", C.c_int32),
        ("diverged", C.c_int32),
        ("history_len", C.c_int32),
        ("rho", C.c_double),
        ("chi_oc", C.c_double),
        ("chi_cc", C.c_double),
        ("work_units_solve", C.c_double),
        ("work_units_setup", C.c_double),
    ]


class StrengthConfigC(C.Structure):
    _fields_ = [("measure", C.c_int32), ("drop_tol", C.c_double), ("evolution_steps", C.c_int32),
                ("weighting", C.c_int32)]


def as_i32(a):
    return np.ascontiguousarray(a, dtype=np.int32)


def as_f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def ptr_i32(a):
    return a.ctypes.data_as(i32p)


def ptr_f64(a):
    return a.ctypes.data_as(f64p) if a is not None else None
