"""B200-native root-node AMG core (arXiv 1610.03154 RN-AMG setup + solve).

The compute lives in libamgcu.so (hand-written sm_100a CUDA behind the C ABI
in include/amgcu.h); this package is the host-side mirror of the reference's
API (namespace amg in /root/reference/proj/include/amg) for Python callers
and tests.
"""
from .types import (AmgError, CandidateSet, CycleKind, EvolutionWeighting, FilterRule, InterpConfig, KrylovKind,
                    Level, RelaxConfig, RelaxScheme, SetupMethod, SetupOptions, SolveMethod, SolveOptions,
                    SolveReport, SparseMatrix, StrengthConfig, StrengthMeasure, constant_candidates, from_triplets,
                    identity)


def __getattr__(name):
    # the compute API loads libamgcu lazily so that the types stay importable
    # in environments without the built library (CPU-only tests of the oracle)
    if name.startswith("__"):
        raise AttributeError(name)
    import importlib
    if name in ("build", "api", "types", "replicas", "_abi"):
        # submodules: `from paper_1610_03154_b200 import build` must work before
        # libamgcu.so exists (a fresh checkout builds through it)
        return importlib.import_module(__name__ + "." + name)
    api = importlib.import_module(__name__ + ".api")
    if hasattr(api, name):
        return getattr(api, name)
    raise AttributeError(name)
