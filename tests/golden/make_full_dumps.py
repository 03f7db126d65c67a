"""Full-size (BASELINE sizes) dumps of the CPU oracle, for the GPU config-scale parity tests.

A full-size CPU setup + solve takes from seconds (C2) to many minutes (C1-256: the
dense COD of its 11,008-row coarsest level; C3/C4 at 4.2 M DOFs), so the GPU tests
(tests/test_gpu_config_scale.py) compare against these committed dumps instead of
running the oracle on the box.  A dump holds, per level, the SHA-256 of every array
of A, P, R (row offsets, column indices, values) and of the candidates B and Bc, the
symmetry flag, the Jacobi weights, and for the solve the iteration count, the whole
residual history and x sampled every `XSTRIDE`-th entry.

  --kind port  the own-code restatement (oracle/rnamg_port.cpp) -- default
  --kind ref   the reference build (oracle/_ref; needs it built from /root/reference)

Both kinds write the same keys; `tests/test_full_dumps.py` checks that every committed
reference dump equals the port's (the restatement pinned against the reference at full
size).  The dump is keyed by a hash of the generated problem (A, B, b bytes) and the
options, so a changed generator invalidates it loudly.

Usage: python tests/golden/make_full_dumps.py [--kind port|ref] [C1 C2 ...]
"""
import argparse
import hashlib
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

from oracle.pyoracle import Oracle, config_options, generate_config  # noqa: E402

FULL = {"C1": (1, 256, 0), "C2": (2, 1024, 0), "C3": (3, 2048, 2), "C4": (4, 2048, 3), "C5": (5, 1024, 0)}
XSTRIDE = 64
OUT = os.path.join(HERE, "full")


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def problem_key(A, B, Bh, b, so, vo):
    h = hashlib.sha256()
    for a in (A.row_offsets, A.col_indices, A.values, B.data, b):
        h.update(np.ascontiguousarray(a).tobytes())
    if Bh is not None:
        h.update(np.ascontiguousarray(Bh.data).tobytes())
    h.update(repr(sorted(vars(so).items())).encode())
    h.update(repr(sorted(vars(vo).items())).encode())
    return h.hexdigest()


def hierarchy_hashes(h):
    """{key: sha256} of every array of the hierarchy (the same keys for the GPU side)"""
    out = {}
    L = h.n_levels()
    for l in range(L):
        for which, tag in [(0, "A")] + ([(1, "P"), (2, "R")] if l + 1 < L else []):
            M = h.matrix(l, which)
            out[f"L{l}_{tag}_ro"] = sha(M.row_offsets)
            out[f"L{l}_{tag}_ci"] = sha(M.col_indices)
            out[f"L{l}_{tag}_va"] = sha(M.values)
            out[f"L{l}_{tag}_shape"] = f"{M.n_rows}x{M.n_cols}/{M.block_size}/{M.nnz()}"
        out[f"L{l}_B"] = sha(h.candidates(l, 0).data)
        if l + 1 < L:
            out[f"L{l}_Bc"] = sha(h.candidates(l, 1).data)
        out[f"L{l}_sym"] = str(int(h.symmetric(l)))
    return out


def solve_restarts(orc, h, b, vo, restarts):
    x, rep = orc.solve(h, b, None, vo)
    hist = list(rep.residual_history)
    its = rep.iterations
    for _ in range(restarts):  # GMRES(m) restarted from the current x (bench.py's loop)
        if rep.converged or rep.diverged:
            break
        x, rep = orc.solve(h, b, x, vo)
        hist += list(rep.residual_history)
        its += rep.iterations
    return x, its, bool(rep.converged), np.array(hist)


def dump(name, kind):
    cfg, size, restarts = FULL[name]
    A, B, Bh, b = generate_config(cfg, size)
    so, vo = config_options(cfg)
    orc = Oracle(kind)
    t0 = time.time()
    h = orc.setup(A, B, so, Bh)
    t1 = time.time()
    x, its, conv, hist = solve_restarts(orc, h, b, vo, restarts)
    t2 = time.time()
    hh = hierarchy_hashes(h)
    keys = sorted(hh)
    os.makedirs(OUT, exist_ok=True)
    np.savez_compressed(os.path.join(OUT, f"{name.lower()}_{kind}.npz"),
                        problem=np.array(problem_key(A, B, Bh, b, so, vo)), keys=np.array(keys),
                        values=np.array([hh[k] for k in keys]), levels=np.array([h.n_levels(), int(h.stagnated)]),
                        its=np.array([its, int(conv), restarts]), hist=hist, x_sample=x[::XSTRIDE].copy(),
                        x_norm=np.array([float(np.linalg.norm(x))]), times=np.array([t1 - t0, t2 - t1]))
    print(f"{name} {kind}: levels {h.n_levels()} its {its} converged {conv} setup {t1 - t0:.1f}s solve {t2 - t1:.1f}s",
          flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--kind", default="port", choices=["port", "ref"])
    ap.add_argument("names", nargs="*", default=list(FULL))
    a = ap.parse_args()
    for name in a.names:
        dump(name, a.kind)


if __name__ == "__main__":
    main()
