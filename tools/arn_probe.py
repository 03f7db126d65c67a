"""Spectral-radius estimate of a BASELINE config's finest matrix in parity mode
(reference order) and production mode (cooperative Arnoldi): relative gap."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1610_03154_b200.api as api
cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 2
size = int(sys.argv[2]) if len(sys.argv) > 2 else 1024
A, B, Bh, b = api.generate_config(cfg, size)
seq = api.Context(0, sequential_reductions=True)
prod = api.Context(0)
r1 = api.spectral_radius_estimate(A, ctx=seq)
r2 = api.spectral_radius_estimate(A, ctx=prod)
print(f"C{cfg}/{size} n {A.n_rows} rho seq {r1!r} prod {r2!r} rel {abs(r1 - r2) / r1:.3e}")
