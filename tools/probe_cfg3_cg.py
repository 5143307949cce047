"""Probe: plain CG on BASELINE cfg 3 (1M x 100k, |N(0,1)| values, Zipf(1.1)) for every
beta of the sweep, one right-hand side (seed 42): iteration counts and device time.
These are the like-for-like (same algorithm) counterparts of the reference's cg.
usage: python tools/probe_cfg3_cg.py [N F maxit]"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

import paper_1806_05826_b200 as R

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1_000_000
f = int(sys.argv[2]) if len(sys.argv) > 2 else 100_000
maxit = int(sys.argv[3]) if len(sys.argv) > 3 else 400_000
t = time.time()
x = R.synth_sparse_zipf(n, f, 50.0, 1.1, True, 0, row_streams=True)
print(f"generate {time.time() - t:.1f} s, nnz {x.nnz}", flush=True)
m = R.DeviceMatrix(x)
b = R.rng_normals(42, n)
for beta in (10.0, 1.0, 1e-1, 1e-2, 1e-3):
    pm = R.PreparedMethod(m, beta, R.MethodSpec(kind=R.CG, solver=R.SolverConfig(1e-6, maxit)))
    t = time.time()
    w, r = pm.solve(b)
    dt = time.time() - t
    print(f"cg beta {beta:g}: {r.iterations} iterations, converged {r.converged}, {dt:.2f} s wall, "
          f"{1e3 * dt / max(1, r.iterations):.3f} ms/it, |w| {np.linalg.norm(w):.6e}", flush=True)
    pm.close()
