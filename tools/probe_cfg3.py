"""Probe: BASELINE cfg 3 end to end (1M x 100k, ~50 nnz/row |N(0,1)|, Zipf(1.1);
4 levels 10k/1k/100 by sketched k-means; beta sweep; one RHS per beta).
usage: RMG_SETUP_LOG=1 python tools/probe_cfg3.py [N F]"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

import paper_1806_05826_b200 as R

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1_000_000
f = int(sys.argv[2]) if len(sys.argv) > 2 else 100_000
ks = [int(v) for v in sys.argv[3].split(",")] if len(sys.argv) > 3 else [10_000, 1_000, 100]
method = sys.argv[4] if len(sys.argv) > 4 else "fcg_multilevel"
t = time.time()
x = R.synth_sparse_zipf(n, f, 50.0, 1.1, True, 0, row_streams=True)
print(f"generate {time.time() - t:.1f} s, nnz {x.nnz}", flush=True)
t = time.time()
m = R.DeviceMatrix(x)
print(f"upload {time.time() - t:.1f} s", flush=True)
levels = []
for i, k in enumerate(ks):
    last = i == len(ks) - 1
    levels.append(R.LevelSpec(clustering=R.ClusteringChoice(kind=R.KMEANS_SKETCH, target_size=k, seed=0,
                                                           normalize_columns=True, sketch_dim=32),
                              solver=R.CoarseSolveChoice(kind=R.DIRECT_CHOLESKY if last else R.INNER_FCG,
                                                         tol=1e-6, max_iters=500)))
t = time.time()
pm = R.PreparedMethod(m, 1.0, R.MethodSpec(kind=R.method_from_string(method), levels=levels,
                                            solver=R.SolverConfig(1e-6, 1000)))
print(f"prepare {time.time() - t:.1f} s; levels", [pm.level(i)["n_features"] for i in range(pm.n_levels)], flush=True)
for beta in (1.0, 10.0, 1e-1, 1e-2, 1e-3):
    pm.set_beta(beta)
    b = R.rng_normals(42, n)
    pm.solve(b)  # warm
    t = time.time()
    w, r = pm.solve(b)
    inner = r.inner_iterations
    print(f"beta {beta:g}: {1e3 * (time.time() - t):.0f} ms wall, {r.iterations} outer, inner mean "
          f"{np.mean(inner) if len(inner) else 0:.1f}, converged {r.converged}", flush=True)
