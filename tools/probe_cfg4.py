"""Probe: BASELINE cfg 4 end to end (dense fp32 storage, 3 levels 128/16,
k-means on unit-normalised columns, beta 1e-4, FCG multilevel to 1e-6) at N rows.
usage: RMG_SETUP_LOG=1 python tools/probe_cfg4.py [N]"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

import bench
import paper_1806_05826_b200 as R

n = int(sys.argv[1]) if len(sys.argv) > 1 else 500_000
t = time.time()
a = bench.cfg4_shard_matrix(n=n)
print(f"generate {time.time() - t:.1f} s", flush=True)
t = time.time()
m = R.DeviceMatrix.from_dense(a)
print(f"upload {time.time() - t:.1f} s", flush=True)
specs = []
for i, k in enumerate([128, 16]):
    last = i == 1
    specs.append(R.LevelSpec(clustering=R.ClusteringChoice(kind=R.KMEANS, target_size=k, seed=0, kmeans_max_iters=100,
                                                           normalize_columns=True),
                             solver=R.CoarseSolveChoice(kind=R.DIRECT_CHOLESKY if last else R.INNER_FCG, tol=1e-6,
                                                        max_iters=500)))
t = time.time()
pm = R.PreparedMethod(m, 1e-4, R.MethodSpec(kind=R.FCG_MULTILEVEL, levels=specs, solver=R.SolverConfig(1e-6, 1000)))
print(f"prepare {time.time() - t:.1f} s", flush=True)
b = R.rng_normals(42, n)
for rep in range(3):
    t = time.time()
    w, r = pm.solve(b)
    print(f"solve {1e3 * (time.time() - t):.1f} ms wall, {r.iterations} iterations, inner {r.inner_iterations}, "
          f"converged {r.converged}, solver {1e3 * r.wall_time_s:.2f} ms", flush=True)
cg = R.PreparedMethod(m, 1e-4, R.MethodSpec(kind=R.CG, solver=R.SolverConfig(1e-6, 1000)))
w2, r2 = cg.solve(b)
print(f"CG {r2.iterations} iterations, {1e3 * r2.wall_time_s:.2f} ms; |w-w_cg|/|w| = "
      f"{np.linalg.norm(w - w2) / np.linalg.norm(w2):.2e}")
