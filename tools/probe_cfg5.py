"""Probe: BASELINE cfg 5 end to end on one GPU (16M x 500k binary, Poisson(64),
Zipf(1.05); levels 50k/5k/500 by sketched k-means; pcg_vcycle; beta 0.5).
usage: RMG_SETUP_LOG=1 python tools/probe_cfg5.py [N]"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import psutil

import paper_1806_05826_b200 as R

n = int(sys.argv[1]) if len(sys.argv) > 1 else 16_000_000
method = sys.argv[2] if len(sys.argv) > 2 else "pcg_vcycle"
proc = psutil.Process()


def mem():
    import torch
    free, total = torch.cuda.mem_get_info()
    return f"host RSS {proc.memory_info().rss / 2**30:.1f} GiB, device used {(total - free) / 2**30:.1f} GiB"


t = time.time()
x = R.synth_sparse_zipf(n, 500_000, 64.0, 1.05, False, 0, row_streams=True)
print(f"generate {time.time() - t:.1f} s, nnz {x.nnz}; {mem()}", flush=True)
t = time.time()
m = R.DeviceMatrix(x)
print(f"upload {time.time() - t:.1f} s; {mem()}", flush=True)
levels = []
ks = [50_000, 5_000, 500]
for i, k in enumerate(ks):
    last = i == len(ks) - 1
    levels.append(R.LevelSpec(clustering=R.ClusteringChoice(kind=R.KMEANS_SKETCH, target_size=k, seed=0,
                                                           normalize_columns=True, sketch_dim=32),
                              solver=R.CoarseSolveChoice(kind=R.DIRECT_CHOLESKY if last else R.INNER_FCG)))
t = time.time()
pm = R.PreparedMethod(m, 0.5, R.MethodSpec(kind=R.method_from_string(method), levels=levels,
                                           solver=R.SolverConfig(1e-6, 1000)))
print(f"prepare {time.time() - t:.1f} s; levels", [(pm.level(i)["n_features"], pm.level(i)["nnz"])
                                                   for i in range(pm.n_levels)], f"; {mem()}", flush=True)
b = R.rng_normals(42, n)
for rep in range(3):
    t = time.time()
    w, r = pm.solve(b)
    print(f"solve {1e3 * (time.time() - t):.1f} ms wall, {r.iterations} iterations, converged {r.converged}, "
          f"solver {1e3 * r.wall_time_s:.1f} ms", flush=True)
for lv in range(pm.n_levels):
    print("level", lv, "operator cold ms", pm.time_operator(lv, 5, True)[0], flush=True)
