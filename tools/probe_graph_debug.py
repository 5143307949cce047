"""Debug: cfg3 pieces with progress prints (graphs on/off via RMG_NO_GRAPH)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import bench
import paper_1806_05826_b200 as R
cfg = bench.CONFIGS["cfg3"]
n = int(sys.argv[1]) if len(sys.argv) > 1 else cfg["n"]
x = R.synth_sparse_zipf(n, cfg["f"] * n // cfg["n"], 50.0, 1.1, True, 0, row_streams=True)
m = R.DeviceMatrix(x)
ks = [k * n // cfg["n"] for k in cfg["ks"]]
spec = R.MethodSpec(kind=R.PCG_VCYCLE, levels=bench.level_specs(dict(cfg, ks=ks)), solver=R.SolverConfig(1e-6, 1000))
pm = R.PreparedMethod(m, 1.0, spec)
print("prepared", flush=True)
b = R.rng_normals(42, n)
t = time.time(); w, r = pm.solve(b); print("single", r.iterations, time.time() - t, flush=True)
B = np.stack([R.rng_normals(42 + q, n) for q in range(16)], axis=1)
t = time.time(); W, reps = pm.solve_batch(B); print("batch", [q.iterations for q in reps], time.time() - t, flush=True)
pm.set_beta(10.0)
t = time.time(); W, reps = pm.solve_batch(B); print("batch beta10", [q.iterations for q in reps], time.time() - t, flush=True)
pc = R.PreparedMethod(m, 1.0, R.MethodSpec(kind=R.CG, solver=R.SolverConfig(1e-6, 50000)))
t = time.time(); w, r = pc.solve(b); print("cg", r.iterations, time.time() - t, flush=True)
