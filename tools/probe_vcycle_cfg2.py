"""Probe: one cfg 2 solve with pcg_vcycle (for a kernel launch list)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench
import paper_1806_05826_b200 as R

cfg = bench.CONFIGS["cfg2"]
x = bench.make_matrix(cfg)
m = R.DeviceMatrix(x)
spec = R.MethodSpec(kind=R.PCG_VCYCLE, levels=bench.level_specs(cfg, bench.load_golden_labels(cfg)),
                    solver=R.SolverConfig(cfg["tol"], cfg["max_iters"]))
pm = R.PreparedMethod(m, cfg["beta"], spec)
b = R.rng_normals(42, x.n_samples)
w, rep = pm.solve(b)
print("iterations", rep.iterations, "wall ms", rep.wall_time_s * 1e3)
