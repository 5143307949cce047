"""Probe: pcg_vcycle against the reference's methods on cfg 1 and cfg 2."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

import bench
import paper_1806_05826_b200 as R

for name in ("cfg1", "cfg2"):
    cfg = bench.CONFIGS[name]
    x = bench.make_matrix(cfg)
    m = R.DeviceMatrix.from_dense(x.dense()) if cfg["kind"] == "dense" else R.DeviceMatrix(x)
    labels = bench.load_golden_labels(cfg)
    b = R.rng_normals(42, x.n_samples)
    for method in (cfg["method"], "pcg_vcycle"):
        spec = R.MethodSpec(kind=R.method_from_string(method), levels=bench.level_specs(cfg, labels),
                            solver=R.SolverConfig(cfg["tol"], cfg["max_iters"]))
        pm = R.PreparedMethod(m, cfg["beta"], spec)
        pm.solve(b)
        ts = []
        for _ in range(3):
            t = time.time()
            w, rep = pm.solve(b)
            ts.append(time.time() - t)
        print(f"{name} {method:15s}: {rep.iterations} iterations, {1e3 * min(ts):.2f} ms, converged {rep.converged}",
              flush=True)
        pm.close()
