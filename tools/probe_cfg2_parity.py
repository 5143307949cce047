"""Probe: cfg2_full GPU solve vs the reference golden (seed-42 RHS)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np
import paper_1806_05826_b200 as R
import bench
from helpers import rel_diff
cfg = bench.CONFIGS["cfg2"]
g = np.load("tests/golden/cfg2_full.npz")
x = bench.make_matrix(cfg)
m = R.DeviceMatrix(x)
labels = [g["labels0"].astype(np.int64), g["labels1"].astype(np.int64)]
for dense in ("1", "0"):
    if dense == "0":
        os.environ["RMG_DISABLE_DENSE_INNER"] = "1"
    pm = R.PreparedMethod(m, 1.0, R.MethodSpec(kind=R.FCG_MULTILEVEL, levels=bench.level_specs(cfg, labels),
                                               solver=R.SolverConfig(1e-6, 1000)))
    w, rep = pm.solve(g["b"])
    gi = g["ml_inner"].astype(np.int64)
    k = min(len(gi), rep.iterations)
    print(f"dense={dense}: iters {rep.iterations} (ref {int(g['ml_iterations'])}) w rel {rel_diff(w, g['ml_w']):.3e} "
          f"inner mean {rep.inner_iterations.mean():.2f} (ref {gi.mean():.2f}) first-50 inner |d| "
          f"{np.mean(np.abs(rep.inner_iterations[:50].astype(np.int64) - gi[:50])):.2f} "
          f"omega {[pm.level(i)['omega'] for i in range(2)]} ref {list(g['ml_omega'])}", flush=True)
    h = rep.residual_history
    gh = g["ml_hist"]
    for it in (0, 1, 10, 100, 300, 600):
        if it < len(h) and it < len(gh):
            print(f"   it {it}: rel {h[it]:.6e} ref {gh[it]:.6e}")
    pm.close()
