"""Probe: cfg 2 plain CG iteration count under the K1 layouts."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests"))
import paper_1806_05826_b200 as R
from helpers import load_golden, rel_diff
for name, n, f in (("cfg2_small", 10000, 2000), ("cfg2_full", 100000, 20000)):
    g = load_golden(name)
    m = R.DeviceMatrix(R.synth_sparse_zipf(n, f, 40.0, 1.1, False, 0))
    cg = R.solve_system(m, 1.0, g["b"], R.MethodSpec(kind=R.CG, solver=R.SolverConfig(1e-6, 5000)))
    print(os.environ.get("RMG_K1", "sell"), name, "cg", cg.report.iterations, "ref", int(g["cg_iterations"]),
          "w", rel_diff(cg.w, g["cg_w"]), flush=True)
    m.close()
