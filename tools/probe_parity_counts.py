"""Probe: the GPU's iteration counts / w differences on the rounding-sensitive parity
cases, next to the reference goldens: lpsc105 CG and LF-52, CNAE CG,
cfg 2 small / full multilevel FCG and CG, smoke()'s small multilevel case.
usage: python tools/probe_parity_counts.py [full]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np

import oracle
import paper_1806_05826_b200 as R
from helpers import golden_matrix, load_golden, rel_diff

R.load()
dm = R.DeviceMatrix
g = load_golden("lpsc105")
m = dm(golden_matrix(g))
sol = R.solve_system(m, 1e-6, g["b"], R.MethodSpec(kind=R.CG, solver=R.SolverConfig(1e-6, 20000)))
print("lpsc105 cg:", sol.report.iterations, "ref", int(g["cg_iterations"]), "w diff", rel_diff(sol.w, g["cg_w"]))
lv = R.LevelSpec(clustering=R.ClusteringChoice(kind=R.LEADER_TARGET, target_size=56))
pm = R.PreparedMethod(m, 1e-6, R.MethodSpec(kind=R.FCG_TWOLEVEL, levels=[lv], solver=R.SolverConfig(1e-6, 5000)))
w, rep = pm.solve(g["b"])
print("lpsc105 LF-52:", rep.iterations, "ref (shim)", int(g["lf56_iterations"]), "w diff", rel_diff(w, g["lf56_w"]))
c = load_golden("cnae")
mc = dm(golden_matrix(c))
cg = R.solve_system(mc, 1e-6, c["b"], R.MethodSpec(kind=R.CG, solver=R.SolverConfig(1e-6, 20000)))
print("cnae cg:", cg.report.iterations, "ref", int(c["cg_iterations"]), "w diff", rel_diff(cg.w, c["cg_w"]))
cases = [("cfg2_small", 10000, 2000, [200, 20])]
if "full" in sys.argv[1:]:
    cases.append(("cfg2_full", 100000, 20000, [2000, 200]))
for name, n, f, ks in cases:
    gg = load_golden(name)
    x = R.synth_sparse_zipf(n, f, 40.0, 1.1, False, 0)
    mx = dm(x)
    levels = [R.LevelSpec(clustering=R.ClusteringChoice(kind=R.IMPORTED, labels=gg[f"labels{i}"].astype(np.int64),
                                                        n_clusters=k),
                          solver=R.CoarseSolveChoice(kind=R.DIRECT_CHOLESKY if i == len(ks) - 1 else R.INNER_FCG,
                                                     tol=1e-6, max_iters=500)) for i, k in enumerate(ks)]
    pm = R.PreparedMethod(mx, 1.0, R.MethodSpec(kind=R.FCG_MULTILEVEL, levels=levels,
                                                solver=R.SolverConfig(1e-6, 1000)))
    w, rep = pm.solve(gg["b"])
    print(f"{name} fcg_multilevel:", rep.iterations, "ref", int(gg["ml_iterations"]), "w diff",
          rel_diff(w, gg["ml_w"]), "omega", [pm.level(k)["omega"] for k in range(len(ks))], flush=True)
    cgr = R.solve_system(mx, 1.0, gg["b"], R.MethodSpec(kind=R.CG, solver=R.SolverConfig(1e-6, 5000)))
    print(f"{name} cg:", cgr.report.iterations, "ref", int(gg["cg_iterations"]), "w diff", rel_diff(cgr.w, gg["cg_w"]))
    pm.close()
    mx.close()
# smoke()'s multilevel case
orc = oracle.Checker("oracle")
x = R.synth_sparse_zipf(3000, 400, 20.0, 1.1, True, 11)
mx = dm(x)
om = orc.matrix(x.n_samples, x.n_features, x.row_offsets, x.column_indices, x.value_array())
b = R.rng_normals(42, x.n_samples)
levels, olevels = [], []
for i, k in enumerate([60, 12]):
    last = i == 1
    levels.append(R.LevelSpec(clustering=R.ClusteringChoice(kind=R.KMEANS, target_size=k, seed=0),
                              solver=R.CoarseSolveChoice(kind=R.DIRECT_CHOLESKY if last else R.INNER_FCG)))
    olevels.append(dict(clustering_kind=oracle.CLUSTER_KMEANS, target_size=k, seed=0,
                        coarse_kind=oracle.COARSE_DIRECT if last else oracle.COARSE_INNER_FCG))
s = R.solve_system(mx, 0.5, b, R.MethodSpec(kind=R.FCG_MULTILEVEL, levels=levels, solver=R.SolverConfig(1e-10, 500)))
ref = orc.solve(om, 0.5, b, "fcg_multilevel", levels=olevels, tol=1e-10, max_iters=500)
print("smoke fcg_multilevel:", s.report.iterations, "oracle", ref.iterations, "w diff", rel_diff(s.w, ref.w))
