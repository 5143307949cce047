import os, sys, time
sys.path.insert(0, os.getcwd())
import paper_1806_05826_b200 as R, bench
cfg = bench.CONFIGS["cfg2"]
x = bench.make_matrix(cfg)
m = R.DeviceMatrix(x)
t = time.time()
pm = R.PreparedMethod(m, 1.0, R.MethodSpec(kind=R.FCG_MULTILEVEL, levels=bench.level_specs(cfg), solver=R.SolverConfig(1e-6, 1000)))
print("prepare total", time.time() - t)
