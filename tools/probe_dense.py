"""Probe: time the cfg2 persistent inner solve in situ (one solve)."""
import sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_1806_05826_b200 as R
import bench
cfg = bench.CONFIGS["cfg2"]
x = bench.make_matrix(cfg)
m = R.DeviceMatrix(x)
labels = bench.load_golden_labels(cfg)
pm = R.PreparedMethod(m, 1.0, R.MethodSpec(kind=R.FCG_MULTILEVEL, levels=bench.level_specs(cfg, labels),
                                           solver=R.SolverConfig(1e-6, int(sys.argv[1]) if len(sys.argv) > 1 else 20)))
b = R.rng_normals(42, x.n_samples)
pm.set_profiling(True)
t = time.time(); w, rep = pm.solve(b); el = time.time() - t
print("outer", rep.iterations, "inner mean", np.mean(rep.inner_iterations), "wall", el)
for lv in range(pm.n_levels):
    print("level", lv, pm.profile(lv))
if os.environ.get("RMG_DENSE_TIMING"):
    import ctypes as C
    buf = (C.c_ulonglong * 512)()
    lib = R.load()
    lib.rmg_debug_dense_timing.argtypes = [C.c_void_p, C.c_uint64, C.c_void_p]
    if lib.rmg_debug_dense_timing(pm.h, 1, buf) == 0:
        t = np.array(buf[:256], dtype=np.float64).reshape(16, 16)
        if os.environ.get("RMG_DENSE_4B"):
            names = ["start", "z(Mr)", "GSdots", "B1", "gsums", "p", "B2", "Ap", "pap", "B3", "gsums2", "upd", "B4", "gsums3"]
        else:  # two-barrier kernel (k_dense_krylov2): marks 0..7, then the next iteration's 0
            names = ["start", "pap sums+upd", "S, z", "publish", "B1", "loads+sums", "A z", "p, Ap, publish"]
        nm_ = len(names)
        rows = t[4:15]  # iterations 4..14 (all phases present)
        nxt = t[5:16, 0:1]
        deltas = np.diff(np.concatenate([rows[:, :nm_], nxt], axis=1), axis=1)
        for i, nm in enumerate(names[1:] + ["B3/B4 -> next"]):
            print(f"  phase {nm:>15}: {np.mean(deltas[:, i]) / 1e3:7.3f} us")
        print("  iteration:", np.mean(np.diff(rows[:, 0])) / 1e3, "us")
        arr = np.array(buf[256:512], dtype=np.float64)
        arr = arr[arr > 0]
        if len(arr):
            rel = (arr - arr.min()) / 1e3
            order = np.argsort(rel)
            print(f"  per-CTA Ap end (it 8): spread {rel.max():.2f} us; slowest CTAs {order[-8:].tolist()} "
                  f"({np.round(rel[order[-8:]], 2).tolist()} us); fastest {order[:4].tolist()}")
            print("  per-CTA lateness histogram (us):", np.histogram(rel, bins=8)[0].tolist(),
                  np.round(np.histogram(rel, bins=8)[1], 2).tolist())
n, k1, k2 = pm.profile(1)
if n:
    print("dense inner solve: %.3f ms per launch, %.2f us per inner iteration" % (k1 / n, k1 / n / np.mean(rep.inner_iterations) * 1e3))
