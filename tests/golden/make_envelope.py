"""Measure the REFERENCE's own rounding-sensitivity envelope on cfg 2.

The reference's opt-in threaded matvecs (proj/src/sparse.cpp:127-176) change
only the floating-point summation order.  Running its unmodified solve with
1 to 16 threads on identical inputs shows how far two correct
implementations of the same algorithm drift apart on these workloads
(iterations, relative L2 difference of w).  tests/test_gpu_parity.py bounds
the GPU's deviation by this envelope at tol 1e-6, and by the strict 1e-8 bar
at tol 1e-12 (SURVEY.md Appendix B protocol).

    python tests/golden/make_envelope.py   # writes tests/golden/envelope.json
"""
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
sys.path.insert(0, os.path.dirname(HERE))
import oracle  # noqa: E402
import paper_1806_05826_b200 as R  # noqa: E402
from helpers import rel_diff  # noqa: E402

path = os.path.join(HERE, "envelope.json")
out = json.load(open(path)) if os.path.exists(path) else {}
names = os.environ.get("ENVELOPE_CASES", "cfg2_small,cfg2_full").split(",")
ref = oracle.Checker("ref")
for name, n, f, ks in (("cfg2_small", 10000, 2000, [200, 20]), ("cfg2_full", 100000, 20000, [2000, 200])):
    if name not in names:
        continue
    g = np.load(os.path.join(HERE, name + ".npz"))
    x = R.synth_sparse_zipf(n, f, 40.0, 1.1, False, 0)
    m = ref.matrix(x.n_samples, x.n_features, x.row_offsets, x.column_indices, x.value_array())
    lv = [dict(labels=g[f"labels{i}"].astype(np.int64), n_clusters=k,
               coarse_kind=oracle.COARSE_DIRECT if i == len(ks) - 1 else oracle.COARSE_INNER_FCG,
               coarse_tol=1e-6, coarse_max_iters=500) for i, k in enumerate(ks)]
    e = out.get(name) or {"threads": {}}
    e.update({"ml_iterations_seq": int(g["ml_iterations"]), "cg_iterations_seq": int(g["cg_iterations"])})
    for th in [int(t) for t in (sys.argv[1:] or ["2", "3", "4", "5", "6", "7", "8"])]:
        ref.set_num_threads(th)
        s = ref.solve(m, 1.0, g["b"], "fcg_multilevel", levels=lv, tol=1e-6, max_iters=1000)
        c = ref.solve(m, 1.0, g["b"], "cg", tol=1e-6, max_iters=5000)
        e["threads"][str(th)] = {"ml_iterations": s.iterations, "ml_w_rel_diff": rel_diff(s.w, g["ml_w"]),
                                 "cg_iterations": c.iterations, "cg_w_rel_diff": rel_diff(c.w, g["cg_w"])}
        print(name, th, e["threads"][str(th)], flush=True)
        out[name] = e
        json.dump(out, open(path, "w"), indent=1)
    t = e["threads"].values()
    its = [e["ml_iterations_seq"]] + [v["ml_iterations"] for v in t]
    e["ml_iterations_range"] = [min(its), max(its)]
    cits = [e["cg_iterations_seq"]] + [v["cg_iterations"] for v in t]
    e["cg_iterations_range"] = [min(cits), max(cits)]
    e["ml_iter_spread"] = max(abs(v["ml_iterations"] - e["ml_iterations_seq"]) for v in t)
    e["cg_iter_spread"] = max(abs(v["cg_iterations"] - e["cg_iterations_seq"]) for v in t)
    e["ml_w_spread"] = max(v["ml_w_rel_diff"] for v in t)
    e["cg_w_spread"] = max(v["cg_w_rel_diff"] for v in t)
    out[name] = e
    ref.set_num_threads(1)
json.dump(out, open(path, "w"), indent=1)
