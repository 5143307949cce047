"""Measure the rounding-sensitivity envelope of the REFERENCE's algorithm on cfg 2.

Two kinds of perturbation, identical inputs (X from the checker's own generator,
the golden labels and b):

* threads: the reference's opt-in threaded matvecs (proj/src/sparse.cpp:127-176)
  change only the floating-point summation order of X^T u; its unmodified solve
  with 1 to 8 threads;
* variants: the sequential CPU restatement (oracle/restatement.cpp, pinned bit
  for bit to the reference's sequential run) with rounding-level changes, each a
  choice the GPU makes: dot products summed as 256-wide or fully pairwise trees
  (ORC_DOT_TREE=1/2), X^T sums in row segments (ORC_XT_SEG), FMA-contracted
  vector updates (the oracle_fma build), the coarsest level applied through its
  explicit inverse (ORC_COARSE_INV), omega_k moved by +-1 ulp (ORC_OMEGA_ULP);
  for plain CG every combination of the first three, plus the GPU's own orders
  (column-popularity row sums ORC_K1_POP, per-column entry segments ORC_XT_SEGNNZ).

The spread of iteration counts and of w over these runs is the envelope two
correct implementations of the same algorithm can land in;
tests/test_gpu_parity.py holds the GPU to it at tol 1e-6 and to the strict 1e-8
bar at tol 1e-12 (SURVEY.md Appendix B protocol).

    python tests/golden/make_envelope.py [threads ...]   # writes tests/golden/envelope.json
    ENVELOPE_VARIANTS=1 python tests/golden/make_envelope.py
"""
import json
import os
import subprocess
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
sys.path.insert(0, os.path.dirname(HERE))
import oracle  # noqa: E402

CASES = (("cfg2_small", 10000, 2000, [200, 20]), ("cfg2_full", 100000, 20000, [2000, 200]), ("cnae", 0, 0, []),
         ("lpsc105", 0, 0, []))
BETA = {"cnae": 1e-6, "lpsc105": 1e-6}
VARIANTS = {  # name -> environment; ENVELOPE_LIB picks the FMA-contracted build
    "dot_tree": {"ORC_DOT_TREE": "1"},
    "coarse_inverse": {"ORC_COARSE_INV": "1"},
    "omega_plus_1ulp": {"ORC_OMEGA_ULP": "1"},
    "omega_minus_1ulp": {"ORC_OMEGA_ULP": "-1"},
    "all_gpu_choices": {"ORC_DOT_TREE": "1", "ORC_COARSE_INV": "1"},
    # the GPU's accuracy class: pairwise dot products, segmented X^T sums, FMA updates
    "gpu_accuracy_class": {"ORC_DOT_TREE": "2", "ORC_XT_SEG": "8192", "ORC_COARSE_INV": "1",
                           "ENVELOPE_LIB": "oracle_fma"},
}
# plain CG only (its ~500 iterations are cheap): every combination of the three
# accuracy choices
CG_VARIANTS = {f"cg_dot{d}_xtseg{x}_{'fma' if f else 'nofma'}": dict(
    {"ORC_DOT_TREE": str(d), "ORC_XT_SEG": str(x), "ENVELOPE_CG_ONLY": "1"}, **({"ENVELOPE_LIB": "oracle_fma"} if f else {}))
    for d in (0, 1, 2) for x in (0, 4096, 16384) for f in (0, 1) if (d, x, f) != (0, 0, 0)}
# + the GPU's own summation orders: SELL rows in column-popularity order (K1), X^T
# columns in segments of their own entries (the segmented schedule's C = nnz / 592)
CG_VARIANTS.update({f"cg_gpuorder_dot{d}_{'fma' if f else 'nofma'}{'_k1pop' if p else ''}": dict(
    {"ORC_DOT_TREE": str(d), "ORC_XT_SEGNNZ": "6757", "ORC_K1_POP": str(p), "ENVELOPE_CG_ONLY": "1"},
    **({"ENVELOPE_LIB": "oracle_fma"} if f else {})) for d in (1, 2) for f in (0, 1) for p in (0, 1)})


def rel_diff(a, b):
    return float(np.linalg.norm(np.asarray(a) - np.asarray(b)) / np.linalg.norm(b))


def setup(chk, name, n, f, ks):
    g = np.load(os.path.join(HERE, name + ".npz"))
    if name in ("cnae", "lpsc105"):  # the bundled CNAE-9 / netlib SC105 matrices, beta = 1e-6, plain CG only
        m = chk.matrix(int(g["x_shape"][0]), int(g["x_shape"][1]), g["x_row_offsets"], g["x_column_indices"],
                       g["x_values"])
        return g, m, []
    m = chk.synth_sparse_zipf(n, f, 40.0, 1.1, False, 0)
    lv = [dict(labels=g[f"labels{i}"].astype(np.int64), n_clusters=k,
               coarse_kind=oracle.COARSE_DIRECT if i == len(ks) - 1 else oracle.COARSE_INNER_FCG,
               coarse_tol=1e-6, coarse_max_iters=500) for i, k in enumerate(ks)]
    return g, m, lv


def run_variant(case):
    """child process: the restatement under the perturbation set in the environment"""
    name, n, f, ks = next(c for c in CASES if c[0] == case)
    lib = os.environ.get("ENVELOPE_LIB", "oracle")
    if not oracle.available(lib):
        oracle.build(lib)
    chk = oracle.Checker(lib)
    g, m, lv = setup(chk, name, n, f, ks)
    out = {}
    beta = BETA.get(name, 1.0)
    if not os.environ.get("ENVELOPE_CG_ONLY") and lv:
        s = chk.solve(m, beta, g["b"], "fcg_multilevel", levels=lv, tol=1e-6, max_iters=1000)
        out.update(ml_iterations=s.iterations, ml_w_rel_diff=rel_diff(s.w, g["ml_w"]))
    c = chk.solve(m, beta, g["b"], "cg", tol=1e-6, max_iters=20000)
    out.update(cg_iterations=c.iterations, cg_w_rel_diff=rel_diff(c.w, g["cg_w"]))
    print(json.dumps(out))


def summarize(e):
    runs = list(e.get("threads", {}).values()) + list(e.get("variants", {}).values())
    ml = [v for v in runs if "ml_iterations" in v]
    if not ml:
        cits = [e["cg_iterations_seq"]] + [v["cg_iterations"] for v in runs]
        e["cg_iterations_range"] = [min(cits), max(cits)]
        e["cg_iter_spread"] = max(abs(v["cg_iterations"] - e["cg_iterations_seq"]) for v in runs)
        e["cg_w_spread"] = max(v["cg_w_rel_diff"] for v in runs)
        return
    its = [e["ml_iterations_seq"]] + [v["ml_iterations"] for v in ml]
    cits = [e["cg_iterations_seq"]] + [v["cg_iterations"] for v in runs]
    e["ml_iterations_range"] = [min(its), max(its)]
    e["cg_iterations_range"] = [min(cits), max(cits)]
    e["ml_iter_spread"] = max(abs(v["ml_iterations"] - e["ml_iterations_seq"]) for v in ml)
    e["cg_iter_spread"] = max(abs(v["cg_iterations"] - e["cg_iterations_seq"]) for v in runs)
    e["ml_w_spread"] = max(v["ml_w_rel_diff"] for v in ml)
    e["cg_w_spread"] = max(v["cg_w_rel_diff"] for v in runs)


def main():
    if os.environ.get("ENVELOPE_CHILD"):
        run_variant(os.environ["ENVELOPE_CHILD"])
        return
    path = os.path.join(HERE, "envelope.json")
    out = json.load(open(path)) if os.path.exists(path) else {}
    names = os.environ.get("ENVELOPE_CASES", "cfg2_small,cfg2_full").split(",")
    for name, n, f, ks in CASES:
        if name not in names:
            continue
        g = np.load(os.path.join(HERE, name + ".npz"))
        e = out.get(name) or {"threads": {}}
        e.update({"cg_iterations_seq": int(g["cg_iterations"])})
        if "ml_iterations" in g.files:
            e["ml_iterations_seq"] = int(g["ml_iterations"])
        if os.environ.get("ENVELOPE_VARIANTS"):
            todo = dict(VARIANTS) if os.environ["ENVELOPE_VARIANTS"] != "cg" else {}
            todo.update(CG_VARIANTS)
            e.setdefault("variants", {})
            items, width = list(todo.items()), int(os.environ.get("ENVELOPE_PARALLEL", "8"))
            for i in range(0, len(items), width):
                procs = {k: subprocess.Popen([sys.executable, __file__],
                                             env={**os.environ, **v, "ENVELOPE_CHILD": name},
                                             stdout=subprocess.PIPE, text=True) for k, v in items[i:i + width]}
                for k, p in procs.items():
                    res, _ = p.communicate()
                    e["variants"][k] = json.loads(res.strip().splitlines()[-1])
                    print(name, k, e["variants"][k], flush=True)
                out[name] = e
                json.dump(out, open(path, "w"), indent=1)
        else:
            ref = oracle.Checker("ref")
            _, m, lv = setup(ref, name, n, f, ks)
            beta = BETA.get(name, 1.0)
            for th in [int(t) for t in (sys.argv[1:] or ["2", "3", "4", "5", "6", "7", "8"])]:
                ref.set_num_threads(th)
                c = ref.solve(m, beta, g["b"], "cg", tol=1e-6, max_iters=20000)
                run = {"cg_iterations": c.iterations, "cg_w_rel_diff": rel_diff(c.w, g["cg_w"])}
                if lv:
                    s = ref.solve(m, beta, g["b"], "fcg_multilevel", levels=lv, tol=1e-6, max_iters=1000)
                    run.update(ml_iterations=s.iterations, ml_w_rel_diff=rel_diff(s.w, g["ml_w"]))
                e["threads"][str(th)] = run
                print(name, th, e["threads"][str(th)], flush=True)
                out[name] = e
                json.dump(out, open(path, "w"), indent=1)
            ref.set_num_threads(1)
        summarize(e)
        out[name] = e
        json.dump(out, open(path, "w"), indent=1)


if __name__ == "__main__":
    main()
