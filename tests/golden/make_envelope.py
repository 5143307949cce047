"""Measure the rounding-sensitivity envelope of the REFERENCE's algorithm on cfg 2.

Two kinds of perturbation, identical inputs (X from the checker's own generator,
the golden labels and b):

* threads: the reference's opt-in threaded matvecs (proj/src/sparse.cpp:127-176)
  change only the floating-point summation order of X^T u; its unmodified solve
  with 1 to 8 threads;
* variants: the sequential CPU restatement (oracle/restatement.cpp, pinned bit
  for bit to the reference's sequential run) with one rounding-level change at a
  time, each a choice the GPU makes: dot products summed as 256-wide pairwise
  trees (ORC_DOT_TREE), the coarsest level applied through its explicit inverse
  (ORC_COARSE_INV), omega_k moved by +-1 ulp (ORC_OMEGA_ULP) -- and all together.

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

CASES = (("cfg2_small", 10000, 2000, [200, 20]), ("cfg2_full", 100000, 20000, [2000, 200]))
VARIANTS = {
    "dot_tree": {"ORC_DOT_TREE": "1"},
    "coarse_inverse": {"ORC_COARSE_INV": "1"},
    "omega_plus_1ulp": {"ORC_OMEGA_ULP": "1"},
    "omega_minus_1ulp": {"ORC_OMEGA_ULP": "-1"},
    "all_gpu_choices": {"ORC_DOT_TREE": "1", "ORC_COARSE_INV": "1"},
}


def rel_diff(a, b):
    return float(np.linalg.norm(np.asarray(a) - np.asarray(b)) / np.linalg.norm(b))


def setup(chk, name, n, f, ks):
    g = np.load(os.path.join(HERE, name + ".npz"))
    m = chk.synth_sparse_zipf(n, f, 40.0, 1.1, False, 0)
    lv = [dict(labels=g[f"labels{i}"].astype(np.int64), n_clusters=k,
               coarse_kind=oracle.COARSE_DIRECT if i == len(ks) - 1 else oracle.COARSE_INNER_FCG,
               coarse_tol=1e-6, coarse_max_iters=500) for i, k in enumerate(ks)]
    return g, m, lv


def run_variant(case):
    """child process: the restatement under the perturbation set in the environment"""
    name, n, f, ks = next(c for c in CASES if c[0] == case)
    chk = oracle.Checker("oracle")
    g, m, lv = setup(chk, name, n, f, ks)
    s = chk.solve(m, 1.0, g["b"], "fcg_multilevel", levels=lv, tol=1e-6, max_iters=1000)
    c = chk.solve(m, 1.0, g["b"], "cg", tol=1e-6, max_iters=5000)
    print(json.dumps({"ml_iterations": s.iterations, "ml_w_rel_diff": rel_diff(s.w, g["ml_w"]),
                      "cg_iterations": c.iterations, "cg_w_rel_diff": rel_diff(c.w, g["cg_w"])}))


def summarize(e):
    runs = list(e.get("threads", {}).values()) + list(e.get("variants", {}).values())
    its = [e["ml_iterations_seq"]] + [v["ml_iterations"] for v in runs]
    cits = [e["cg_iterations_seq"]] + [v["cg_iterations"] for v in runs]
    e["ml_iterations_range"] = [min(its), max(its)]
    e["cg_iterations_range"] = [min(cits), max(cits)]
    e["ml_iter_spread"] = max(abs(v["ml_iterations"] - e["ml_iterations_seq"]) for v in runs)
    e["cg_iter_spread"] = max(abs(v["cg_iterations"] - e["cg_iterations_seq"]) for v in runs)
    e["ml_w_spread"] = max(v["ml_w_rel_diff"] for v in runs)
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
        e.update({"ml_iterations_seq": int(g["ml_iterations"]), "cg_iterations_seq": int(g["cg_iterations"])})
        if os.environ.get("ENVELOPE_VARIANTS"):
            procs = {k: subprocess.Popen([sys.executable, __file__], env={**os.environ, **v, "ENVELOPE_CHILD": name},
                                         stdout=subprocess.PIPE, text=True) for k, v in VARIANTS.items()}
            e.setdefault("variants", {})
            for k, p in procs.items():
                res, _ = p.communicate()
                e["variants"][k] = json.loads(res.strip().splitlines()[-1])
                print(name, k, e["variants"][k], flush=True)
        else:
            ref = oracle.Checker("ref")
            _, m, lv = setup(ref, name, n, f, ks)
            for th in [int(t) for t in (sys.argv[1:] or ["2", "3", "4", "5", "6", "7", "8"])]:
                ref.set_num_threads(th)
                s = ref.solve(m, 1.0, g["b"], "fcg_multilevel", levels=lv, tol=1e-6, max_iters=1000)
                c = ref.solve(m, 1.0, g["b"], "cg", tol=1e-6, max_iters=5000)
                e["threads"][str(th)] = {"ml_iterations": s.iterations, "ml_w_rel_diff": rel_diff(s.w, g["ml_w"]),
                                         "cg_iterations": c.iterations, "cg_w_rel_diff": rel_diff(c.w, g["cg_w"])}
                print(name, th, e["threads"][str(th)], flush=True)
                out[name] = e
                json.dump(out, open(path, "w"), indent=1)
            ref.set_num_threads(1)
        summarize(e)
        out[name] = e
        json.dump(out, open(path, "w"), indent=1)


if __name__ == "__main__":
    main()
