"""Generate the cfg 3 reference fixture (run once in the build container, ~1 h on 8 cores).

    python tests/golden/make_cfg3_ref.py

BASELINE cfg 3's system (1 M x 100 k, nnz/row max(1, Poisson(50)), Zipf(1.1),
|N(0,1)| values; generator oracle/synth.hpp on the reference's own CounterRng,
one stream per row; SHA-256 of the CSR recorded), solved by the reference's own
solvers (oracle/_ref: the unmodified reference sources, PreparedMethod,
krylov.cpp:617-668) with b = normals(42):

* `jacobi_cg` (krylov.cpp:94-157 with JacobiPreconditioner :41-47) -- the
  reference's fastest method on this system (19 iterations; its multilevel FCG
  needs > 1000 outer iterations here):
  - tol 1e-6, every beta of the sweep, sequential (threads = 1, the
    reference's bitwise-deterministic default) and with 8 threads: iteration
    counts (the GPU is held to +-2) and the reference timer per iteration;
  - tol 1e-12 at beta = 10, 1, 1e-3: the solution w (tests/test_cfg3_parity.py
    holds the GPU's jacobi_cg and pcg_vcycle solutions to 1e-8 of it);
* plain `cg`, tol 1e-6, every beta, threads = 1 and 8: iteration counts.  At
  ~1700 iterations plain CG is rounding-chaotic: the two thread counts of the
  reference itself disagree by tens of iterations (the envelope the GPU's
  count is reported against), and tol 1e-12 at beta = 10 gives w.

Writes tests/golden/cfg3_ref.json and tests/golden/cfg3_ref_w.npz (resumable).
"""
from __future__ import annotations

import hashlib
import json
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
import oracle  # noqa: E402

CFG3 = dict(n=1_000_000, f=100_000, mean=50.0, zipf=1.1, values=True, seed=0)
BETAS = [10.0, 1.0, 0.1, 0.01, 0.001]
OUT_JSON = os.path.join(HERE, "cfg3_ref.json")
OUT_W = os.path.join(HERE, "cfg3_ref_w.npz")


def csr_sha(m):
    rp, ci, v = m.export()
    h = hashlib.sha256()
    h.update(rp.tobytes())
    h.update(ci.tobytes())
    h.update(v.tobytes())
    return h.hexdigest()


def main():
    res = json.load(open(OUT_JSON)) if os.path.exists(OUT_JSON) else {}
    ws = dict(np.load(OUT_W)) if os.path.exists(OUT_W) else {}
    c = oracle.Checker("ref")
    c.set_num_threads(os.cpu_count() or 1)
    m = c.synth_sparse_zipf(CFG3["n"], CFG3["f"], CFG3["mean"], CFG3["zipf"], CFG3["values"], CFG3["seed"],
                            row_streams=True)
    if "sha256" not in res:
        res.update(dict(config=CFG3, nnz=m.nnz, sha256=csr_sha(m), rhs_seed=42,
                        checker="oracle/_ref (reference sources compiled verbatim, oracle/Makefile)",
                        host_cpus=os.cpu_count()))
    b = c.normals(42, m.n_samples)

    def save():
        json.dump(res, open(OUT_JSON, "w"), indent=1)
        np.savez_compressed(OUT_W, **ws)

    def run(method, threads, tol, beta, keep_w=False):
        key = f"{method}/threads{threads}/tol{tol:g}"
        sub = res.setdefault(key, {})
        bk = f"{beta:g}"
        if bk in sub and (not keep_w or f"{method}_tol{tol:g}_beta{bk}" in ws):
            return
        c.set_num_threads(threads)
        t = time.time()
        s = c.solve(m, beta, b, method, tol=tol, max_iters=400_000)
        sub[bk] = dict(iterations=int(s.iterations), converged=bool(s.converged), wall_time_s=float(s.wall_time_s),
                       wall_total_s=time.time() - t, ms_per_iteration=1e3 * s.wall_time_s / max(1, s.iterations),
                       w_norm=float(np.linalg.norm(s.w)),
                       final_residual=float(s.residual_history[-1]) if len(s.residual_history) else None)
        if keep_w:
            ws[f"{method}_tol{tol:g}_beta{bk}"] = s.w
        print(key, bk, sub[bk], flush=True)
        save()

    for threads in (1, 8):
        for beta in BETAS:
            run("jacobi_cg", threads, 1e-6, beta)
    for beta in (10.0, 1.0, 0.001):
        run("jacobi_cg", 1, 1e-12, beta, keep_w=True)
    for threads in (8, 1):
        for beta in BETAS:
            run("cg", threads, 1e-6, beta)
    run("cg", 8, 1e-12, 10.0, keep_w=True)
    save()


if __name__ == "__main__":
    main()
