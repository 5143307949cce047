"""Generate the golden fixtures under tests/golden/ from the REFERENCE build.

    python tests/golden/make_golden.py [lpsc105 cnae random cfg1 cfg2_small cfg2_full]

Every expected value here comes from oracle/_ref/libridgemg_ref.so, i.e. the
reference's own sources (/root/reference/proj/src) compiled by oracle/Makefile,
called through its public API (PreparedMethod, kmeans, leader_follower, coarsen,
estimate_lambda_max, ...).  Inputs: the two matrices bundled with the reference
(proj/data: netlib SC105 constraint matrix; UCI CNAE-9, CC BY 4.0), seeded
random matrices built like proj/tests/oracles.hpp, and the BASELINE synthetic
generators of this repo (pinned by the SHA-256 of their CSR arrays).
This script needs /root/reference and runs only in the build container.
"""
from __future__ import annotations

import hashlib
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.dirname(HERE))

import oracle  # noqa: E402
import paper_1806_05826_b200 as R  # noqa: E402
from helpers import random_matrix, to_checker  # noqa: E402

DATA = "/root/reference/proj/data"


def csr_sha(x: R.FeatureMatrix) -> str:
    h = hashlib.sha256()
    h.update(np.ascontiguousarray(x.row_offsets, np.uint64).tobytes())
    h.update(np.ascontiguousarray(x.column_indices, np.uint64).tobytes())
    h.update(np.ascontiguousarray(x.value_array(), np.float64).tobytes())
    return h.hexdigest()


def pack_matrix(out: dict, x: R.FeatureMatrix, prefix="x"):
    out[prefix + "_shape"] = np.array([x.n_samples, x.n_features], np.int64)
    out[prefix + "_row_offsets"] = x.row_offsets.astype(np.int64)
    out[prefix + "_column_indices"] = x.column_indices.astype(np.int32)
    if x.values is not None:
        out[prefix + "_values"] = x.values


def from_ref_matrix(m) -> R.FeatureMatrix:
    rp, ci, v = m.export()
    return R.FeatureMatrix(m.n_samples, m.n_features, rp, ci, v)


def solve_pack(out, key, ref, m, beta, b, method, levels=(), tol=1e-6, max_iters=1000):
    t = time.time()
    s = ref.solve(m, beta, b, method, levels=levels, tol=tol, max_iters=max_iters)
    out[key + "_iterations"] = np.int64(s.iterations)
    out[key + "_converged"] = np.int64(s.converged)
    out[key + "_w"] = s.w
    out[key + "_hist"] = s.residual_history
    if len(s.inner_iterations):
        out[key + "_inner"] = s.inner_iterations.astype(np.int64)
    if s.omega:
        out[key + "_omega"] = np.array(s.omega)
    print(f"  {key}: {s.iterations} iterations, converged={s.converged}, {time.time() - t:.1f}s", flush=True)
    return s


def save(name, out):
    np.savez_compressed(os.path.join(HERE, name + ".npz"), **out)
    print("wrote", name, flush=True)


def make_lpsc105(ref):
    out = {}
    m = ref.read_matrix_market(os.path.join(DATA, "lpsc105.mtx"))
    x = from_ref_matrix(m)
    pack_matrix(out, x)
    b, rhs = ref.generate_rhs(m, 42)
    out["b"], out["rhs"] = b, rhs
    beta = 1e-6
    solve_pack(out, "cg", ref, m, beta, b, "cg", tol=1e-6, max_iters=20000)
    for target in (134, 56):
        lab, nc, exact, tol = ref.leader_follower_target(m, target)
        out[f"lf{target}_labels"], out[f"lf{target}_nc"] = lab, np.int64(nc)
        out[f"lf{target}_exact"], out[f"lf{target}_tol"] = np.int64(exact), np.float64(tol)
        solve_pack(out, f"lf{target}", ref, m, beta, b, "fcg_twolevel",
                   levels=[dict(labels=lab, n_clusters=nc)], tol=1e-6, max_iters=5000)
    w = ref.normals(5, x.n_features)
    out["apply_w"] = w
    out["apply_out"] = ref.ridge_apply(m, beta, w)
    out["gram_diag"] = ref.gram_diagonal(m, beta)
    lam, it, cv = ref.lambda_max(m, 1e-4, 200, 0x5EED)
    out["lambda"], out["lambda_iters"] = np.float64(lam), np.int64(it)
    save("lpsc105", out)


def make_cnae(ref):
    out = {}
    m = ref.read_matrix_market(os.path.join(DATA, "cnae.mtx"))
    x = from_ref_matrix(m)
    pack_matrix(out, x)
    b, rhs = ref.generate_rhs(m, 42)
    out["b"] = b
    lab, nc = ref.leader_follower(m, 0.5)
    out["lf_labels"], out["lf_nc"] = lab, np.int64(nc)
    solve_pack(out, "lf", ref, m, 1e-6, b, "fcg_twolevel", levels=[dict(labels=lab, n_clusters=nc)],
               tol=1e-6, max_iters=5000)
    solve_pack(out, "cg", ref, m, 1e-6, b, "cg", tol=1e-6, max_iters=20000)
    save("cnae", out)


RANDOM_CASES = [  # (rows, cols, seed, fill, beta, k)  shapes from proj/tests/test_krylov.cpp
    (20, 20, 1234, 0.6, 0.5, 6),
    (24, 18, 1357, 0.5, 1e-3, 6),
    (40, 32, 2468, 0.4, 1e-4, 16),
    (30, 12, 8080, 0.7, 1e-6, 4),
    (120, 60, 77, 0.3, 1e-2, 12),
]


def make_random(ref):
    out = {}
    for i, (rows, cols, seed, fill, beta, k) in enumerate(RANDOM_CASES):
        x = random_matrix(rows, cols, seed, fill)
        m = to_checker(ref, x)
        p = f"r{i}"
        pack_matrix(out, x, p)
        v = ref.normals(seed + 1, cols)
        u = ref.normals(seed + 2, rows)
        out[p + "_v"], out[p + "_u"] = v, u
        out[p + "_spmv"] = ref.spmv(m, v)
        out[p + "_spmv_t"] = ref.spmv_transpose(m, u)
        out[p + "_ridge"] = ref.ridge_apply(m, beta, v)
        out[p + "_diag"] = ref.gram_diagonal(m, beta)
        lam, it, _ = ref.lambda_max(m, 1e-4, 200, 0x5EED)
        out[p + "_lambda"], out[p + "_lambda_iters"] = np.float64(lam), np.int64(it)
        out[p + "_kpp"] = ref.kmeanspp_seed(m, k, 3)
        lab, iters, _ = ref.kmeans(m, k, 100, 0)
        out[p + "_km_labels"] = lab
        xc = from_ref_matrix(ref.coarsen(m, lab, k, beta))
        pack_matrix(out, xc, p + "_xc")
        out[p + "_z"] = ref.two_level_apply(m, beta, lab, k, 0.37, v)
        b, _ = ref.generate_rhs(m, seed % 97)
        out[p + "_b"] = b
        out[p + "_beta"] = np.float64(beta)
        lv1 = dict(clustering_kind=oracle.CLUSTER_KMEANS, target_size=k)
        for meth in ("cg", "jacobi_cg", "fcg_twolevel"):
            solve_pack(out, f"{p}_{meth}", ref, m, beta, b, meth, levels=[lv1], tol=1e-8, max_iters=2000)
        if k >= 8:
            mid = dict(clustering_kind=oracle.CLUSTER_KMEANS, target_size=k,
                       coarse_kind=oracle.COARSE_INNER_FCG, coarse_tol=1e-6)
            last = dict(clustering_kind=oracle.CLUSTER_KMEANS, target_size=k // 2)
            solve_pack(out, f"{p}_fcg_multilevel", ref, m, beta, b, "fcg_multilevel", levels=[mid, last],
                       tol=1e-8, max_iters=400)
    save("random", out)


def cfg_levels(ks, normalize, inner="fcg"):
    lv = []
    for i, k in enumerate(ks):
        last = i == len(ks) - 1
        lv.append(dict(clustering_kind=oracle.CLUSTER_KMEANS, target_size=k, seed=0, kmeans_max_iters=100,
                       normalize_columns=normalize,
                       coarse_kind=oracle.COARSE_DIRECT if last else
                       (oracle.COARSE_INNER_FCG if inner == "fcg" else oracle.COARSE_INNER_CG),
                       coarse_tol=1e-6, coarse_max_iters=500))
    return lv


def level_labels(chk, m, ks, normalize):
    """Labels of every level, computed like build_hierarchy: cluster, coarsen, repeat."""
    labels, cur = [], m
    for k in ks:
        lab, it, cv = chk.kmeans(cur, k, 100, 0, normalize=normalize)
        print(f"  kmeans k={k}: {it} Lloyd iterations (converged={cv})", flush=True)
        labels.append(lab)
        cur = chk.coarsen(cur, lab, k)
    return labels


def make_cfg1(ref):
    out = {}
    x = R.synth_dense_clustered(2000, 500, 50, 0.1, 0)
    out["sha256"] = np.array(csr_sha(x))
    m = to_checker(ref, x)
    b = ref.normals(42, x.n_samples)
    out["b"] = b
    labels = level_labels(ref, m, [50], False)
    out["labels0"] = labels[0]
    lv = [dict(labels=labels[0], n_clusters=50)]
    solve_pack(out, "fcg", ref, m, 1e-2, b, "fcg_twolevel", levels=lv)
    solve_pack(out, "cg", ref, m, 1e-2, b, "cg")
    solve_pack(out, "fcg12", ref, m, 1e-2, b, "fcg_twolevel", levels=lv, tol=1e-12)
    save("cfg1", out)


def make_cfg2(ref, name, n, f, ks, chk_labels=None):
    out = {}
    x = R.synth_sparse_zipf(n, f, 40.0, 1.1, False, 0)
    out["sha256"] = np.array(csr_sha(x))
    out["shape"] = np.array([n, f, x.nnz])
    m = to_checker(ref, x)
    b = ref.normals(42, n)
    out["b"] = b
    labels = level_labels(chk_labels or ref, to_checker(chk_labels, x) if chk_labels else m, ks, True)
    for i, lab in enumerate(labels):
        out[f"labels{i}"] = lab.astype(np.int32)
    lv = cfg_levels(ks, True)
    for i, l in enumerate(lv):
        l["labels"], l["n_clusters"] = labels[i], ks[i]
    solve_pack(out, "ml", ref, m, 1.0, b, "fcg_multilevel", levels=lv)
    solve_pack(out, "cg", ref, m, 1.0, b, "cg")
    # the same solves driven to tol 1e-12, where w parity is sharp
    solve_pack(out, "ml12", ref, m, 1.0, b, "fcg_multilevel", levels=lv, tol=1e-12)
    solve_pack(out, "cg12", ref, m, 1.0, b, "cg", tol=1e-12, max_iters=5000)
    save(name, out)


if __name__ == "__main__":
    which = sys.argv[1:] or ["lpsc105", "cnae", "random", "cfg1", "cfg2_small"]
    ref = oracle.Checker("ref")
    for w in which:
        print("==", w, flush=True)
        if w == "lpsc105":
            make_lpsc105(ref)
        elif w == "cnae":
            make_cnae(ref)
        elif w == "random":
            make_random(ref)
        elif w == "cfg1":
            make_cfg1(ref)
        elif w == "cfg2_small":
            make_cfg2(ref, "cfg2_small", 10000, 2000, [200, 20])
        elif w == "cfg2_full":
            # labels from this repo's oracle restatement (threaded; the verbatim
            # reference k-means takes hours at this size) - tests/test_oracle_pin.py
            # pins oracle == reference labels on cfg2_small; the solve is the reference's.
            orc = oracle.Checker("oracle")
            orc.set_num_threads(os.cpu_count() or 8)
            make_cfg2(ref, "cfg2_full", 100000, 20000, [2000, 200], chk_labels=orc)
