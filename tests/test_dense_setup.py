"""Hierarchy setup for dense X on the device (dense_setup.cu).

A dense X created without a host CSR runs k-means (seeding distances and Lloyd
iterations), X_c = X P and the coarse Gram matrices on the GPU.  Bars: labels
and X_c values bit-identical to the oracle (the restatement pinned to the
reference build, run on the CSR of the same values); solves as elsewhere
(iterations +-2, w 1e-8 at tol 1e-10); the host-CSR setup of the same matrix
(RMG_DENSE_HOST_SETUP=1) gives the same labels.
"""
import os

import numpy as np
import pytest

import oracle
import paper_1806_05826_b200 as R
from helpers import rel_diff, to_checker

pytestmark = pytest.mark.gpu


def prepare(a, ks, normalize, beta=1e-2, seed=0, tol=1e-10, host_setup=False):
    if host_setup:
        os.environ["RMG_DENSE_HOST_SETUP"] = "1"
    try:
        m = R.DeviceMatrix.from_dense(a)
    finally:
        os.environ.pop("RMG_DENSE_HOST_SETUP", None)
    levels = []
    for i, k in enumerate(ks):
        last = i == len(ks) - 1
        levels.append(R.LevelSpec(clustering=R.ClusteringChoice(kind=R.KMEANS, target_size=k, seed=seed,
                                                                normalize_columns=normalize),
                                  solver=R.CoarseSolveChoice(kind=R.DIRECT_CHOLESKY if last else R.INNER_FCG)))
    kind = R.FCG_TWOLEVEL if len(ks) == 1 else R.FCG_MULTILEVEL
    return m, R.PreparedMethod(m, beta, R.MethodSpec(kind=kind, levels=levels, solver=R.SolverConfig(tol, 2000)))


def dense_from_csr(x: R.FeatureMatrix) -> np.ndarray:
    return x.dense()


def oracle_dense(om):
    rp, ci, v = om.export()
    out = np.zeros((om.n_samples, om.n_features))
    for r in range(om.n_samples):
        out[r, ci[rp[r]:rp[r + 1]].astype(np.int64)] = v[rp[r]:rp[r + 1]]
    return out


def matrix_with_structure(n, f, seed, fp32=False):
    """Normal entries plus the corner cases of the reference's column merge:
    an all-zero column, exact zeros, duplicated columns (zero k-means++ mass)."""
    rng = np.random.default_rng(seed)
    a = rng.standard_normal((n, f))
    a[:, 5 % f] = 0.0
    a[rng.random((n, f)) < 0.05] = 0.0
    for j in range(0, f - 1, 9):
        a[:, j + 1] = a[:, j]
    return a.astype(np.float32) if fp32 else a


@pytest.mark.parametrize("fp32", [False, True])
@pytest.mark.parametrize("normalize", [False, True])
@pytest.mark.parametrize("n,f,k", [(600, 150, 7), (600, 150, 33), (300, 150, 149), (257, 70, 40)])
def test_dense_kmeans_labels_bit_exact(gpu, orc, n, f, k, normalize, fp32):
    a = matrix_with_structure(n, f, n + f + k, fp32)
    _, pm = prepare(a, [k], normalize)
    om = to_checker(orc, R.from_dense(a.astype(np.float64)))
    want, _, _ = orc.kmeans(om, k, 100, 0, normalize=normalize)
    assert np.array_equal(pm.labels(0), want)


@pytest.mark.parametrize("normalize", [False, True])
def test_dense_three_level_matches_oracle(gpu, orc, normalize):
    """Both clusterings, X_c1 (bit-exact values) and the multilevel solve."""
    rng = np.random.default_rng(17)
    z = rng.standard_normal((1500, 30))
    a = z[:, np.arange(240) % 30] + 0.3 * rng.standard_normal((1500, 240))  # cfg 1-like groups
    _, pm = prepare(a, [48, 8], normalize)
    om = to_checker(orc, R.from_dense(a))
    lab0, _, _ = orc.kmeans(om, 48, 100, 0, normalize=normalize)
    assert np.array_equal(pm.labels(0), lab0)
    oxc = orc.coarsen(om, lab0, 48)
    assert np.array_equal(dense_from_csr(pm.level_matrix(1)), oracle_dense(oxc))
    lab1, _, _ = orc.kmeans(oxc, 8, 100, 0, normalize=normalize)
    assert np.array_equal(pm.labels(1), lab1)
    b = rng.standard_normal(1500)
    w, rep = pm.solve(b)
    levels = [dict(clustering_kind=oracle.CLUSTER_KMEANS, target_size=48, seed=0, normalize_columns=normalize,
                   coarse_kind=oracle.COARSE_INNER_FCG),
              dict(clustering_kind=oracle.CLUSTER_KMEANS, target_size=8, seed=0, normalize_columns=normalize,
                   coarse_kind=oracle.COARSE_DIRECT)]
    ref = orc.solve(om, 1e-2, b, "fcg_multilevel", levels=levels, tol=1e-10, max_iters=2000)
    assert rep.converged
    assert abs(rep.iterations - ref.iterations) <= 2
    assert rel_diff(w, ref.w) <= 1e-8


def test_dense_device_setup_equals_host_setup(gpu):
    """The same matrix through the host-CSR setup (diagnostics switch): same labels,
    same iterations, w to rounding of the coarse operators."""
    a = matrix_with_structure(800, 120, 5, fp32=True)
    b = np.random.default_rng(1).standard_normal(800)
    _, pd = prepare(a, [20, 5], True)
    _, ph = prepare(a, [20, 5], True, host_setup=True)
    for lv in (0, 1):
        assert np.array_equal(pd.labels(lv), ph.labels(lv))
    wd, rd = pd.solve(b)
    wh, rh = ph.solve(b)
    assert abs(rd.iterations - rh.iterations) <= 1
    assert rel_diff(wd, wh) <= 1e-9


@pytest.mark.parametrize("method", ["jacobi_cg", "fcg_twolevel", "fgmres_twolevel", "fcg_multilevel"])
def test_dense_device_levels_set_beta_and_methods(gpu, orc, method):
    """Every method kind on a device-resident dense hierarchy; a beta sweep over it
    (cached X_k^T X_k) equals a fresh prepare bit for bit."""
    a = matrix_with_structure(900, 96, 21, fp32=True)
    m = R.DeviceMatrix.from_dense(a)
    ks = [24, 6] if method == "fcg_multilevel" else [24] if method != "jacobi_cg" else []
    levels = [R.LevelSpec(clustering=R.ClusteringChoice(kind=R.KMEANS, target_size=k, normalize_columns=True),
                          solver=R.CoarseSolveChoice(kind=R.DIRECT_CHOLESKY if i == len(ks) - 1 else R.INNER_FCG))
              for i, k in enumerate(ks)]
    spec = R.MethodSpec(kind=R.method_from_string(method), levels=levels, solver=R.SolverConfig(1e-10, 2000))
    b = np.random.default_rng(2).standard_normal(900)
    pm = R.PreparedMethod(m, 1e-3, spec)
    om = to_checker(orc, R.from_dense(a.astype(np.float64)))
    for beta in (1e-2, 1.0):
        pm.set_beta(beta)
        w1, r1 = pm.solve(b)
        fresh = R.PreparedMethod(m, beta, spec)
        w2, r2 = fresh.solve(b)
        assert r1.iterations == r2.iterations and np.array_equal(w1, w2), (method, beta)
        olv = [dict(clustering_kind=oracle.CLUSTER_KMEANS, target_size=k, normalize_columns=True,
                    coarse_kind=oracle.COARSE_DIRECT if i == len(ks) - 1 else oracle.COARSE_INNER_FCG)
               for i, k in enumerate(ks)]
        ref = orc.solve(om, beta, b, method, levels=olv, tol=1e-10, max_iters=2000)
        assert abs(r1.iterations - ref.iterations) <= 2, (method, beta, r1.iterations, ref.iterations)
        assert rel_diff(w1, ref.w) <= 1e-8
        fresh.close()


def test_dense_device_leader_follower_and_imported(gpu, orc):
    """Clusterings without a device kernel (leader-follower) build the host CSR on
    first use; imported labels skip clustering; both match the oracle."""
    a = matrix_with_structure(400, 60, 8)
    om = to_checker(orc, R.from_dense(a))
    m = R.DeviceMatrix.from_dense(a)
    want, nc, _, _ = orc.leader_follower_target(om, 12)
    lv = R.LevelSpec(clustering=R.ClusteringChoice(kind=R.LEADER_TARGET, target_size=12),
                     solver=R.CoarseSolveChoice(kind=R.DIRECT_CHOLESKY))
    pm = R.PreparedMethod(m, 1e-2, R.MethodSpec(kind=R.FCG_TWOLEVEL, levels=[lv]))
    assert np.array_equal(pm.labels(0), want)
    lab = np.arange(60, dtype=np.int64) % 7
    lv = R.LevelSpec(clustering=R.ClusteringChoice(kind=R.IMPORTED, labels=lab, n_clusters=7),
                     solver=R.CoarseSolveChoice(kind=R.DIRECT_CHOLESKY))
    pm = R.PreparedMethod(m, 1e-2, R.MethodSpec(kind=R.FCG_TWOLEVEL, levels=[lv], solver=R.SolverConfig(1e-10, 500)))
    b = np.random.default_rng(0).standard_normal(400)
    w, rep = pm.solve(b)
    ref = orc.solve(om, 1e-2, b, "fcg_twolevel", levels=[dict(labels=lab, n_clusters=7)], tol=1e-10, max_iters=500)
    assert np.array_equal(pm.labels(0), lab)
    assert abs(rep.iterations - ref.iterations) <= 2 and rel_diff(w, ref.w) <= 1e-8
