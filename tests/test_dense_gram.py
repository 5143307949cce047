"""Dense Gram matrices of coarse levels and the batched plain /
Jacobi CG.

* G_k = X_k^T X_k assembled on the device must be bit-identical to the host
  restatement of the reference's coarse Gram (krylov.cpp:350-365): prepared
  methods built with RMG_HOST_GRAM=1 (host sums) and without (device sums) give
  bitwise-equal solves -- the coarsest Cholesky and the dense inner levels are
  formed from it.
* pcg_vcycle applying dense G_k (the default where it is fewer bytes than the
  X_k sweeps) equals the sweep path (RMG_VC_DENSE=0) to rounding: iterations
  +-1 and both at the reference's solution (oracle CG to 1e-12) to 1e-8.
* rmg_method_solve_batch with cg / jacobi_cg runs the k columns in lock step
  over the block operator: each column equals its single-RHS solve (iterations
  +-5% -- plain CG at ~200 iterations is rounding-chaotic -- w 1e-8 at tol 1e-10), the reference's solution (1e-12) to 1e-8 and, for
  jacobi_cg, the reference's own iteration count at tol 1e-6 +-2."""
import os

import numpy as np
import pytest

import paper_1806_05826_b200 as R
from helpers import rel_diff, to_checker

pytestmark = pytest.mark.gpu


def levels(ks):
    return [R.LevelSpec(clustering=R.ClusteringChoice(kind=R.KMEANS, target_size=k, seed=0),
                        solver=R.CoarseSolveChoice(kind=R.DIRECT_CHOLESKY if i == len(ks) - 1 else R.INNER_FCG))
            for i, k in enumerate(ks)]


def with_env(name, value, fn):
    old = os.environ.get(name)
    os.environ[name] = value
    try:
        return fn()
    finally:
        if old is None:
            os.environ.pop(name)
        else:
            os.environ[name] = old


@pytest.mark.parametrize("values", [True, False])
def test_device_gram_bit_identical_to_host_gram(gpu, values):
    x = R.synth_sparse_zipf(3000, 500, 20.0, 1.1, values, 5)
    m = R.DeviceMatrix(x)
    b = R.rng_normals(42, x.n_samples)
    spec = R.MethodSpec(kind=R.FCG_MULTILEVEL, levels=levels([60, 12]), solver=R.SolverConfig(1e-10, 500))

    def run():
        pm = R.PreparedMethod(m, 0.5, spec)
        w, rep = pm.solve(b)
        pm.close()
        return w, rep

    w_dev, r_dev = run()
    w_host, r_host = with_env("RMG_HOST_GRAM", "1", run)
    assert r_dev.iterations == r_host.iterations
    assert np.array_equal(w_dev, w_host)


@pytest.mark.parametrize("ks", [[80, 12], [120, 30, 6]])
def test_vcycle_dense_levels_match_sweeps(gpu, orc, ks):
    x = R.synth_sparse_zipf(4000, 700, 20.0, 1.1, True, 7)
    m = R.DeviceMatrix(x)
    b = R.rng_normals(42, x.n_samples)
    spec = R.MethodSpec(kind=R.PCG_VCYCLE, levels=levels(ks), solver=R.SolverConfig(1e-10, 2000))

    def run():
        pm = R.PreparedMethod(m, 0.5, spec)
        w, rep = pm.solve(b)
        B = np.stack([R.rng_normals(100 + q, x.n_samples) for q in range(4)], axis=1)
        W, reps = pm.solve_batch(B)
        pm.close()
        return w, rep, W, reps

    w_d, r_d, W_d, rs_d = run()
    w_s, r_s, W_s, rs_s = with_env("RMG_VC_DENSE", "0", run)
    assert r_d.converged and abs(r_d.iterations - r_s.iterations) <= 1
    ref = orc.solve(to_checker(orc, x), 0.5, b, "cg", tol=1e-12, max_iters=5000)
    assert rel_diff(w_d, ref.w) <= 1e-8 and rel_diff(w_s, ref.w) <= 1e-8
    for q in range(4):
        assert rs_d[q].converged and abs(rs_d[q].iterations - rs_s[q].iterations) <= 1
        assert rel_diff(W_d[:, q], W_s[:, q]) <= 1e-8


@pytest.mark.parametrize("method", ["cg", "jacobi_cg"])
def test_batched_cg_equals_single_and_reference(gpu, ref, method):
    x = R.synth_sparse_zipf(5000, 800, 25.0, 1.1, True, 9)
    m = R.DeviceMatrix(x)
    k = 16
    B = np.stack([R.rng_normals(42 + q, x.n_samples) for q in range(k)], axis=1)
    B[:, 1] *= 1e-3
    om = to_checker(ref, x)
    # tol 1e-10: the block operator sums in another order (~1e-16), so columns equal
    # their single-RHS solves to the solve's own accuracy
    pm = R.PreparedMethod(m, 0.1, R.MethodSpec(kind=R.method_from_string(method),
                                               solver=R.SolverConfig(1e-10, 20000)))
    W, reps = pm.solve_batch(B)
    for q in range(k):
        w1, r1 = pm.solve(B[:, q])
        assert reps[q].converged and abs(reps[q].iterations - r1.iterations) <= max(2, r1.iterations // 20), (
            q, reps[q].iterations, r1.iterations)
        assert rel_diff(W[:, q], w1) <= 1e-8
    for q in range(2):
        s = ref.solve(om, 0.1, B[:, q], "cg", tol=1e-12, max_iters=20000)
        assert rel_diff(W[:, q], s.w) <= 1e-8
    # the reference's own iteration count at the config tolerance: +-2 for the
    # Jacobi-preconditioned solve (plain CG's hundreds of iterations are rounding
    # chaotic)
    if method == "jacobi_cg":
        pm6 = R.PreparedMethod(m, 0.1, R.MethodSpec(kind=R.JACOBI_CG, solver=R.SolverConfig(1e-6, 20000)))
        W6, reps6 = pm6.solve_batch(B)
        for q in range(3):
            s = ref.solve(om, 0.1, B[:, q], method, tol=1e-6, max_iters=20000)
            assert abs(reps6[q].iterations - s.iterations) <= 2, (q, reps6[q].iterations, s.iterations)


def _level_arrays(pm, k):
    x = pm.level_matrix(k)
    return x.row_offsets.copy(), x.column_indices.copy(), x.values.copy()


@pytest.mark.parametrize("case", ["zipf_values", "zipf_pattern", "signed_cancel"])
def test_device_coarsen_bit_identical_to_host(gpu, case):
    """X_c = X P on the device (k_coarsen_rows) equals the host restatement of
    coarsening.cpp:112-148 bit for bit: same coarse columns (ascending), same values
    (products summed from 0.0 in fine-column order), explicit zeros from exact
    cancellation kept."""
    if case == "signed_cancel":
        # features 2j and 2j + 1 share a cluster with weight 1/sqrt(2); rows hold +v / -v pairs
        rng = np.random.default_rng(3)
        n, f = 400, 60
        rows, cols, vals = [], [], []
        for r in range(n):
            for j in rng.choice(f // 2, 5, replace=False):
                v = float(rng.standard_normal())
                rows += [r, r]
                cols += [2 * j, 2 * j + 1]
                vals += [v, -v if r % 3 == 0 else 0.5 * v]
        x = R.csr_from_triplets(n, f, rows, cols, vals)
        labels = [np.arange(f) // 2, np.arange(f // 2) // 5]
        ks = [f // 2, f // 10]
        lv = [R.LevelSpec(clustering=R.ClusteringChoice(kind=R.IMPORTED, labels=labels[i], n_clusters=k),
                          solver=R.CoarseSolveChoice(kind=R.DIRECT_CHOLESKY if i == 1 else R.INNER_FCG))
              for i, k in enumerate(ks)]
    else:
        x = R.synth_sparse_zipf(4000, 600, 20.0, 1.1, case == "zipf_values", 4)
        lv = levels([70, 9])
    m = R.DeviceMatrix(x)
    spec = R.MethodSpec(kind=R.FCG_MULTILEVEL, levels=lv, solver=R.SolverConfig(1e-10, 500))

    def run():
        pm = R.PreparedMethod(m, 0.5, spec)
        out = [_level_arrays(pm, k) for k in (1, 2)]
        w, rep = pm.solve(R.rng_normals(42, x.n_samples))
        pm.close()
        return out, w, rep

    dev, w_dev, r_dev = run()
    host, w_host, r_host = with_env("RMG_HOST_COARSEN", "1", run)
    for (a, b) in zip(dev, host):
        for u, v in zip(a, b):
            assert np.array_equal(u, v)
    if case == "signed_cancel":
        assert np.any(dev[0][2] == 0.0)  # the cancelled entries are stored
    assert r_dev.iterations == r_host.iterations and np.array_equal(w_dev, w_host)
