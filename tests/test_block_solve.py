"""Batched pcg_vcycle (BASELINE cfg 3's "16 right-hand sides solved
as a batched block operator"): rmg_method_solve_batch runs the k columns in lock
step over the block operator.  Each column must equal its single-RHS solve (same
iterations +-1 -- the block operator sums in another order, ~1e-16 -- and w to
1e-10 at tol 1e-10), finished columns must freeze, and the reference's solution of
each system (oracle CG to 1e-12) must be met to 1e-8."""
import os

import numpy as np
import pytest

import paper_1806_05826_b200 as R
from helpers import random_matrix, rel_diff, to_checker

pytestmark = pytest.mark.gpu


def vspec(ks, tol=1e-10):
    levels = [R.LevelSpec(clustering=R.ClusteringChoice(kind=R.KMEANS, target_size=k, seed=0),
                          solver=R.CoarseSolveChoice(kind=R.DIRECT_CHOLESKY if i == len(ks) - 1 else R.INNER_FCG))
              for i, k in enumerate(ks)]
    return R.MethodSpec(kind=R.PCG_VCYCLE, levels=levels, solver=R.SolverConfig(tol, 2000))


@pytest.mark.parametrize("k", [2, 5, 16])
def test_block_equals_single_solves(gpu, orc, k):
    x = R.synth_sparse_zipf(4000, 600, 20.0, 1.1, True, 3)
    m = R.DeviceMatrix(x)
    pm = R.PreparedMethod(m, 0.5, vspec([80, 12]))
    B = np.stack([R.rng_normals(100 + q, 4000) for q in range(k)], axis=1)
    B[:, 0] *= 1e3  # columns of very different scale converge independently
    W, reps = pm.solve_batch(B)
    om = to_checker(orc, x)
    for q in range(k):
        w1, r1 = pm.solve(B[:, q])
        assert reps[q].converged and abs(reps[q].iterations - r1.iterations) <= 1, (q, reps[q].iterations,
                                                                                    r1.iterations)
        assert rel_diff(W[:, q], w1) <= 1e-10
        assert len(reps[q].residual_history) == reps[q].iterations
        if q < 2:
            ref = orc.solve(om, 0.5, B[:, q], "cg", tol=1e-12, max_iters=5000)
            assert rel_diff(W[:, q], ref.w) <= 1e-8


def test_block_zero_column_and_sequential_fallback(gpu):
    x = random_matrix(300, 90, 4, 0.3)
    m = R.DeviceMatrix(x)
    pm = R.PreparedMethod(m, 1e-2, vspec([20]))
    B = np.stack([R.rng_normals(1, 300), np.zeros(300), R.rng_normals(2, 300)], axis=1)
    W, reps = pm.solve_batch(B)
    assert reps[1].converged and reps[1].iterations == 0 and not W[:, 1].any()
    os.environ["RMG_BATCH_SEQ"] = "1"
    try:
        W2, reps2 = pm.solve_batch(B)
    finally:
        os.environ.pop("RMG_BATCH_SEQ")
    for q in (0, 2):
        assert abs(reps[q].iterations - reps2[q].iterations) <= 1
        assert rel_diff(W[:, q], W2[:, q]) <= 1e-10


def test_block_rejects_non_finite_rhs(gpu):
    x = random_matrix(200, 60, 5, 0.3)
    pm = R.PreparedMethod(R.DeviceMatrix(x), 1e-2, vspec([12]))
    B = np.stack([R.rng_normals(1, 200), R.rng_normals(2, 200)], axis=1)
    B[3, 1] = np.nan
    with pytest.raises(ValueError):
        pm.solve_batch(B)


@pytest.mark.parametrize("fp32", [False, True])
@pytest.mark.parametrize("kind", ["jacobi_cg", "pcg_vcycle", "pcg_vcycle_additive"])
def test_dense_block_solve_beta_sweep(gpu, fp32, kind):
    """Dense X with several right-hand sides over a beta sweep: every
    operator application of the lock-step solve is a DMMA GEMM with G = X^T X (formed once
    on the tensor cores, reused across the sweep); each column meets numpy's direct
    solution and its own single-RHS solve."""
    x = R.synth_dense_clustered(1500, 200, 25, 0.1, 3)
    a = x.dense().astype(np.float32) if fp32 else x.dense()
    m = R.DeviceMatrix.from_dense(a)
    a64 = a.astype(np.float64)
    spec = vspec([25, 5]) if kind != "jacobi_cg" else R.MethodSpec(kind=R.JACOBI_CG, solver=R.SolverConfig(1e-10, 5000))
    spec.kind = R.method_from_string(kind)
    pm = R.PreparedMethod(m, 1.0, spec)
    B = np.stack([R.rng_normals(300 + q, 1500) for q in range(6)], axis=1)
    for beta in (1.0, 1e-2):
        pm.set_beta(beta)
        W, reps = pm.solve_batch(B)
        exact = np.linalg.solve(a64.T @ a64 + beta * np.eye(200), a64.T @ B)
        for q in range(6):
            assert reps[q].converged
            assert rel_diff(W[:, q], exact[:, q]) <= 1e-8, (beta, q, rel_diff(W[:, q], exact[:, q]))
        # the single-RHS solve applies X^T (X v) by sweeps, the batch G V with G = X^T X: two
        # roundings of one operator, so near the 1e-10 floor the counts may part by a few
        w1, r1 = pm.solve(B[:, 2].copy())
        assert abs(reps[2].iterations - r1.iterations) <= max(2, round(0.05 * r1.iterations))
        assert rel_diff(W[:, 2], w1) <= 1e-8
