"""Regularization sweep over a fixed hierarchy (rmg_method_set_beta; BASELINE
cfg 3): after set_beta(b2) a prepared method solves exactly like a fresh
prepare at b2 (same clustering, bit-identical w and iteration counts)."""
import numpy as np
import pytest

import paper_1806_05826_b200 as R
from helpers import random_matrix

pytestmark = pytest.mark.gpu


def lvl(k, kind=R.DIRECT_CHOLESKY):
    return R.LevelSpec(clustering=R.ClusteringChoice(kind=R.KMEANS, target_size=k),
                       solver=R.CoarseSolveChoice(kind=kind))


@pytest.mark.parametrize("method", ["cg", "jacobi_cg", "fcg_twolevel", "fgmres_twolevel", "fcg_multilevel"])
def test_set_beta_equals_fresh_prepare(gpu, method):
    x = R.synth_sparse_zipf(3000, 400, 15.0, 1.1, True, 4)
    m = R.DeviceMatrix(x, R.default_context())
    kind = R.method_from_string(method)
    levels = [] if "cg" == method or method == "jacobi_cg" else (
        [lvl(60, R.INNER_FCG), lvl(12)] if method == "fcg_multilevel" else [lvl(40)])
    spec = R.MethodSpec(kind=kind, levels=levels, solver=R.SolverConfig(1e-10, 2000))
    b = R.rng_normals(7, 3000)
    pm = R.PreparedMethod(m, 1e-3, spec)
    for beta in (1e-2, 1.0, 10.0):
        pm.set_beta(beta)
        w1, r1 = pm.solve(b)
        fresh = R.PreparedMethod(m, beta, spec)
        w2, r2 = fresh.solve(b)
        assert r1.iterations == r2.iterations and np.array_equal(w1, w2), (method, beta)
        if levels:
            assert np.array_equal(pm.labels(0), fresh.labels(0))
        fresh.close()
    with pytest.raises(ValueError):
        pm.set_beta(-1.0)


@pytest.mark.parametrize("method", ["jacobi_cg", "pcg_vcycle", "pcg_vcycle_additive"])
def test_set_beta_batched_equals_fresh_prepare(gpu, method):
    """Batched solves: set_beta rebuilds the lock-step loop's CUDA graph itself (beta and
    the rebuilt coarse buffers are baked into its nodes); the next batch equals a fresh
    prepare at that beta bit for bit, also when set_beta is called twice in a row or
    before any batch was solved."""
    x = R.synth_sparse_zipf(4000, 500, 15.0, 1.1, True, 6)
    m = R.DeviceMatrix(x, R.default_context())
    levels = [] if method == "jacobi_cg" else [lvl(70, R.INNER_FCG), lvl(10)]
    spec = R.MethodSpec(kind=R.method_from_string(method), levels=levels, solver=R.SolverConfig(1e-10, 2000))
    B = np.stack([R.rng_normals(30 + q, 4000) for q in range(4)], axis=1)
    pm = R.PreparedMethod(m, 1e-3, spec)
    pm.set_beta(5e-3)  # no batch solved yet: nothing to rebuild
    pm.solve_batch(B)
    for betas in ((1e-2,), (0.5, 1.0), (10.0,)):
        for beta in betas:
            pm.set_beta(beta)
        W1, r1 = pm.solve_batch(B)
        fresh = R.PreparedMethod(m, betas[-1], spec)
        W2, r2 = fresh.solve_batch(B)
        assert [r.iterations for r in r1] == [r.iterations for r in r2] and np.array_equal(W1, W2), (method, betas)
        fresh.close()
    W3, r3 = pm.solve_batch(B[:, :2])  # another k: the graph is rebuilt for it inside the solve
    assert all(r.converged for r in r3)
    assert np.linalg.norm(W3 - W1[:, :2]) <= 1e-7 * np.linalg.norm(W1[:, :2])
    pm.close()
