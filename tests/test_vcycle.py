"""pcg_vcycle (extension): plain PCG with a symmetric V-cycle over
the reference's hierarchy -- damped-Jacobi pre- and post-smoothing (BASELINE cfg 1's
"1 pre-sweep, 1 post-sweep"), coarsest level direct.  The reference has no such
routine, so it is pinned against a numpy restatement of the same
cycle on the same hierarchy (labels, X_k, beta_k and Jacobi weights read back from
the prepared method), and its solves against the reference's solution of the same
system (oracle CG to 1e-12)."""
import numpy as np
import pytest

import paper_1806_05826_b200 as R
from helpers import random_matrix, rel_diff, to_checker

pytestmark = pytest.mark.gpu


def spec(ks, tol=1e-10, max_iters=2000, normalize=False):
    levels = [R.LevelSpec(clustering=R.ClusteringChoice(kind=R.KMEANS, target_size=k, seed=0,
                                                        normalize_columns=normalize),
                          solver=R.CoarseSolveChoice(kind=R.DIRECT_CHOLESKY if i == len(ks) - 1 else R.INNER_FCG))
              for i, k in enumerate(ks)]
    return R.MethodSpec(kind=R.PCG_VCYCLE, levels=levels, solver=R.SolverConfig(tol, max_iters))


def restated_cycle(pm, r):
    """The cycle in numpy: z = x2 + w D^-1 (r - A x2), x2 = x1 + P A_c^-1 P^T (r - A x1),
    x1 = w D^-1 r, recursively; P = adjusted average (weights 1/sqrt(n_S))."""
    L = pm.n_levels - 1  # smoothed levels 0..L-1, level L direct
    mats = [pm.x.x.dense() if pm.x.x is not None else None] + [pm.level_matrix(k).dense() for k in range(1, L + 1)]
    betas = [pm.level(k)["beta"] for k in range(L + 1)]
    ws = [pm.level(k)["omega"] for k in range(L)]
    labs = [pm.labels(k) for k in range(L)]

    def cycle(k, rk):
        x = mats[k]
        a = x.T @ x + betas[k] * np.eye(x.shape[1])
        dinv = 1.0 / np.diag(a)
        lab = labs[k]
        nc = lab.max() + 1
        size = np.bincount(lab, minlength=nc)
        p = np.zeros((x.shape[1], nc))
        p[np.arange(x.shape[1]), lab] = 1.0 / np.sqrt(size[lab])
        x1 = ws[k] * dinv * rk
        rc = p.T @ (rk - a @ x1)
        if k + 1 == L:
            xc = mats[k + 1]
            ec = np.linalg.solve(xc.T @ xc + betas[k + 1] * np.eye(nc), rc)
        else:
            ec = cycle(k + 1, rc)
        x2 = x1 + p @ ec
        return x2 + ws[k] * dinv * (rk - a @ x2)

    return cycle(0, r)


@pytest.mark.parametrize("ks", [[30], [40, 8]])
def test_vcycle_matches_restatement_and_is_symmetric(gpu, ks):
    x = random_matrix(300, 120, 7, 0.3)
    m = R.DeviceMatrix(x)
    pm = R.PreparedMethod(m, 0.5, spec(ks))
    rng = np.random.default_rng(1)
    u, v = rng.standard_normal(120), rng.standard_normal(120)
    mu, mv = pm.precondition(u), pm.precondition(v)
    assert abs(u @ mv - v @ mu) <= 1e-12 * abs(u @ mv)
    assert rel_diff(mv, restated_cycle(pm, v)) <= 1e-12
    for k in range(len(ks)):
        assert 0.0 < pm.level(k)["omega"] < 2.0


@pytest.mark.parametrize("ks", [[30], [40, 8]])
def test_vcycle_solve_matches_reference_solution(gpu, orc, ks):
    x = random_matrix(300, 120, 8, 0.3)
    m = R.DeviceMatrix(x)
    b = R.rng_normals(42, 300)
    sol = R.solve_system(m, 0.5, b, spec(ks))
    ref = orc.solve(to_checker(orc, x), 0.5, b, "cg", tol=1e-12, max_iters=5000)
    assert sol.report.converged
    assert rel_diff(sol.w, ref.w) <= 1e-8
    assert sol.report.iterations < ref.iterations


def test_vcycle_cfg1_dense(gpu):
    """cfg 1 (dense 2000 x 500, 50 clusters) with Jacobi pre + post smoothing."""
    x = R.synth_dense_clustered(2000, 500, 50, 0.1, 0)
    a = x.dense()
    m = R.DeviceMatrix.from_dense(a)
    b = R.rng_normals(42, 2000)
    sol = R.solve_system(m, 1e-2, b, spec([50]))
    exact = np.linalg.solve(a.T @ a + 1e-2 * np.eye(500), a.T @ b)
    assert sol.report.converged
    assert rel_diff(sol.w, exact) <= 1e-8
    cg = R.solve_system(m, 1e-2, b, R.MethodSpec(kind=R.CG, solver=R.SolverConfig(1e-10, 5000)))
    assert sol.report.iterations < cg.report.iterations


def test_vcycle_set_beta_and_errors(gpu):
    x = random_matrix(200, 80, 9, 0.3)
    m = R.DeviceMatrix(x)
    pm = R.PreparedMethod(m, 1e-2, spec([20]))
    b = R.rng_normals(3, 200)
    for beta in (1.0, 1e-3):
        pm.set_beta(beta)
        w1, r1 = pm.solve(b)
        fresh = R.PreparedMethod(m, beta, spec([20]))
        w2, r2 = fresh.solve(b)
        assert r1.iterations == r2.iterations and np.array_equal(w1, w2)
    with pytest.raises(ValueError):
        R.PreparedMethod(m, 1e-2, R.MethodSpec(kind=R.PCG_VCYCLE, levels=[]))


# ---------------------------------------------------------------- pcg_vcycle_additive
def aspec(ks, tol=1e-10, max_iters=2000, additive=()):
    s = spec(ks, tol, max_iters)
    s.kind = R.PCG_VCYCLE_ADDITIVE
    for k in additive:  # further additive levels (rmg_level_spec.additive)
        s.levels[k].additive = True
    return s


def restated_additive(pm, r, additive=(0,)):
    """z = D_0^-1 r + P_0 V_1(P_0^T r), V_1 the symmetric cycle of levels >= 1 (or the
    coarsest direct solve for two levels); every level in `additive` enters the same way."""
    L = pm.n_levels - 1
    mats = [pm.x.x.dense()] + [pm.level_matrix(k).dense() for k in range(1, L + 1)]
    betas = [pm.level(k)["beta"] for k in range(L + 1)]
    ws = [pm.level(k)["omega"] for k in range(L)]
    labs = [pm.labels(k) for k in range(L)]

    def pmat(k):
        lab = labs[k]
        nc = lab.max() + 1
        size = np.bincount(lab, minlength=nc)
        p = np.zeros((lab.size, nc))
        p[np.arange(lab.size), lab] = 1.0 / np.sqrt(size[lab])
        return p

    def gram(k):
        return mats[k].T @ mats[k] + betas[k] * np.eye(mats[k].shape[1])

    def cycle(k, rk):
        if k == L:
            return np.linalg.solve(gram(k), rk)
        a, p = gram(k), pmat(k)
        dinv = 1.0 / np.diag(a)
        if k in additive:
            return dinv * rk + p @ cycle(k + 1, p.T @ rk)
        x1 = ws[k] * dinv * rk
        x2 = x1 + p @ cycle(k + 1, p.T @ (rk - a @ x1))
        return x2 + ws[k] * dinv * (rk - a @ x2)

    return cycle(0, r)


@pytest.mark.parametrize("ks", [[30], [40, 8], [60, 15, 4]])
def test_additive_matches_restatement_and_is_spd(gpu, ks):
    x = random_matrix(300, 120, 7, 0.3)
    m = R.DeviceMatrix(x)
    pm = R.PreparedMethod(m, 0.5, aspec(ks))
    rng = np.random.default_rng(2)
    u, v = rng.standard_normal(120), rng.standard_normal(120)
    mu, mv = pm.precondition(u), pm.precondition(v)
    assert abs(u @ mv - v @ mu) <= 1e-12 * abs(u @ mv)
    assert u @ mu > 0 and v @ mv > 0
    assert rel_diff(mv, restated_additive(pm, v)) <= 1e-12
    assert pm.level(0)["omega"] == 1.0  # the additive level applies D^-1 unweighted
    for k in range(1, len(ks)):
        assert 0.0 < pm.level(k)["omega"] < 2.0


@pytest.mark.parametrize("additive", [(1,), (1, 2), (2,)])
def test_additive_levels_flag(gpu, orc, additive):
    """rmg_level_spec.additive: deeper levels entered additively too (no operator
    application at those levels); M stays SPD and equals the restatement; single and
    batched solves reach the reference's solution."""
    x = random_matrix(300, 120, 7, 0.3)
    m = R.DeviceMatrix(x)
    pm = R.PreparedMethod(m, 0.5, aspec([60, 15, 4], additive=additive))
    rng = np.random.default_rng(3)
    u, v = rng.standard_normal(120), rng.standard_normal(120)
    mu, mv = pm.precondition(u), pm.precondition(v)
    assert abs(u @ mv - v @ mu) <= 1e-12 * abs(u @ mv)
    assert u @ mu > 0 and v @ mv > 0
    assert rel_diff(mv, restated_additive(pm, v, additive=(0,) + tuple(additive))) <= 1e-12
    B = np.stack([R.rng_normals(70 + q, 300) for q in range(3)], axis=1)
    W, reps = pm.solve_batch(B)
    for q in range(3):
        ref = orc.solve(to_checker(orc, x), 0.5, B[:, q].copy(), "cg", tol=1e-12, max_iters=5000)
        w1, r1 = pm.solve(B[:, q].copy())
        assert reps[q].converged and r1.converged and abs(reps[q].iterations - r1.iterations) <= 1
        assert rel_diff(W[:, q], ref.w) <= 1e-8 and rel_diff(w1, ref.w) <= 1e-8


@pytest.mark.parametrize("ks", [[30], [40, 8]])
def test_additive_solve_matches_reference_solution(gpu, orc, ks):
    x = random_matrix(300, 120, 8, 0.3)
    m = R.DeviceMatrix(x)
    b = R.rng_normals(42, 300)
    sol = R.solve_system(m, 0.5, b, aspec(ks))
    ref = orc.solve(to_checker(orc, x), 0.5, b, "cg", tol=1e-12, max_iters=5000)
    assert sol.report.converged
    assert rel_diff(sol.w, ref.w) <= 1e-8
    assert sol.report.iterations < ref.iterations


def test_additive_batch_equals_single(gpu, orc):
    x = R.synth_sparse_zipf(4000, 600, 20.0, 1.1, False, 5)
    m = R.DeviceMatrix(x)
    pm = R.PreparedMethod(m, 0.5, aspec([80, 12]))
    B = np.stack([R.rng_normals(200 + q, 4000) for q in range(4)], axis=1)
    W, reps = pm.solve_batch(B)
    ref = orc.solve(to_checker(orc, x), 0.5, B[:, 0], "cg", tol=1e-12, max_iters=5000)
    assert rel_diff(W[:, 0], ref.w) <= 1e-8
    for q in range(4):
        w1, r1 = pm.solve(B[:, q])
        assert reps[q].converged and abs(reps[q].iterations - r1.iterations) <= 1
        assert rel_diff(W[:, q], w1) <= 1e-10


@pytest.mark.gpu
@pytest.mark.parametrize("kind", ["pcg_vcycle", "pcg_vcycle_additive"])
def test_deferred_coarse_layouts_equal_eager(gpu, monkeypatch, kind):
    """Coarse levels of a V-cycle hierarchy build their K1 layout and hot X^T blocks on a
    first application only (Matrix::ensure_operator); RMG_EAGER_LEVELS=1 builds them at
    prepare as before.  Same preconditioner, same solves (single and batched) either way;
    timing a deferred level's operator builds its layouts on the spot."""
    x = R.synth_sparse_zipf(5000, 700, 18.0, 1.1, True, 9)
    m = R.DeviceMatrix(x)
    sp = aspec([90, 20, 5], additive=(1,)) if kind == "pcg_vcycle_additive" else spec([90, 20, 5])
    b = R.rng_normals(11, 5000)
    B = np.stack([R.rng_normals(300 + q, 5000) for q in range(3)], axis=1)
    v = np.random.default_rng(4).standard_normal(700)
    out = {}
    for eager in (False, True):
        if eager:
            monkeypatch.setenv("RMG_EAGER_LEVELS", "1")
        else:
            monkeypatch.delenv("RMG_EAGER_LEVELS", raising=False)
        pm = R.PreparedMethod(m, 0.3, sp)
        w, rep = pm.solve(b.copy())
        W, reps = pm.solve_batch(B)
        pm.set_beta(0.05)  # rebuilds the cycle: the deferred levels stay consistent
        w2, rep2 = pm.solve(b.copy())
        out[eager] = (pm.precondition(v), w, rep.iterations, W, [r.iterations for r in reps], w2, rep2.iterations)
        assert rep.converged and rep2.converged and all(r.converged for r in reps)
        for lv in range(1, pm.n_levels):
            assert pm.time_operator(lv, 1, False)[0] > 0.0
        pm.close()
    d, e = out[False], out[True]
    assert rel_diff(d[0], e[0]) <= 1e-12
    assert rel_diff(d[1], e[1]) <= 1e-9 and abs(d[2] - e[2]) <= 1
    assert rel_diff(d[3], e[3]) <= 1e-9 and all(abs(a - c) <= 1 for a, c in zip(d[4], e[4]))
    assert rel_diff(d[5], e[5]) <= 1e-9 and abs(d[6] - e[6]) <= 1
