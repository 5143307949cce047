"""GPU parity: the sm_100a path (through the C ABI) against the reference's
golden vectors (tests/golden, produced by the verbatim reference build) and
against the CPU oracle restatement.

Tolerances (the reference's own ladder, SURVEY.md §4, and BASELINE north_star):
  kernels 1e-13 relative (GPU reduction order differs from the sequential CPU sum),
  bit-exact where the order is the reference's (gram diagonal, labels, X_c),
  preconditioner 1e-10, w 1e-8 relative L2, iteration counts +-2.
"""
import numpy as np
import pytest

import paper_1806_05826_b200 as R
from helpers import (golden_matrix, ideal_instance, load_golden, random_matrix, rel_diff, to_checker)

pytestmark = pytest.mark.gpu

KERNEL_TOL = 1e-13
W_TOL = 1e-8


def dm(x):
    return R.DeviceMatrix(x, R.default_context())


def kmeans_level(k, normalize=False, kind=R.DIRECT_CHOLESKY, seed=0):
    return R.LevelSpec(clustering=R.ClusteringChoice(kind=R.KMEANS, target_size=k, seed=seed,
                                                     normalize_columns=normalize),
                       solver=R.CoarseSolveChoice(kind=kind))


def imported(labels, nc, kind=R.DIRECT_CHOLESKY, omega=None):
    return R.LevelSpec(clustering=R.ClusteringChoice(kind=R.IMPORTED, labels=labels, n_clusters=nc),
                       solver=R.CoarseSolveChoice(kind=kind), omega_override=omega)


# ---------------------------------------------------------------- kernels
@pytest.mark.parametrize("case", range(5))
def test_operator_kernels_match_reference(gpu, case):
    g = load_golden("random")
    p = f"r{case}"
    x = golden_matrix(g, p)
    m = dm(x)
    beta = float(g[p + "_beta"])
    assert rel_diff(m.spmv(g[p + "_v"]), g[p + "_spmv"]) <= KERNEL_TOL
    assert rel_diff(m.spmv_transpose(g[p + "_u"]), g[p + "_spmv_t"]) <= KERNEL_TOL
    assert rel_diff(m.ridge_apply(beta, g[p + "_v"]), g[p + "_ridge"]) <= KERNEL_TOL
    assert np.array_equal(m.gram_diagonal(beta), g[p + "_diag"])  # same order as ridge.cpp:30-37
    lam, it, cv = m.lambda_max()
    assert abs(lam - float(g[p + "_lambda"])) <= 1e-10 * lam
    assert abs(it - int(g[p + "_lambda_iters"])) <= 1


def test_lpsc105_operator(gpu):
    g = load_golden("lpsc105")
    m = dm(golden_matrix(g))
    assert rel_diff(m.ridge_apply(1e-6, g["apply_w"]), g["apply_out"]) <= KERNEL_TOL
    assert np.array_equal(m.gram_diagonal(1e-6), g["gram_diag"])
    b = R.generate_rhs(m, 42)
    assert np.array_equal(b.b, g["b"])
    assert rel_diff(b.rhs, g["rhs"]) <= KERNEL_TOL


def test_zipf_operator_vs_oracle(gpu, orc):
    """Zipf-skewed columns exercise the split long-column path of the X^T kernel."""
    x = R.synth_sparse_zipf(20000, 3000, 40.0, 1.1, False, 7)
    m = dm(x)
    assert m.is_pattern
    om = to_checker(orc, x)
    w = np.random.default_rng(0).standard_normal(x.n_features)
    assert rel_diff(m.ridge_apply(0.5, w), orc.ridge_apply(om, 0.5, w)) <= KERNEL_TOL
    u = np.random.default_rng(1).standard_normal(x.n_samples)
    assert rel_diff(m.spmv_transpose(u), orc.spmv_transpose(om, u)) <= KERNEL_TOL
    xv = R.synth_sparse_zipf(20000, 3000, 40.0, 1.1, True, 7)  # |N(0,1)| values
    mv, omv = dm(xv), to_checker(orc, xv)
    assert not mv.is_pattern
    assert rel_diff(mv.ridge_apply(0.5, w), orc.ridge_apply(omv, 0.5, w)) <= KERNEL_TOL


# ---------------------------------------------------------------- setup parity (bit-exact)
@pytest.mark.parametrize("case", range(5))
def test_kmeans_labels_and_coarse_matrix_bit_exact(gpu, case):
    g = load_golden("random")
    p = f"r{case}"
    x = golden_matrix(g, p)
    k = int(g[p + "_kpp"].shape[0])
    pm = R.PreparedMethod(dm(x), float(g[p + "_beta"]),
                          R.MethodSpec(kind=R.FCG_TWOLEVEL, levels=[kmeans_level(k)]))
    assert np.array_equal(pm.labels(0), g[p + "_km_labels"])
    xc = pm.level_matrix(1)
    gx = golden_matrix(g, p + "_xc")
    assert np.array_equal(xc.row_offsets, gx.row_offsets)
    assert np.array_equal(xc.column_indices, gx.column_indices)
    assert np.array_equal(xc.values, gx.values)


@pytest.mark.parametrize("case", range(5))
def test_two_level_apply(gpu, case):
    g = load_golden("random")
    p = f"r{case}"
    x = golden_matrix(g, p)
    k = int(g[p + "_kpp"].shape[0])
    pm = R.PreparedMethod(dm(x), float(g[p + "_beta"]),
                          R.MethodSpec(kind=R.FCG_TWOLEVEL, levels=[imported(g[p + "_km_labels"], k, omega=0.37)]))
    assert rel_diff(pm.precondition(g[p + "_v"]), g[p + "_z"]) <= 1e-10


# ---------------------------------------------------------------- solves
@pytest.mark.parametrize("case", range(5))
@pytest.mark.parametrize("method", ["cg", "jacobi_cg", "fcg_twolevel", "fcg_multilevel"])
def test_random_solves(gpu, case, method):
    g = load_golden("random")
    p = f"r{case}"
    key = f"{p}_{method}"
    if key + "_iterations" not in g.files:
        pytest.skip("no multilevel golden for this case")
    x = golden_matrix(g, p)
    k = int(g[p + "_kpp"].shape[0])
    if method == "fcg_multilevel":
        levels = [kmeans_level(k, kind=R.INNER_FCG), kmeans_level(k // 2)]
    else:
        levels = [kmeans_level(k)]
    spec = R.MethodSpec(kind=R.method_from_string(method), levels=levels, solver=R.SolverConfig(1e-8, 2000 if method != "fcg_multilevel" else 400))
    sol = R.solve_system(dm(x), float(g[p + "_beta"]), g[p + "_b"], spec)
    assert sol.report.converged
    assert abs(sol.report.iterations - int(g[key + "_iterations"])) <= 2
    assert rel_diff(sol.w, g[key + "_w"]) <= W_TOL
    if method.startswith("fcg"):
        assert len(sol.report.inner_iterations) == sol.report.iterations


def test_lpsc105_cg_66(gpu):
    g = load_golden("lpsc105")
    m = dm(golden_matrix(g))
    sol = R.solve_system(m, 1e-6, g["b"], R.MethodSpec(kind=R.CG, solver=R.SolverConfig(1e-6, 20000)))
    assert sol.report.converged
    assert int(g["cg_iterations"]) == 66
    assert abs(sol.report.iterations - 66) <= 2
    # kappa(A) ~ 1e7 at beta = 1e-6: two CG trajectories that differ only in
    # reduction rounding agree to ~7e-8 at tol 1e-6 -- the reference's own
    # threaded runs differ from its sequential run by up to envelope cg_w_spread ...
    env = _envelope("lpsc105")
    assert rel_diff(sol.w, g["cg_w"]) <= env["cg_w_spread"], (rel_diff(sol.w, g["cg_w"]), env["cg_w_spread"])
    assert sol.coarse_size == 0
    # ... and to the 1e-8 bar once both are driven to tol 1e-12 (SURVEY App. B protocol)
    ref_tight = R.solve_system(m, 1e-6, g["b"], R.MethodSpec(kind=R.CG, solver=R.SolverConfig(1e-12, 20000)))
    import oracle
    o = oracle.Checker("oracle")
    om = to_checker(o, golden_matrix(g))
    tight = o.solve(om, 1e-6, g["b"], "cg", tol=1e-12, max_iters=20000)
    assert rel_diff(ref_tight.w, tight.w) <= W_TOL


def test_lpsc105_leader_follower_134_one_iteration(gpu):
    g = load_golden("lpsc105")
    m = dm(golden_matrix(g))
    lv = R.LevelSpec(clustering=R.ClusteringChoice(kind=R.LEADER_TARGET, target_size=134))
    pm = R.PreparedMethod(m, 1e-6, R.MethodSpec(kind=R.FCG_TWOLEVEL, levels=[lv], solver=R.SolverConfig(1e-6, 5000)))
    assert np.array_equal(pm.labels(0), g["lf134_labels"])
    w, rep = pm.solve(g["b"])
    assert rep.converged and rep.iterations == 1
    assert rel_diff(w, g["lf134_w"]) <= 1e-6  # one step: w = M^-1 rhs scaled


def test_lpsc105_leader_follower_52(gpu):
    """LF closest to 56 yields 52 clusters.  Its coarse system (beta = 1e-6) is so
    ill-conditioned that the iteration count depends on the Cholesky rounding:
    reference+Eigen recorded 43 (proj/test_output.txt:41), reference+our LLT
    shim 37 (golden); the shim build with 4, 7 or 8 threads gives 40.  The GPU
    (explicit inverse of the same Cholesky factor) is held to +-2 of the golden."""
    g = load_golden("lpsc105")
    m = dm(golden_matrix(g))
    lv = R.LevelSpec(clustering=R.ClusteringChoice(kind=R.LEADER_TARGET, target_size=56))
    pm = R.PreparedMethod(m, 1e-6, R.MethodSpec(kind=R.FCG_TWOLEVEL, levels=[lv], solver=R.SolverConfig(1e-6, 5000)))
    assert pm.coarse_size() == 52
    assert np.array_equal(pm.labels(0), g["lf56_labels"])
    w, rep = pm.solve(g["b"])
    assert rep.converged and abs(rep.iterations - int(g["lf56_iterations"])) <= 2, rep.iterations


def test_cnae_duplicate_merging(gpu):
    g = load_golden("cnae")
    m = dm(golden_matrix(g))
    lv = R.LevelSpec(clustering=R.ClusteringChoice(kind=R.LEADER_TOLERANCE, tolerance=0.5))
    pm = R.PreparedMethod(m, 1e-6, R.MethodSpec(kind=R.FCG_TWOLEVEL, levels=[lv], solver=R.SolverConfig(1e-6, 5000)))
    assert pm.coarse_size() == int(g["lf_nc"]) == 694
    assert np.array_equal(pm.labels(0), g["lf_labels"])
    w, rep = pm.solve(g["b"])
    assert rep.converged and rep.iterations == 1
    # Unpreconditioned CG needs 656 iterations on an 856-dimensional, beta = 1e-6
    # system: far past the point where finite-precision CG loses orthogonality,
    # so the count follows the summation accuracy.  The bar is the measured
    # envelope of the same algorithm (tests/golden/envelope.json "cnae": the
    # reference's threads, and the restatement with pairwise dots / segmented
    # X^T sums / FMA updates -- the GPU's accuracy class -- which gives 640-657).
    env = _envelope("cnae")
    cg = R.solve_system(m, 1e-6, g["b"], R.MethodSpec(kind=R.CG, solver=R.SolverConfig(1e-6, 20000)))
    assert cg.report.converged
    lo, hi = env["cg_iterations_range"]
    assert lo - 2 <= cg.report.iterations <= hi + 2, (cg.report.iterations, env["cg_iterations_range"])
    assert rel_diff(cg.w, g["cg_w"]) <= env["cg_w_spread"], (rel_diff(cg.w, g["cg_w"]), env["cg_w_spread"])


def test_cfg1_two_level(gpu):
    g = load_golden("cfg1")
    x = R.synth_dense_clustered(2000, 500, 50, 0.1, 0)
    m = dm(x)
    lv = kmeans_level(50)
    pm = R.PreparedMethod(m, 1e-2, R.MethodSpec(kind=R.FCG_TWOLEVEL, levels=[lv]))
    assert np.array_equal(pm.labels(0), g["labels0"])
    w, rep = pm.solve(g["b"])
    assert rep.converged
    assert abs(rep.iterations - int(g["fcg_iterations"])) <= 2
    assert rel_diff(w, g["fcg_w"]) <= W_TOL
    cg = R.solve_system(m, 1e-2, g["b"], R.MethodSpec(kind=R.CG))
    assert abs(cg.report.iterations - int(g["cg_iterations"])) <= 2
    assert rel_diff(cg.w, g["cg_w"]) <= W_TOL


def test_ideal_datasets_one_iteration(gpu):
    """acceptance.cpp criterion 1: two-level FCG is exact on duplicated columns."""
    worst = 0
    for seed in range(1, 51):
        x, labels, nc = ideal_instance(seed)
        m = dm(x)
        for beta in (1e-6, 1e-2):
            spec = R.MethodSpec(kind=R.FCG_TWOLEVEL, levels=[imported(labels, nc)], solver=R.SolverConfig(1e-10, 5000))
            sol = R.solve_system(m, beta, R.generate_rhs(m, 42).b, spec)
            assert sol.report.converged
            worst = max(worst, sol.report.iterations)
    assert worst == 1


def test_deterministic(gpu):
    x = R.synth_sparse_zipf(5000, 800, 30.0, 1.1, False, 3)
    m = dm(x)
    spec = R.MethodSpec(kind=R.FCG_MULTILEVEL,
                        levels=[kmeans_level(80, True, R.INNER_FCG), kmeans_level(10, True)])
    pm = R.PreparedMethod(m, 1.0, spec)
    b = R.rng_normals(42, x.n_samples)
    w1, r1 = pm.solve(b)
    w2, r2 = pm.solve(b)
    assert r1.iterations == r2.iterations
    assert np.array_equal(w1, w2)
    assert np.array_equal(r1.residual_history, r2.residual_history)


# ---------------------------------------------------------------- errors and edges
def test_errors_and_edges(gpu):
    x = random_matrix(12, 8, 99, 0.5)
    m = dm(x)
    with pytest.raises(ValueError):
        m.ridge_apply(-1.0, np.zeros(8))
    with pytest.raises(ValueError):
        R.PreparedMethod(m, -1.0, R.MethodSpec(kind=R.CG))
    with pytest.raises(ValueError):  # coarsest level must be direct
        R.PreparedMethod(m, 1.0, R.MethodSpec(kind=R.FCG_MULTILEVEL, levels=[kmeans_level(4, kind=R.INNER_CG)]))
    with pytest.raises(ValueError):  # only the last level may be direct
        R.PreparedMethod(m, 1.0, R.MethodSpec(kind=R.FCG_MULTILEVEL, levels=[kmeans_level(4), kmeans_level(2)]))
    with pytest.raises(ValueError):  # not fewer clusters than features
        R.PreparedMethod(m, 1.0, R.MethodSpec(kind=R.FCG_TWOLEVEL, levels=[kmeans_level(8)]))
    with pytest.raises(ValueError):
        R.PreparedMethod(m, 1.0, R.MethodSpec(kind=R.FCG_TWOLEVEL, levels=[]))
    pm = R.PreparedMethod(m, 1.0, R.MethodSpec(kind=R.CG))
    with pytest.raises(ValueError):
        pm.solve(np.zeros(5))
    # zero right-hand side: converged at once, history [0] (krylov.cpp:170-175)
    w, rep = pm.solve(np.zeros(12))
    assert rep.converged and rep.iterations == 0 and list(rep.residual_history) == [0.0]
    assert not np.any(w)
    # non-finite rhs
    with pytest.raises(ValueError):
        pm.solve_rhs(np.full(8, np.nan))
    # A = diag(1, 0) is singular: CG must report the breakdown (test_krylov.cpp:106-113)
    sing = R.csr_from_triplets(1, 2, [0], [0], [1.0])
    pm2 = R.PreparedMethod(dm(sing), 0.0, R.MethodSpec(kind=R.CG))
    with pytest.raises(RuntimeError):
        pm2.solve_rhs(np.array([0.0, 1.0]))
    # empty matrix (no nonzeros): A = beta I and rhs = 0
    empty = R.FeatureMatrix(5, 3, np.zeros(6, np.uint64), np.zeros(0, np.uint64), np.zeros(0))
    sol = R.solve_system(dm(empty), 1.0, np.ones(5), R.MethodSpec(kind=R.CG))
    assert sol.report.converged and not np.any(sol.w)
    # diag(2, 5) in <= 2 iterations (test_krylov.cpp:42-53)
    d = R.csr_from_triplets(2, 2, [0, 1], [0, 1], [np.sqrt(2.0), np.sqrt(5.0)])
    pm3 = R.PreparedMethod(dm(d), 0.0, R.MethodSpec(kind=R.CG, solver=R.SolverConfig(1e-12)))
    w, rep = pm3.solve_rhs(np.array([2.0, 5.0]))
    assert rep.converged and rep.iterations <= 2
    assert np.allclose(w, [1.0, 1.0], rtol=1e-10)
    # max_iters reached: not converged, not an error
    pm4 = R.PreparedMethod(m, 1e-3, R.MethodSpec(kind=R.CG, solver=R.SolverConfig(1e-14, 2)))
    w, rep = pm4.solve(np.ones(12))
    assert not rep.converged and rep.iterations == 2


# ---------------------------------------------------------------- BASELINE cfg 2 (scaled and full)
def _cfg2_spec(ks, labels=None):
    levels = []
    for i, k in enumerate(ks):
        last = i == len(ks) - 1
        if labels is None:
            cl = R.ClusteringChoice(kind=R.KMEANS, target_size=k, seed=0, normalize_columns=True)
        else:
            cl = R.ClusteringChoice(kind=R.IMPORTED, labels=labels[i], n_clusters=k)
        levels.append(R.LevelSpec(clustering=cl, solver=R.CoarseSolveChoice(
            kind=R.DIRECT_CHOLESKY if last else R.INNER_FCG, tol=1e-6, max_iters=500)))
    return R.MethodSpec(kind=R.FCG_MULTILEVEL, levels=levels, solver=R.SolverConfig(1e-6, 1000))


def _envelope(name):
    """The measured rounding envelope of the reference's algorithm on a case
    (tests/golden/make_envelope.py): iteration-count range over the reference's
    threaded runs and the restatement under the GPU's arithmetic orders, and the
    largest w difference among them.  Counts are held to the range +-2 (the
    north star's +-2 applied to the set of counts the algorithm produces)."""
    import json
    import os
    return json.load(open(os.path.join(os.path.dirname(__file__), "golden", "envelope.json")))[name]


def _csr_sha(x):
    import hashlib
    h = hashlib.sha256()
    h.update(np.ascontiguousarray(x.row_offsets, np.uint64).tobytes())
    h.update(np.ascontiguousarray(x.column_indices, np.uint64).tobytes())
    h.update(np.ascontiguousarray(x.value_array(), np.float64).tobytes())
    return h.hexdigest()


@pytest.mark.parametrize("name,n,f,ks", [("cfg2_small", 10000, 2000, [200, 20]),
                                         ("cfg2_full", 100000, 20000, [2000, 200])])
def test_cfg2_multilevel(gpu, name, n, f, ks):
    g = load_golden(name)
    x = R.synth_sparse_zipf(n, f, 40.0, 1.1, False, 0)
    assert _csr_sha(x) == str(g["sha256"])  # generator pinned
    m = dm(x)
    pm = R.PreparedMethod(m, 1.0, _cfg2_spec(ks))
    for i in range(len(ks)):  # k-means on normalised columns, bit-exact per level
        assert np.array_equal(pm.labels(i), g[f"labels{i}"].astype(np.int64))
    # At tol 1e-6 the bar is the measured rounding envelope of the reference's
    # algorithm (tests/golden/envelope.json): its own threaded runs (2-8 threads) and
    # the restatement under the GPU's arithmetic choices (pairwise dots, segmented
    # X^T sums, FMA updates, explicit coarse inverse, omega +-1 ulp).
    env = _envelope(name)
    w, rep = pm.solve(g["b"])
    assert rep.converged
    lo, hi = env["ml_iterations_range"]
    assert lo - 2 <= rep.iterations <= hi + 2, (rep.iterations, env["ml_iterations_range"])
    # w at tol 1e-6: within the envelope's w spread; the strict 1e-8 comparison is
    # made at tol 1e-12 below
    assert rel_diff(w, g["ml_w"]) <= env["ml_w_spread"], (rel_diff(w, g["ml_w"]), env["ml_w_spread"])
    assert len(rep.inner_iterations) == rep.iterations
    gi = g["ml_inner"].astype(np.int64)
    # the first inner solves (same outer trajectory so far) take the reference's counts
    assert np.all(np.abs(rep.inner_iterations[:3].astype(np.int64) - gi[:3]) <= 2)
    cg = R.solve_system(m, 1.0, g["b"], R.MethodSpec(kind=R.CG, solver=R.SolverConfig(1e-6, 5000)))
    lo, hi = env["cg_iterations_range"]
    assert lo - 2 <= cg.report.iterations <= hi + 2, (cg.report.iterations, env["cg_iterations_range"])
    assert rel_diff(cg.w, g["cg_w"]) <= env["cg_w_spread"], (rel_diff(cg.w, g["cg_w"]), env["cg_w_spread"])
    # Driven to tol 1e-12: the strict bar.  The reference's CG converges there
    # (cg12); its multilevel FCG converges on cfg2_small but stagnates near 1e-9
    # on cfg2_full (inexact inner solves, ml12_converged = 0 in the golden) at a
    # w 1.2e-9 from the CG solution, so there the GPU multilevel w is held to
    # the CG solution at the same 1e-8 bar.
    if "ml12_w" in g.files:
        spec12 = _cfg2_spec(ks, [g[f"labels{i}"].astype(np.int64) for i in range(len(ks))])
        spec12.solver = R.SolverConfig(1e-12, 1000)
        w12, rep12 = R.PreparedMethod(m, 1.0, spec12).solve(g["b"])
        cg12 = R.solve_system(m, 1.0, g["b"], R.MethodSpec(kind=R.CG, solver=R.SolverConfig(1e-12, 5000)))
        assert rel_diff(cg12.w, g["cg12_w"]) <= W_TOL, rel_diff(cg12.w, g["cg12_w"])
        if int(g["ml12_converged"]):
            assert rep12.converged
            assert rel_diff(w12, g["ml12_w"]) <= W_TOL, rel_diff(w12, g["ml12_w"])
        else:
            assert rel_diff(g["ml12_w"], g["cg12_w"]) <= W_TOL  # the reference's own gap
            assert float(rep12.residual_history[-1]) <= 10 * float(g["ml12_hist"][-1])
            assert rel_diff(w12, g["cg12_w"]) <= W_TOL, rel_diff(w12, g["cg12_w"])


# ---------------------------------------------------------------- FGMRES
@pytest.mark.parametrize("case", range(3))
def test_fgmres_twolevel_matches_oracle(gpu, orc, case):
    """fgmres_twolevel (krylov.cpp:229-328, 628-635): GPU MGS sweep + host
    Givens against the oracle (pinned bit-exact to the reference build)."""
    n, f, seed = [(300, 120, 5), (800, 300, 7), (2000, 500, 0)][case]
    x = random_matrix(n, f, seed, 0.3) if case < 2 else R.synth_dense_clustered(2000, 500, 50, 0.1, 0)
    m = dm(x)
    om = to_checker(orc, x)
    b = orc.normals(seed + 1, n)
    k = [20, 40, 50][case]
    sol = R.solve_system(m, 1e-2, b, R.MethodSpec(kind=R.FGMRES_TWOLEVEL, levels=[kmeans_level(k)],
                                                  solver=R.SolverConfig(1e-10, 400)))
    ref = orc.solve(om, 1e-2, b, "fgmres_twolevel", levels=[dict(target_size=k)], tol=1e-10, max_iters=400)
    assert sol.report.converged == ref.converged
    assert abs(sol.report.iterations - ref.iterations) <= 2, (sol.report.iterations, ref.iterations)
    assert rel_diff(sol.w, ref.w) <= W_TOL, rel_diff(sol.w, ref.w)
    assert len(sol.report.inner_iterations) == sol.report.iterations
    assert np.all(sol.report.inner_iterations == 0)  # direct coarse solve


def test_fgmres_edges(gpu, orc):
    x = random_matrix(200, 60, 3, 0.4)
    m = dm(x)
    spec = R.MethodSpec(kind=R.FGMRES_TWOLEVEL, levels=[kmeans_level(10)], solver=R.SolverConfig(1e-12, 5))
    pm = R.PreparedMethod(m, 0.1, spec)
    w, rep = pm.solve(np.zeros(200))  # zero rhs: converged at 0 iterations, w = 0
    assert rep.converged and rep.iterations == 0 and not np.any(w)
    b = orc.normals(4, 200)
    w, rep = pm.solve(b)  # max_iters cut-off: least-squares iterate, not converged
    ref = orc.solve(to_checker(orc, x), 0.1, b, "fgmres_twolevel", levels=[dict(target_size=10)], tol=1e-12,
                    max_iters=5)
    assert not rep.converged and rep.iterations == 5 and rel_diff(w, ref.w) <= 1e-10
    bad = b.copy()
    bad[3] = np.nan
    with pytest.raises(ValueError):
        pm.solve(bad)
    with pytest.raises(ValueError):  # two-level method requires one level spec
        R.PreparedMethod(m, 0.1, R.MethodSpec(kind=R.FGMRES_TWOLEVEL))


def test_pair_variant_within_bars(gpu):
    """The persistent inner solver's PAIR variant (even n, A in SMEM: A z summed over
    column pairs) and the plain variant (RMG_DENSE_NO_PAIR=1, read once per process,
    so in a subprocess) are both held to the cfg2_small bars: iterations in the
    envelope, w within its spread."""
    import json
    import os
    import subprocess
    import sys
    code = (
        "import json, sys, numpy as np; sys.path.insert(0, 'tests');"
        "import paper_1806_05826_b200 as R; from helpers import load_golden, rel_diff;"
        "g = load_golden('cfg2_small'); x = R.synth_sparse_zipf(10000, 2000, 40.0, 1.1, False, 0);"
        "lv = [R.LevelSpec(clustering=R.ClusteringChoice(kind=R.IMPORTED, labels=g[f'labels{i}'].astype(np.int64),"
        " n_clusters=k), solver=R.CoarseSolveChoice(kind=R.DIRECT_CHOLESKY if i == 1 else R.INNER_FCG,"
        " tol=1e-6, max_iters=500)) for i, k in enumerate([200, 20])];"
        "pm = R.PreparedMethod(R.DeviceMatrix(x), 1.0, R.MethodSpec(kind=R.FCG_MULTILEVEL, levels=lv,"
        " solver=R.SolverConfig(1e-6, 1000)));"
        "w, rep = pm.solve(g['b']); print(json.dumps([rep.iterations, rel_diff(w, g['ml_w'])]))")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = _envelope("cfg2_small")
    lo, hi = env["ml_iterations_range"]
    for extra in ({}, {"RMG_DENSE_NO_PAIR": "1"}):
        out = subprocess.run([sys.executable, "-c", code], cwd=root, env={**os.environ, **extra},
                             capture_output=True, text=True, timeout=600)
        assert out.returncode == 0, out.stderr[-2000:]
        its, err = json.loads(out.stdout.strip().splitlines()[-1])
        assert lo - 2 <= its <= hi + 2 and err <= env["ml_w_spread"], (extra, its, err, env)
