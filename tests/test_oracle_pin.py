"""Pin the CPU oracle (oracle/restatement.cpp) to the reference.

1. Against the golden vectors in tests/golden (produced by the verbatim
   reference build, tests/golden/make_golden.py): the restatement keeps the
   reference's floating-point order, so every comparison here is bit-exact
   (labels, X_c, kernels, iteration counts, residual histories and w).
2. Directly against oracle/_ref (the reference compiled here) on fresh seeded
   inputs, when that build is present.
"""
import numpy as np
import pytest

import oracle
from helpers import golden_matrix, load_golden, random_matrix, to_checker


def _om(orc, g, prefix="x"):
    return to_checker(orc, golden_matrix(g, prefix))


def test_lpsc105_known_answers(orc):
    g = load_golden("lpsc105")
    m = _om(orc, g)
    b, rhs = orc.generate_rhs(m, 42)
    assert np.array_equal(b, g["b"]) and np.array_equal(rhs, g["rhs"])
    assert np.array_equal(orc.ridge_apply(m, 1e-6, g["apply_w"]), g["apply_out"])
    assert np.array_equal(orc.gram_diagonal(m, 1e-6), g["gram_diag"])
    lam, it, _ = orc.lambda_max(m)
    assert lam == float(g["lambda"]) and it == int(g["lambda_iters"])
    s = orc.solve(m, 1e-6, g["b"], "cg", tol=1e-6, max_iters=20000)
    assert s.iterations == int(g["cg_iterations"]) == 66  # proj/test_output.txt:42
    assert np.array_equal(s.w, g["cg_w"]) and np.array_equal(s.residual_history, g["cg_hist"])
    for target in (134, 56):
        lab, nc, exact, tol = orc.leader_follower_target(m, target)
        assert np.array_equal(lab, g[f"lf{target}_labels"]) and nc == int(g[f"lf{target}_nc"])
        assert tol == float(g[f"lf{target}_tol"])
        s = orc.solve(m, 1e-6, g["b"], "fcg_twolevel", levels=[dict(labels=lab, n_clusters=nc)], max_iters=5000)
        assert s.iterations == int(g[f"lf{target}_iterations"])
        assert np.array_equal(s.w, g[f"lf{target}_w"])
    assert int(g["lf134_iterations"]) == 1  # proj/test_output.txt:43


def test_cnae_known_answers(orc):
    g = load_golden("cnae")
    m = _om(orc, g)
    lab, nc = orc.leader_follower(m, 0.5)
    assert nc == 694 and np.array_equal(lab, g["lf_labels"])  # proj/test_output.txt:45-49
    s = orc.solve(m, 1e-6, g["b"], "fcg_twolevel", levels=[dict(labels=lab, n_clusters=nc)], max_iters=5000)
    assert s.iterations == 1 and np.array_equal(s.w, g["lf_w"])
    s = orc.solve(m, 1e-6, g["b"], "cg", tol=1e-6, max_iters=20000)
    assert s.iterations == int(g["cg_iterations"]) == 656  # proj/test_output.txt:64
    assert np.array_equal(s.w, g["cg_w"])


@pytest.mark.parametrize("case", range(5))
def test_random_cases(orc, case):
    g = load_golden("random")
    p = f"r{case}"
    m = _om(orc, g, p)
    beta = float(g[p + "_beta"])
    assert np.array_equal(orc.spmv(m, g[p + "_v"]), g[p + "_spmv"])
    assert np.array_equal(orc.spmv_transpose(m, g[p + "_u"]), g[p + "_spmv_t"])
    assert np.array_equal(orc.ridge_apply(m, beta, g[p + "_v"]), g[p + "_ridge"])
    assert np.array_equal(orc.gram_diagonal(m, beta), g[p + "_diag"])
    lam, it, _ = orc.lambda_max(m)
    assert lam == float(g[p + "_lambda"]) and it == int(g[p + "_lambda_iters"])
    k = int(g[p + "_kpp"].shape[0])
    assert np.array_equal(orc.kmeanspp_seed(m, k, 3), g[p + "_kpp"])
    lab, _, _ = orc.kmeans(m, k, 100, 0)
    assert np.array_equal(lab, g[p + "_km_labels"])
    xc = orc.coarsen(m, lab, k)
    rp, ci, v = xc.export()
    gx = golden_matrix(g, p + "_xc")
    assert np.array_equal(rp, gx.row_offsets) and np.array_equal(ci, gx.column_indices)
    assert np.array_equal(v, gx.values)
    # two-level apply: dense coarse factor rounding is not pinned by the reference
    z = orc.two_level_apply(m, beta, lab, k, 0.37, g[p + "_v"])
    assert np.linalg.norm(z - g[p + "_z"]) <= 1e-12 * np.linalg.norm(g[p + "_z"])
    lv = [dict(clustering_kind=oracle.CLUSTER_KMEANS, target_size=k)]
    for meth in ("cg", "jacobi_cg", "fcg_twolevel"):
        s = orc.solve(m, beta, g[p + "_b"], meth, levels=lv, tol=1e-8, max_iters=2000)
        assert s.iterations == int(g[f"{p}_{meth}_iterations"])
        if meth != "fcg_twolevel":
            assert np.array_equal(s.w, g[f"{p}_{meth}_w"])
        else:
            assert np.linalg.norm(s.w - g[f"{p}_{meth}_w"]) <= 1e-10 * np.linalg.norm(g[f"{p}_{meth}_w"])


def test_cfg1(orc):
    import paper_1806_05826_b200 as R
    g = load_golden("cfg1")
    x = R.synth_dense_clustered(2000, 500, 50, 0.1, 0)
    m = to_checker(orc, x)
    lab, _, _ = orc.kmeans(m, 50, 100, 0)
    assert np.array_equal(lab, g["labels0"])
    s = orc.solve(m, 1e-2, g["b"], "fcg_twolevel", levels=[dict(labels=lab, n_clusters=50)])
    assert s.iterations == int(g["fcg_iterations"])
    assert np.linalg.norm(s.w - g["fcg_w"]) <= 1e-10 * np.linalg.norm(g["fcg_w"])
    s = orc.solve(m, 1e-2, g["b"], "cg")
    assert s.iterations == int(g["cg_iterations"]) and np.array_equal(s.w, g["cg_w"])


def test_cfg2_small_labels_and_solve(orc):
    import paper_1806_05826_b200 as R
    g = load_golden("cfg2_small")
    x = R.synth_sparse_zipf(10000, 2000, 40.0, 1.1, False, 0)
    m = to_checker(orc, x)
    l0, _, _ = orc.kmeans(m, 200, 100, 0, normalize=True)
    assert np.array_equal(l0, g["labels0"].astype(np.int64))
    l1, _, _ = orc.kmeans(orc.coarsen(m, l0, 200), 20, 100, 0, normalize=True)
    assert np.array_equal(l1, g["labels1"].astype(np.int64))
    lv = [dict(labels=l0, n_clusters=200, coarse_kind=oracle.COARSE_INNER_FCG), dict(labels=l1, n_clusters=20)]
    s = orc.solve(m, 1.0, g["b"], "fcg_multilevel", levels=lv)
    assert s.iterations == int(g["ml_iterations"])
    assert np.array_equal(s.inner_iterations.astype(np.int64), g["ml_inner"].astype(np.int64))
    assert np.linalg.norm(s.w - g["ml_w"]) <= 1e-10 * np.linalg.norm(g["ml_w"])


# ---------------------------------------------------------------- oracle vs verbatim reference
@pytest.mark.parametrize("seed", [11, 23, 47])
def test_oracle_equals_reference_build(orc, ref, seed):
    x = random_matrix(60, 40, seed, 0.3)
    mo, mr = to_checker(orc, x), to_checker(ref, x)
    v = np.random.default_rng(seed).standard_normal(40)
    assert np.array_equal(orc.ridge_apply(mo, 0.1, v), ref.ridge_apply(mr, 0.1, v))
    for k in (5, 12):
        lo, io, _ = orc.kmeans(mo, k, 100, seed)
        lr, ir, _ = ref.kmeans(mr, k, 100, seed)
        assert np.array_equal(lo, lr) and io == ir
        lo, _, _ = orc.kmeans(mo, k, 100, seed, normalize=True)
        lr, _, _ = ref.kmeans(mr, k, 100, seed, normalize=True)
        assert np.array_equal(lo, lr)
    lo, nco = orc.leader_follower(mo, 2.0)
    lr, ncr = ref.leader_follower(mr, 2.0)
    assert nco == ncr and np.array_equal(lo, lr)
    b = ref.normals(seed, 60)
    mid = dict(clustering_kind=oracle.CLUSTER_KMEANS, target_size=12, coarse_kind=oracle.COARSE_INNER_FCG)
    last = dict(clustering_kind=oracle.CLUSTER_KMEANS, target_size=5)
    so = orc.solve(mo, 1e-3, b, "fcg_multilevel", levels=[mid, last], tol=1e-8, max_iters=500)
    sr = ref.solve(mr, 1e-3, b, "fcg_multilevel", levels=[mid, last], tol=1e-8, max_iters=500)
    assert so.iterations == sr.iterations
    assert np.linalg.norm(so.w - sr.w) <= 1e-10 * np.linalg.norm(sr.w)
    so = orc.solve(mo, 1e-3, b, "jacobi_cg", tol=1e-10, max_iters=500)
    sr = ref.solve(mr, 1e-3, b, "jacobi_cg", tol=1e-10, max_iters=500)
    assert so.iterations == sr.iterations and np.array_equal(so.w, sr.w)


@pytest.mark.parametrize("seed", [5, 19])
def test_fgmres_restatement_equals_reference_build(orc, ref, seed):
    """fgmres (krylov.cpp:229-328) with the two-level preconditioner: the
    sequential restatement reproduces the reference build bit for bit
    (iterations, residual history, inner counts, w)."""
    x = random_matrix(300, 120, seed, 0.3)
    mo, mr = to_checker(orc, x), to_checker(ref, x)
    b = ref.normals(seed, 300)
    lv = [dict(clustering_kind=oracle.CLUSTER_KMEANS, target_size=20)]
    so = orc.solve(mo, 0.1, b, "fgmres_twolevel", levels=lv, tol=1e-10, max_iters=200)
    sr = ref.solve(mr, 0.1, b, "fgmres_twolevel", levels=lv, tol=1e-10, max_iters=200)
    assert so.converged and so.iterations == sr.iterations
    assert np.array_equal(so.residual_history, sr.residual_history)
    assert np.array_equal(so.w, sr.w)
    # the max_iters cut-off returns the least-squares iterate, not converged
    so = orc.solve(mo, 0.1, b, "fgmres_twolevel", levels=lv, tol=1e-14, max_iters=5)
    sr = ref.solve(mr, 0.1, b, "fgmres_twolevel", levels=lv, tol=1e-14, max_iters=5)
    assert not so.converged and so.iterations == 5 and np.array_equal(so.w, sr.w)
