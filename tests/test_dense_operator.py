"""GPU parity of the dense-X path (north-star (1) "row-major
dense for dense inputs"): the operator X^T X is one fused sweep over a
row-major fp64 or fp32-storage X.  The reference stores every input as CSR,
so the oracle runs on the CSR of the same values (fp32 values widen exactly).

Bars as in test_gpu_parity.py: kernels 1e-13 relative, labels bit-exact,
w 1e-8 relative L2, iterations +-2 (goldens from the verbatim reference build).
"""
import numpy as np
import pytest

import paper_1806_05826_b200 as R
from helpers import load_golden, rel_diff, to_checker

pytestmark = pytest.mark.gpu

KERNEL_TOL = 1e-13
W_TOL = 1e-8


def dense_of(x: R.FeatureMatrix) -> np.ndarray:
    return x.dense()


@pytest.mark.parametrize("fp32", [False, True])
@pytest.mark.parametrize("n,f", [(2000, 500), (4097, 1024), (300, 37), (1, 5)])
def test_dense_kernels_match_oracle(gpu, orc, n, f, fp32):
    rng = np.random.default_rng(n * 7 + f)
    a = rng.standard_normal((n, f))
    if fp32:
        a = a.astype(np.float32)
    m = R.DeviceMatrix.from_dense(a)
    assert m.is_dense()
    x = R.from_dense(a.astype(np.float64))  # the same values as CSR for the oracle
    om = to_checker(orc, x)
    v, u = rng.standard_normal(f), rng.standard_normal(n)
    assert rel_diff(m.spmv(v), orc.spmv(om, v)) <= KERNEL_TOL
    assert rel_diff(m.spmv_transpose(u), orc.spmv_transpose(om, u)) <= KERNEL_TOL
    assert rel_diff(m.ridge_apply(0.3, v), orc.ridge_apply(om, 0.3, v)) <= KERNEL_TOL
    assert rel_diff(m.gram_diagonal(0.3), orc.gram_diagonal(om, 0.3)) <= KERNEL_TOL


def test_dense_rejects_wide_matrices(gpu):
    with pytest.raises(ValueError):
        R.DeviceMatrix.from_dense(np.ones((4, 1025)))


def test_cfg1_dense_two_level_matches_reference(gpu):
    """cfg 1 (BASELINE configs[0], dense 2000 x 500) through the dense path:
    same labels, iterations and w as the reference goldens."""
    g = load_golden("cfg1")
    x = R.synth_dense_clustered(2000, 500, 50, 0.1, 0)
    m = R.DeviceMatrix.from_dense(dense_of(x))
    lv = R.LevelSpec(clustering=R.ClusteringChoice(kind=R.KMEANS, target_size=50, seed=0),
                     solver=R.CoarseSolveChoice(kind=R.DIRECT_CHOLESKY))
    pm = R.PreparedMethod(m, 1e-2, R.MethodSpec(kind=R.FCG_TWOLEVEL, levels=[lv]))
    assert np.array_equal(pm.labels(0), g["labels0"])
    w, rep = pm.solve(g["b"])
    assert rep.converged
    assert abs(rep.iterations - int(g["fcg_iterations"])) <= 2
    assert rel_diff(w, g["fcg_w"]) <= W_TOL
    cg = R.solve_system(m, 1e-2, g["b"], R.MethodSpec(kind=R.CG))
    assert abs(cg.report.iterations - int(g["cg_iterations"])) <= 2
    assert rel_diff(cg.w, g["cg_w"]) <= W_TOL


def test_dense_fp32_storage_solve(gpu, orc):
    """fp32 storage, fp64 arithmetic: the solve equals the reference's on the
    fp32-rounded values (BASELINE cfg 4's storage mode, small size)."""
    # spectrum 1 .. 256^-0.25 (kappa ~ 16 with beta): ~40 CG steps, so the
    # count is not at the mercy of summation order (an ill-conditioned variant
    # moved by 4 between two equally valid orders)
    rng = np.random.default_rng(4)
    a = (rng.standard_normal((3000, 256)) @ np.diag(np.arange(1, 257) ** -0.25)).astype(np.float32)
    b = rng.standard_normal(3000)
    m = R.DeviceMatrix.from_dense(a)
    om = to_checker(orc, R.from_dense(a.astype(np.float64)))
    sol = R.solve_system(m, 1e-2, b, R.MethodSpec(kind=R.CG, solver=R.SolverConfig(1e-10, 3000)))
    ref = orc.solve(om, 1e-2, b, "cg", tol=1e-10, max_iters=3000)
    assert abs(sol.report.iterations - ref.iterations) <= 2
    assert rel_diff(sol.w, ref.w) <= W_TOL
