"""GPU parity of the hybrid X^T pass: the hot features summed
per sample block from an SMEM copy of t, the cold rest by the segmented K2,
then the shared epilogue.  By default the path only engages for N >= 296 x 4096
samples; RMG_XT_HOT=1 forces it on matrices small enough for the oracle
(296 blocks of a few dozen samples, hot = >= 4 nonzeros per block).

Bars as in test_gpu_parity.py: kernels 1e-13 relative, w 1e-8, iterations +-2.
"""
import os

import numpy as np
import pytest

import paper_1806_05826_b200 as R
from helpers import rel_diff, to_checker

pytestmark = pytest.mark.gpu


@pytest.fixture(params=["unchunked", "chunked"])
def hybrid(monkeypatch, request):
    """Both cold-pass layouts: one segmented pass, and the sample-chunked passes
    (the default above 8 M samples) forced with chunks of 3000 samples."""
    monkeypatch.setenv("RMG_XT_HOT", "1")
    if request.param == "chunked":
        monkeypatch.setenv("RMG_XT_CHUNK", "1")
        monkeypatch.setenv("RMG_XT_CHUNK_ROWS", "3000")
    yield
    for k in ("RMG_XT_HOT", "RMG_XT_CHUNK", "RMG_XT_CHUNK_ROWS"):
        monkeypatch.delenv(k, raising=False)


def zipf(n, f, mean, s, values, seed):
    return R.synth_sparse_zipf(n, f, mean, s, values, seed)


@pytest.mark.parametrize("values", [False, True])
@pytest.mark.parametrize("n,f", [(30000, 2000), (12000, 70000)])
def test_hybrid_operator_matches_oracle(gpu, orc, hybrid, n, f, values):
    x = zipf(n, f, 24.0, 1.1, values, 7)
    m = R.DeviceMatrix(x, R.default_context())
    om = to_checker(orc, x)
    rng = np.random.default_rng(3)
    u = rng.standard_normal(n)
    w = rng.standard_normal(f)
    assert rel_diff(m.spmv_transpose(u), orc.spmv_transpose(om, u)) <= 1e-13
    assert rel_diff(m.ridge_apply(0.5, w), orc.ridge_apply(om, 0.5, w)) <= 1e-13


def test_hybrid_engages_and_matches_plain_path(gpu, orc, monkeypatch):
    """Same matrix, hybrid forced on vs off: identical within rounding; the hot
    part really ran (its K2 launches show in the operator profile)."""
    x = zipf(20000, 3000, 32.0, 1.05, False, 11)
    u = np.random.default_rng(5).standard_normal(20000)
    monkeypatch.setenv("RMG_XT_HOT", "0")
    plain = R.DeviceMatrix(x, R.default_context()).spmv_transpose(u)
    monkeypatch.setenv("RMG_XT_HOT", "1")
    m = R.DeviceMatrix(x, R.default_context())
    hyb = m.spmv_transpose(u)
    assert rel_diff(hyb, plain) <= 1e-13
    assert m.hybrid_hot_features() > 0


def test_hybrid_cg_and_fcg_solves(gpu, orc, hybrid):
    # beta = 128 keeps the Zipf system's CG at ~70 iterations (at beta = 1 it takes
    # 180 and a different summation tree moves the count by 3: rounding, not parity)
    beta = 128.0
    x = zipf(24000, 1500, 20.0, 1.1, False, 13)
    b = R.rng_normals(9, 24000)
    m = R.DeviceMatrix(x, R.default_context())
    om = to_checker(orc, x)
    cg = R.solve_system(m, beta, b, R.MethodSpec(kind=R.CG, solver=R.SolverConfig(1e-10, 2000)))
    ref = orc.solve(om, beta, b, "cg", tol=1e-10, max_iters=2000)
    assert abs(cg.report.iterations - ref.iterations) <= 2
    assert rel_diff(cg.w, ref.w) <= 1e-8
    lv = [R.LevelSpec(clustering=R.ClusteringChoice(kind=R.KMEANS, target_size=60, seed=0),
                      solver=R.CoarseSolveChoice(kind=R.DIRECT_CHOLESKY))]
    fcg = R.solve_system(m, beta, b, R.MethodSpec(kind=R.FCG_TWOLEVEL, levels=lv,
                                                  solver=R.SolverConfig(1e-10, 2000)))
    reff = orc.solve(om, beta, b, "fcg_twolevel", levels=[dict(target_size=60)], tol=1e-10, max_iters=2000)
    assert abs(fcg.report.iterations - reff.iterations) <= 2
    assert rel_diff(fcg.w, reff.w) <= 1e-8
