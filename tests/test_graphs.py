"""Solver loops as CUDA graphs: the device-side while loop runs
the same kernels in the same order as the host loop, so every solve must be
bitwise identical with and without graphs (RMG_NO_GRAPH=1), for every method
the graph path covers, and the inner-solver breakdown must still surface as the
reference's error."""
import os

import numpy as np
import pytest

import paper_1806_05826_b200 as R

pytestmark = pytest.mark.gpu


def lvl(k, kind):
    return R.LevelSpec(clustering=R.ClusteringChoice(kind=R.KMEANS, target_size=k, seed=0), solver=R.CoarseSolveChoice(kind=kind))


def solve(m, beta, spec, b, graphs):
    if not graphs:
        os.environ["RMG_NO_GRAPH"] = "1"
    try:
        pm = R.PreparedMethod(m, beta, spec)
        w, rep = pm.solve(b)
        pm.close()
    finally:
        os.environ.pop("RMG_NO_GRAPH", None)
    return w, rep


@pytest.mark.parametrize("method", ["cg", "jacobi_cg", "fcg_twolevel", "fcg_multilevel", "pcg_vcycle"])
def test_graph_loop_is_bitwise_the_host_loop(gpu, method):
    x = R.synth_sparse_zipf(5000, 700, 20.0, 1.1, True, 8)
    m = R.DeviceMatrix(x)
    levels = {"cg": [], "jacobi_cg": [], "fcg_twolevel": [lvl(60, R.DIRECT_CHOLESKY)],
              "fcg_multilevel": [lvl(90, R.INNER_FCG), lvl(15, R.DIRECT_CHOLESKY)],
              "pcg_vcycle": [lvl(90, R.INNER_FCG), lvl(15, R.DIRECT_CHOLESKY)]}[method]
    spec = R.MethodSpec(kind=R.method_from_string(method), levels=levels, solver=R.SolverConfig(1e-10, 3000))
    b = R.rng_normals(5, 5000)
    w1, r1 = solve(m, 0.3, spec, b, True)
    w2, r2 = solve(m, 0.3, spec, b, False)
    assert r1.converged and r1.iterations == r2.iterations
    assert np.array_equal(w1, w2)
    assert np.array_equal(r1.residual_history, r2.residual_history)
    assert np.array_equal(r1.inner_iterations, r2.inner_iterations)


def test_graph_loop_max_iters_and_repeat(gpu):
    """Stopping at max_iters inside the device loop, and relaunching the same graph."""
    x = R.synth_sparse_zipf(3000, 400, 15.0, 1.1, True, 2)
    m = R.DeviceMatrix(x)
    spec = R.MethodSpec(kind=R.FCG_MULTILEVEL, levels=[lvl(50, R.INNER_FCG), lvl(10, R.DIRECT_CHOLESKY)],
                        solver=R.SolverConfig(1e-14, 7))
    pm = R.PreparedMethod(m, 1e-3, spec)
    b = R.rng_normals(9, 3000)
    w1, r1 = pm.solve(b)
    w2, r2 = pm.solve(b)
    assert r1.iterations == 7 and not r1.converged
    assert r2.iterations == 7 and np.array_equal(w1, w2)
