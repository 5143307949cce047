"""Concurrent solves (krylov.hpp:172-175: prepared methods are immutable and
accept concurrent solves with distinct right-hand sides): every C-ABI call
holds its context, so threads sharing a prepared method -- or two methods
sharing a matrix -- get exactly the sequential results."""
import threading

import numpy as np
import pytest

import paper_1806_05826_b200 as R
from helpers import random_matrix

pytestmark = pytest.mark.gpu


def test_concurrent_solves_match_sequential(gpu):
    x = random_matrix(600, 200, 9, 0.3)
    m = R.DeviceMatrix(x, R.default_context())
    lv = R.LevelSpec(clustering=R.ClusteringChoice(kind=R.KMEANS, target_size=20),
                     solver=R.CoarseSolveChoice(kind=R.DIRECT_CHOLESKY))
    pm = R.PreparedMethod(m, 1e-2, R.MethodSpec(kind=R.FCG_TWOLEVEL, levels=[lv], solver=R.SolverConfig(1e-10, 500)))
    pc = R.PreparedMethod(m, 1e-2, R.MethodSpec(kind=R.CG, solver=R.SolverConfig(1e-10, 2000)))
    bs = [R.rng_normals(100 + i, 600) for i in range(8)]
    want = [(pm.solve(b)[0], pc.solve(b)[0]) for b in bs]
    got = [None] * len(bs)
    errors = []

    def work(i):
        try:
            for _ in range(3):
                got[i] = (pm.solve(bs[i])[0], pc.solve(bs[i])[0])
        except Exception as e:  # pragma: no cover - reported below
            errors.append(e)

    ts = [threading.Thread(target=work, args=(i,)) for i in range(len(bs))]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    assert not errors, errors
    for (a, b), (c, d) in zip(got, want):
        assert np.array_equal(a, c) and np.array_equal(b, d)


def test_solve_batch_equals_single_solves(gpu):
    x = random_matrix(500, 150, 4, 0.3)
    m = R.DeviceMatrix(x, R.default_context())
    lv = R.LevelSpec(clustering=R.ClusteringChoice(kind=R.KMEANS, target_size=15),
                     solver=R.CoarseSolveChoice(kind=R.DIRECT_CHOLESKY))
    pm = R.PreparedMethod(m, 1e-2, R.MethodSpec(kind=R.FCG_TWOLEVEL, levels=[lv], solver=R.SolverConfig(1e-10, 500)))
    B = np.stack([R.rng_normals(10 + q, 500) for q in range(5)], axis=1)
    W, reps = pm.solve_batch(B)
    assert W.shape == (150, 5) and len(reps) == 5
    for q in range(5):
        w, rep = pm.solve(B[:, q])
        assert np.array_equal(W[:, q], w) and reps[q].iterations == rep.iterations
        assert np.array_equal(reps[q].residual_history, rep.residual_history)
