"""Parity at BASELINE's full sizes through size-independent properties (the
reference cannot run these: SURVEY.md §8(c)).

* cfg 4 (4M x 1024 fp32, the whole config on one GPU): the fused operator against
  an independent fp64 torch computation, symmetry, a valid 128/16 hierarchy, the
  solve's true residual against torch, and bitwise determinism.
* cfg 5 per-GPU shard at 4 GPUs (4M x 500k, 256M binary nonzeros): X v and X^T u
  against numpy gathers / bincounts, linearity and symmetry of X^T X + beta I.
Tolerances: 1e-12 relative for single operator applications (fp64 sums of up to
~4M terms in different orders), the solve's own tolerance (1e-6) for residuals.
"""
import numpy as np
import pytest

import paper_1806_05826_b200 as R

pytestmark = pytest.mark.gpu


def rel(a, b):
    return float(np.linalg.norm(np.asarray(a) - np.asarray(b)) / np.linalg.norm(np.asarray(b)))


def test_cfg4_full_scale(gpu):
    import torch

    import bench
    cfg = bench.CONFIGS["cfg4"]
    a = bench.cfg4_shard_matrix(n=cfg["n"], f=cfg["f"], seed=cfg["seed"])
    n, f = a.shape
    m = R.DeviceMatrix.from_dense(a)
    xd = torch.from_numpy(a).cuda()

    def ata(v, beta):  # independent: fp64 GEMVs over row chunks of the fp32 X (torch / cuBLAS)
        v = torch.from_numpy(v).cuda()
        out = beta * v
        for r in range(0, n, 1 << 19):
            blk = xd[r:r + (1 << 19)].double()
            out += blk.T @ (blk @ v)
        return out.cpu().numpy()

    rng = np.random.default_rng(0)
    u, v = rng.standard_normal(f), rng.standard_normal(f)
    beta = cfg["beta"]
    au, av = m.ridge_apply(beta, u), m.ridge_apply(beta, v)
    assert rel(av, ata(v, beta)) <= 1e-12
    assert abs(u @ av - v @ au) <= 1e-12 * abs(u @ av)

    specs = bench.level_specs(cfg)
    pm = R.PreparedMethod(m, beta, R.MethodSpec(kind=R.FCG_MULTILEVEL, levels=specs,
                                                 solver=R.SolverConfig(cfg["tol"], cfg["max_iters"])))
    for lv, k in enumerate(cfg["ks"]):
        lab = pm.labels(lv)
        assert lab.min() == 0 and lab.max() == k - 1 and len(np.unique(lab)) == k
    b = R.rng_normals(42, n)
    w, rep = pm.solve(b)
    assert rep.converged
    rhs = m.spmv_transpose(b)
    assert rel(ata(w, beta), rhs) <= 1.5 * cfg["tol"]
    w2, rep2 = pm.solve(b)
    assert rep2.iterations == rep.iterations and np.array_equal(w, w2)
    pm.close()
    m.close()


def test_cfg5_shard_operator_full_scale(gpu):
    x = R.synth_sparse_zipf(4_000_000, 500_000, 64.0, 1.05, False, 0, row_streams=True)
    m = R.DeviceMatrix(x)
    assert m.is_pattern
    rp = x.row_offsets.astype(np.int64)
    cols = x.column_indices.astype(np.int64)
    rows = np.repeat(np.arange(x.n_samples), np.diff(rp))
    rng = np.random.default_rng(1)
    v = rng.standard_normal(x.n_features)
    u = rng.standard_normal(x.n_samples)
    xv = np.add.reduceat(v[cols], rp[:-1]) if len(cols) else np.zeros(x.n_samples)
    xv[np.diff(rp) == 0] = 0.0
    assert rel(m.spmv(v), xv) <= 1e-12
    assert rel(m.spmv_transpose(u), np.bincount(cols, weights=u[rows], minlength=x.n_features)) <= 1e-12
    beta = 0.5
    w = rng.standard_normal(x.n_features)
    av, aw = m.ridge_apply(beta, v), m.ridge_apply(beta, w)
    assert rel(m.ridge_apply(beta, 2.0 * v - 3.0 * w), 2.0 * av - 3.0 * aw) <= 1e-12
    assert abs(w @ av - v @ aw) <= 1e-12 * abs(w @ av)
    m.close()
