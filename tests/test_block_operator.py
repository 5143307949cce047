"""Block operator (BASELINE cfg 3's k right-hand sides as one SpMM; DESIGN.md
§4.8): every column of X^T (X V) + beta V equals the single-vector operator
(and the oracle) up to summation order."""
import numpy as np
import pytest

import paper_1806_05826_b200 as R
from helpers import rel_diff, to_checker

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("values", [False, True])
@pytest.mark.parametrize("k", [1, 5, 16, 23, 40])
def test_block_matches_columns(gpu, orc, values, k):
    x = R.synth_sparse_zipf(6000, 900, 18.0, 1.1, values, 3)  # long Zipf rows: multi-item X^T rows
    m = R.DeviceMatrix(x, R.default_context())
    v = np.random.default_rng(k).standard_normal((x.n_features, k))
    out = m.ridge_apply_block(0.7, v)
    om = to_checker(orc, x)
    for q in range(k):
        want = orc.ridge_apply(om, 0.7, v[:, q].copy())
        assert rel_diff(out[:, q], want) <= 1e-13, (q, rel_diff(out[:, q], want))


@pytest.mark.parametrize("values", [True, False])
@pytest.mark.parametrize("k", [5, 16, 23])
def test_block_relabeled_wide(gpu, orc, values, k):
    """F = 30000 > 24576: K1 runs on popularity-relabeled columns (V rows permuted);
    its 1400 most popular labels come from shared memory (k_spmm_hot), the rest from
    the cold SELL pass, and the hot X^T features from shared-memory T blocks."""
    x = R.synth_sparse_zipf(20000, 30000, 12.0, 1.05, values, 8)
    m = R.DeviceMatrix(x, R.default_context())
    v = np.random.default_rng(2).standard_normal((x.n_features, k))
    out = m.ridge_apply_block(0.3, v)
    om = to_checker(orc, x)
    for q in sorted({0, k // 2, k - 1}):
        assert rel_diff(out[:, q], orc.ridge_apply(om, 0.3, v[:, q].copy())) <= 1e-13


def test_block_errors(gpu):
    x = R.synth_sparse_zipf(500, 60, 5.0, 1.1, False, 1)
    m = R.DeviceMatrix(x, R.default_context())
    with pytest.raises(ValueError):
        m.ridge_apply_block(0.1, np.zeros((60, 65)))
    with pytest.raises(ValueError):
        m.ridge_apply_block(-1.0, np.zeros((60, 4)))


@pytest.mark.parametrize("fp32", [False, True])
@pytest.mark.parametrize("shape,k", [((3000, 130), 16), ((517, 64), 5), ((2000, 1000), 23), ((40, 7), 1)])
def test_dense_block_matches_numpy(gpu, fp32, shape, k):
    """Dense X, k right-hand sides: G = X^T X formed once on the FP64
    tensor cores (DMMA SYRK), each apply G V + beta V a DMMA skinny GEMM."""
    rng = np.random.default_rng(shape[0] + k)
    a = rng.standard_normal(shape)
    if fp32:
        a = a.astype(np.float32)
    m = R.DeviceMatrix.from_dense(a)
    v = rng.standard_normal((shape[1], k))
    a64 = a.astype(np.float64)
    for beta in (0.7, 1e-3):  # the second apply reuses G
        out = m.ridge_apply_block(beta, v)
        want = a64.T @ (a64 @ v) + beta * v
        assert rel_diff(out, want) <= 1e-12, rel_diff(out, want)
        col = m.ridge_apply(beta, v[:, k // 2].copy())
        assert rel_diff(out[:, k // 2], col) <= 1e-12


def _triplet_matrix(n, f, nnz, seed, skew):
    """A ragged matrix from numpy triplets: empty rows, rows with hot entries only, rows
    with cold entries only (column popularity ~ rank^-skew), n not a multiple of 8."""
    rng = np.random.default_rng(seed)
    p = (np.arange(1, f + 1, dtype=np.float64)) ** -skew
    p /= p.sum()
    rows = rng.integers(0, n, nnz)
    rows[rows % 7 == 3] = 0  # one very long row; every 7th row stays empty
    cols = rng.choice(f, size=nnz, p=p)
    key = np.unique(rows.astype(np.int64) * f + cols)
    rr, cc = key // f, key % f
    vv = rng.standard_normal(len(key))
    return R.csr_from_triplets(n, f, rr.tolist(), cc.tolist(), vv.tolist()), (rr, cc, vv)


@pytest.mark.parametrize("n,f,nnz,skew", [(3001, 25000, 40_000, 1.0), (20011, 26000, 600_000, 1.2),
                                          (1029, 24600, 3_000, 0.5)])
@pytest.mark.parametrize("k", [16, 7])
def test_block_ragged_relabeled(gpu, n, f, nnz, skew, k):
    """The record-streaming K1 (hot labels from shared memory + cold gathers) and the
    hot X^T blocks on ragged inputs: empty rows, one row holding a seventh of the
    nonzeros, a partial last slice / window / sample block; checked against numpy."""
    x, (rr, cc, vv) = _triplet_matrix(n, f, nnz, n + k, skew)
    m = R.DeviceMatrix(x, R.default_context())
    v = np.random.default_rng(5).standard_normal((f, k))
    out = m.ridge_apply_block(0.25, v)
    t = np.zeros((n, k))
    np.add.at(t, rr, vv[:, None] * v[cc])
    want = np.zeros((f, k))
    np.add.at(want, cc, vv[:, None] * t[rr])
    want += 0.25 * v
    assert rel_diff(out, want) <= 1e-12, rel_diff(out, want)
    assert np.array_equal(out, m.ridge_apply_block(0.25, v))  # run-to-run bitwise
