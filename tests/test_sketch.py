"""Sketched k-means (RMG_CLUSTER_KMEANS_SKETCH): the reference's
k-means (clustering.cpp:189-355) applied to S = G^T X, G a seeded N x d sign
matrix.  Bars: S is reproduced here in numpy (sequential sums in increasing row
order, np.cumsum), and the labels equal the oracle's k-means of that S bit for
bit, for sparse (CSR) and dense (device-resident) levels."""
import numpy as np
import pytest

import paper_1806_05826_b200 as R
from helpers import random_matrix, to_checker

pytestmark = pytest.mark.gpu


def sketch_signs(seed, n, d):
    with np.errstate(over="ignore"):
        r = np.arange(n, dtype=np.uint64)[:, None]
        c = np.arange(d, dtype=np.uint64)[None, :]
        z = np.uint64(seed ^ 0xC0FFEE5CE7C4) + (r * np.uint64(d) + c + np.uint64(1)) * np.uint64(0x9E3779B97F4A7C15)
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        z ^= z >> np.uint64(31)
    return np.where((z >> np.uint64(63)) != 0, -1.0, 1.0)


def sketch_numpy(x: R.FeatureMatrix, seed, d, normalize):
    g = sketch_signs(seed, x.n_samples, d)
    rows = np.repeat(np.arange(x.n_samples), np.diff(x.row_offsets.astype(np.int64)))
    cols = x.column_indices.astype(np.int64)
    vals = x.value_array()
    order = np.lexsort((rows, cols))  # by column, rows increasing
    s = np.zeros((d, x.n_features))
    starts = np.searchsorted(cols[order], np.arange(x.n_features + 1))
    for j in range(x.n_features):
        q = order[starts[j]:starts[j + 1]]
        if len(q) == 0:
            continue
        v = vals[q]
        if normalize:
            v = v / np.sqrt(np.cumsum(v * v)[-1])
        s[:, j] = np.cumsum(v[:, None] * g[rows[q], :], axis=0)[-1]
    return s


def sketch_labels(m, k, seed, d, normalize):
    lv = R.LevelSpec(clustering=R.ClusteringChoice(kind=R.KMEANS_SKETCH, target_size=k, seed=seed, sketch_dim=d,
                                                   normalize_columns=normalize),
                     solver=R.CoarseSolveChoice(kind=R.DIRECT_CHOLESKY))
    return R.PreparedMethod(m, 1e-2, R.MethodSpec(kind=R.FCG_TWOLEVEL, levels=[lv])).labels(0)


@pytest.mark.parametrize("normalize", [False, True])
@pytest.mark.parametrize("d,k", [(32, 9), (7, 40), (32, 120)])
def test_sketch_labels_sparse(gpu, orc, normalize, d, k):
    x = random_matrix(500, 150, 3 + d, 0.1)
    s = sketch_numpy(x, 5, d, normalize)
    want, _, _ = orc.kmeans(to_checker(orc, R.from_dense(s)), k, 100, 5)
    assert np.array_equal(sketch_labels(R.DeviceMatrix(x), k, 5, d, normalize), want)


@pytest.mark.parametrize("normalize", [False, True])
def test_sketch_labels_dense(gpu, orc, normalize):
    a = np.random.default_rng(4).standard_normal((700, 90))
    a[:, 3] = 0.0
    x = R.from_dense(a)
    s = sketch_numpy(x, 11, 32, normalize)
    want, _, _ = orc.kmeans(to_checker(orc, R.from_dense(s)), 15, 100, 11)
    assert np.array_equal(sketch_labels(R.DeviceMatrix.from_dense(a), 15, 11, 32, normalize), want)


def test_sketch_rejects_bad_dimension(gpu):
    x = random_matrix(50, 20, 1, 0.3)
    with pytest.raises(ValueError):
        sketch_labels(R.DeviceMatrix(x), 4, 0, 33, False)
