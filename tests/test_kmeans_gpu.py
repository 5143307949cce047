"""GPU k-means (kmeans_gpu.cu; clustering.cpp:189-355) against the oracle:
labels must be bit-identical, including the k-means++ fallback paths
(duplicated columns: zero total mass), empty-cluster repair, normalized
columns and valued matrices.  Driven through PreparedMethod (the product's
setup path), compared with the oracle restatement pinned to the reference."""
import numpy as np
import pytest

import paper_1806_05826_b200 as R
from helpers import ideal_instance, random_matrix, to_checker

pytestmark = pytest.mark.gpu


def labels_gpu(x, k, seed=0, normalize=False):
    m = R.DeviceMatrix(x, R.default_context())
    lv = R.LevelSpec(clustering=R.ClusteringChoice(kind=R.KMEANS, target_size=k, seed=seed,
                                                   normalize_columns=normalize),
                     solver=R.CoarseSolveChoice(kind=R.DIRECT_CHOLESKY))
    pm = R.PreparedMethod(m, 1e-2, R.MethodSpec(kind=R.FCG_TWOLEVEL, levels=[lv]))
    return pm.labels(0)


@pytest.mark.parametrize("seed", [1, 2, 3, 4])
@pytest.mark.parametrize("normalize", [False, True])
def test_kmeans_random_bit_exact(gpu, orc, seed, normalize):
    x = random_matrix(400, 150, seed, 0.2)
    for k in (7, 30, 149):  # 149 of 150 columns: empty clusters get repaired
        want, _, _ = orc.kmeans(to_checker(orc, x), k, 100, seed, normalize=normalize)
        assert np.array_equal(labels_gpu(x, k, seed, normalize), want), (seed, k, normalize)


@pytest.mark.parametrize("seed", [3, 11, 29])
def test_kmeans_duplicated_columns_bit_exact(gpu, orc, seed):
    """Ideal datasets duplicate columns: once every distinct column is a seed the
    remaining mass is zero and k-means++ falls back to a uniform index draw."""
    x, _, nc = ideal_instance(seed)
    for k in (nc, min(x.n_features - 1, nc + 3)):
        want, _, _ = orc.kmeans(to_checker(orc, x), k, 100, seed)
        assert np.array_equal(labels_gpu(x, k, seed), want), (seed, k)


def test_kmeans_zipf_valued_and_wide_k(gpu, orc):
    """|N(0,1)| values, Zipf columns, K above 256 (several prototypes per thread)."""
    x = R.synth_sparse_zipf(3000, 1500, 12.0, 1.1, True, 5)
    want, _, _ = orc.kmeans(to_checker(orc, x), 600, 100, 0, normalize=True)
    assert np.array_equal(labels_gpu(x, 600, 0, True), want)
