"""Test fixtures restated from the reference test suite (proj/tests)."""
from __future__ import annotations

import math
import os

import numpy as np

import paper_1806_05826_b200 as R

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


class CounterRng:
    """rng.hpp:25-72 in Python (math.* is glibc libm, like the C++)."""

    M = (1 << 64) - 1

    def __init__(self, seed: int):
        self.seed, self.k, self.spare = seed & self.M, 0, None

    def u64(self) -> int:
        self.k += 1
        z = (self.seed + self.k * 0x9E3779B97F4A7C15) & self.M
        z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & self.M
        z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & self.M
        return z ^ (z >> 31)

    def next_double(self) -> float:
        return float(self.u64() >> 11) * 2.0 ** -53

    def next_double_open(self) -> float:
        return (float(self.u64() >> 11) + 1.0) * 2.0 ** -53

    def next_normal(self) -> float:
        if self.spare is not None:
            s, self.spare = self.spare, None
            return s
        u1, u2 = self.next_double_open(), self.next_double()
        r = math.sqrt(-2.0 * math.log(u1))
        th = 2.0 * math.pi * u2
        self.spare = r * math.sin(th)
        return r * math.cos(th)

    def next_index(self, n: int) -> int:
        v = int(self.next_double() * float(n))
        return n - 1 if v >= n else v


def random_triplets(rows, cols, fill, seed):
    """tests/oracles.hpp:192-203."""
    rng = CounterRng(seed)
    rr, cc, vv = [], [], []
    for r in range(rows):
        for c in range(cols):
            if rng.next_double() < fill:
                rr.append(r), cc.append(c), vv.append(rng.next_normal())
    if not rr:
        rr, cc, vv = [0], [0], [1.0]
    return rr, cc, vv


def random_matrix(rows, cols, seed, fill=0.5) -> R.FeatureMatrix:
    """test_krylov.cpp:13-16."""
    return R.csr_from_triplets(rows, cols, *random_triplets(rows, cols, fill, seed))


def random_base(n, cols, seed) -> R.FeatureMatrix:
    """acceptance.cpp:62-71."""
    rng = CounterRng(seed)
    rr, cc, vv = [], [], []
    for r in range(n):
        for c in range(cols):
            if rng.next_double() < 0.8:
                rr.append(r), cc.append(c), vv.append(rng.next_normal())
    return R.csr_from_triplets(n, cols, rr, cc, vv)


def make_ideal_dataset(base: R.FeatureMatrix, mult, seed):
    """analysis.cpp:79-135: duplicate column j mult[j] times, seeded shuffle.
    Returns (matrix, labels, n_clusters)."""
    source = []
    for j, m in enumerate(mult):
        source += [j] * m
    total = len(source)
    rng = CounterRng(seed)
    for i in range(total, 1, -1):
        j = rng.next_index(i)
        source[i - 1], source[j] = source[j], source[i - 1]
    d = base.dense()
    cols = d[:, source]
    rr, cc = np.nonzero(cols)
    x = R.csr_from_triplets(base.n_samples, total, rr, cc, cols[rr, cc])
    return x, np.asarray(source, np.int64), base.n_features


def ideal_instance(seed):
    """acceptance.cpp:79-89."""
    rng = CounterRng(seed * 7919 + 1)
    f_c = 5 + rng.next_index(36)
    n = f_c + 20
    mult = [1 + rng.next_index(5) for _ in range(f_c)]
    return make_ideal_dataset(random_base(n, f_c, seed * 31 + 7), mult, seed)


def rel_diff(a, b) -> float:
    """tests/oracles.hpp:181-189."""
    a, b = np.asarray(a), np.asarray(b)
    num = float(np.sum((a - b) ** 2))
    den = float(np.sum(b * b))
    return math.sqrt(num) if den == 0.0 else math.sqrt(num / den)


def to_checker(chk, x: R.FeatureMatrix):
    return chk.matrix(x.n_samples, x.n_features, x.row_offsets, x.column_indices, x.value_array())


def dense_gram(x: R.FeatureMatrix, beta: float) -> np.ndarray:
    d = x.dense()
    return d.T @ d + beta * np.eye(x.n_features)


def load_golden(name: str):
    return np.load(os.path.join(GOLDEN, name + ".npz"), allow_pickle=False)


def golden_matrix(g, prefix="x") -> R.FeatureMatrix:
    n, f = (int(v) for v in g[prefix + "_shape"])
    vals = g[prefix + "_values"] if (prefix + "_values") in g.files else None
    return R.FeatureMatrix(n, f, g[prefix + "_row_offsets"].astype(np.uint64),
                           g[prefix + "_column_indices"].astype(np.uint64), vals)
