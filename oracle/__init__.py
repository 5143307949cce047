"""TEST INFRASTRUCTURE ONLY — CPU checkers for the ridgemg solve path.

Two interchangeable CPU implementations share one ctypes surface:

* ``Checker("oracle")`` — this repo's sequential CPU restatement
  (``oracle/restatement.cpp``), always buildable from in-repo sources;
* ``Checker("ref")`` — the reference's own, unmodified sources
  (``/root/reference/proj/src``) compiled with an Eigen-subset shim into
  ``oracle/_ref/libridgemg_ref.so`` (present only where it was built; the
  ``.so`` travels to the GPU box with the gpurun snapshot).

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s cpu_baseline /
``--impl reference`` legs may import this package, and only as the checker or
the timed CPU baseline — never as part of the product path.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass, field

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIBS = {
    "oracle": (os.path.join(HERE, "_build", "libridgemg_oracle.so"), "orc_"),
    "ref": (os.path.join(HERE, "_ref", "libridgemg_ref.so"), "ref_"),
    # rounding-envelope diagnostics only (FMA-contracted restatement, tests/golden/make_envelope.py)
    "oracle_fma": (os.path.join(HERE, "_build", "libridgemg_oracle_fma.so"), "orc_"),
}

CLUSTER_LEADER_TOLERANCE, CLUSTER_LEADER_TARGET, CLUSTER_KMEANS = 0, 1, 2
COARSE_DIRECT, COARSE_INNER_CG, COARSE_INNER_FCG = 0, 1, 2
METHOD_CG, METHOD_JACOBI_CG, METHOD_FCG_TWOLEVEL, METHOD_FCG_MULTILEVEL = 0, 1, 2, 3
METHODS = {"cg": 0, "jacobi_cg": 1, "fcg_twolevel": 2, "fcg_multilevel": 3, "fgmres_twolevel": 4}


class LevelSpec(C.Structure):
    _fields_ = [
        ("clustering_kind", C.c_int32),
        ("tolerance", C.c_double),
        ("target_size", C.c_uint64),
        ("seed", C.c_uint64),
        ("kmeans_max_iters", C.c_uint64),
        ("normalize_columns", C.c_int32),
        ("labels", C.c_void_p),
        ("n_clusters", C.c_uint64),
        ("coarse_kind", C.c_int32),
        ("coarse_tol", C.c_double),
        ("coarse_max_iters", C.c_uint64),
        ("coarse_truncation", C.c_uint64),
        ("has_beta_override", C.c_int32),
        ("beta_override", C.c_double),
    ]


class SolverConfig(C.Structure):
    _fields_ = [("tol", C.c_double), ("max_iters", C.c_uint64), ("truncation", C.c_uint64)]


class SolveReport(C.Structure):
    _fields_ = [
        ("iterations", C.c_uint64),
        ("converged", C.c_int32),
        ("wall_time_s", C.c_double),
        ("residual_history", C.c_void_p),
        ("residual_capacity", C.c_uint64),
        ("inner_iterations", C.c_void_p),
        ("inner_capacity", C.c_uint64),
        ("omega", C.c_double * 8),
        ("level_sizes", C.c_uint64 * 8),
        ("n_levels", C.c_uint64),
    ]


class OracleError(RuntimeError):
    pass


def build(kind: str = "oracle") -> str:
    """Compile a checker library with oracle/Makefile; returns its path."""
    target = {"oracle": "oracle", "ref": "ref", "oracle_fma": "oracle_fma"}[kind]
    subprocess.run(["make", "-s", "-C", HERE, target], check=True)
    return LIBS[kind][0]


def available(kind: str) -> bool:
    return os.path.exists(LIBS[kind][0])


@dataclass
class Solution:
    w: np.ndarray
    iterations: int
    converged: bool
    wall_time_s: float
    residual_history: np.ndarray
    inner_iterations: np.ndarray
    omega: list = field(default_factory=list)
    level_sizes: list = field(default_factory=list)


def _p(a):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


class Matrix:
    def __init__(self, chk: "Checker", handle: int):
        self.chk, self.h = chk, C.c_void_p(handle)
        n, f, z = C.c_uint64(), C.c_uint64(), C.c_uint64()
        chk._fn("matrix_shape")(self.h, C.byref(n), C.byref(f), C.byref(z))
        self.n_samples, self.n_features, self.nnz = n.value, f.value, z.value

    def __del__(self):
        try:
            self.chk._fn("matrix_free")(self.h)
        except Exception:
            pass

    def export(self):
        rp = np.zeros(self.n_samples + 1, np.uint64)
        ci = np.zeros(self.nnz, np.uint64)
        v = np.zeros(self.nnz, np.float64)
        self.chk._fn("matrix_export")(self.h, _p(rp), _p(ci), _p(v))
        return rp, ci, v


class Checker:
    def __init__(self, kind: str = "oracle"):
        path, self.prefix = LIBS[kind]
        if not os.path.exists(path):
            build(kind)
        self.kind = kind
        self.lib = C.CDLL(path)
        for name in ("matrix_from_csr", "coarsen", "synth_sparse_zipf", "synth_dense_clustered") + (("read_matrix_market", "matrix_from_triplets") if kind == "ref" else ()):
            getattr(self.lib, self.prefix + name).restype = C.c_void_p
        getattr(self.lib, self.prefix + "last_error").restype = C.c_char_p

    def _fn(self, name):
        return getattr(self.lib, self.prefix + name)

    def _check(self, rc):
        if rc != 0:
            msg = self._fn("last_error")().decode()
            if rc == 1:
                raise ValueError(msg)
            raise OracleError(msg)

    def set_num_threads(self, t: int):
        self._fn("set_num_threads")(C.c_uint(t))

    # ------------------------------------------------------------ matrices
    def matrix(self, n, f, row_offsets, column_indices, values=None) -> Matrix:
        rp = np.ascontiguousarray(row_offsets, np.uint64)
        ci = np.ascontiguousarray(column_indices, np.uint64)
        v = None if values is None else np.ascontiguousarray(values, np.float64)
        h = self._fn("matrix_from_csr")(C.c_uint64(n), C.c_uint64(f), C.c_uint64(len(ci)), _p(rp), _p(ci), _p(v))
        return Matrix(self, h)

    def synth_sparse_zipf(self, n, f, mean_nnz, zipf_s, abs_normal_values, seed, row_streams=False) -> Matrix:
        """BASELINE cfg 2/3/5 generator (oracle/synth.hpp) on this checker's CounterRng."""
        h = self._fn("synth_sparse_zipf")(C.c_uint64(n), C.c_uint64(f), C.c_double(mean_nnz), C.c_double(zipf_s),
                                          C.c_int32(int(abs_normal_values)), C.c_uint64(seed),
                                          C.c_int32(int(row_streams)))
        return Matrix(self, h)

    def synth_dense_clustered(self, n, f, groups, noise, seed) -> Matrix:
        """BASELINE cfg 1 generator (oracle/synth.hpp)."""
        h = self._fn("synth_dense_clustered")(C.c_uint64(n), C.c_uint64(f), C.c_uint64(groups), C.c_double(noise),
                                              C.c_uint64(seed))
        return Matrix(self, h)

    def read_matrix_market(self, path: str) -> Matrix:
        h = self.lib.ref_read_matrix_market(path.encode())
        if not h:
            self._check(2)
        return Matrix(self, h)

    def from_triplets(self, n, f, rows, cols, vals) -> Matrix:
        r = np.ascontiguousarray(rows, np.uint64)
        c = np.ascontiguousarray(cols, np.uint64)
        v = np.ascontiguousarray(vals, np.float64)
        h = self.lib.ref_matrix_from_triplets(C.c_uint64(n), C.c_uint64(f), C.c_uint64(len(r)), _p(r), _p(c), _p(v))
        if not h:
            self._check(1)
        return Matrix(self, h)

    # ------------------------------------------------------------ kernels
    def spmv(self, m: Matrix, v):
        v = np.ascontiguousarray(v, np.float64)
        y = np.zeros(m.n_samples)
        self._check(self._fn("spmv")(m.h, _p(v), _p(y)))
        return y

    def spmv_transpose(self, m: Matrix, u):
        u = np.ascontiguousarray(u, np.float64)
        y = np.zeros(m.n_features)
        self._check(self._fn("spmv_transpose")(m.h, _p(u), _p(y)))
        return y

    def ridge_apply(self, m: Matrix, beta: float, w):
        w = np.ascontiguousarray(w, np.float64)
        out = np.zeros(m.n_features)
        self._check(self._fn("ridge_apply")(m.h, C.c_double(beta), _p(w), _p(out)))
        return out

    def gram_diagonal(self, m: Matrix, beta: float):
        out = np.zeros(m.n_features)
        self._check(self._fn("gram_diagonal")(m.h, C.c_double(beta), _p(out)))
        return out

    def lambda_max(self, m: Matrix, tol=1e-4, max_iters=200, seed=0x5EED):
        v, it, cv = C.c_double(), C.c_uint64(), C.c_int32()
        self._check(self._fn("lambda_max")(m.h, C.c_double(tol), C.c_uint64(max_iters), C.c_uint64(seed),
                                           C.byref(v), C.byref(it), C.byref(cv)))
        return v.value, it.value, bool(cv.value)

    def normals(self, seed: int, n: int):
        out = np.zeros(n)
        self._fn("normals")(C.c_uint64(seed), C.c_uint64(n), _p(out))
        return out

    def generate_rhs(self, m: Matrix, seed: int):
        b = np.zeros(m.n_samples)
        rhs = np.zeros(m.n_features)
        self._check(self._fn("generate_rhs")(m.h, C.c_uint64(seed), _p(b), _p(rhs)))
        return b, rhs

    # ------------------------------------------------------------ clustering
    def kmeanspp_seed(self, m: Matrix, k: int, seed: int):
        out = np.zeros(k, np.int64)
        self._check(self._fn("kmeanspp_seed")(m.h, C.c_uint64(k), C.c_uint64(seed), _p(out)))
        return out

    def kmeans(self, m: Matrix, k: int, max_iters=100, seed=0, normalize=False):
        lab = np.zeros(m.n_features, np.int64)
        it, cv = C.c_uint64(), C.c_int32()
        self._check(self._fn("kmeans")(m.h, C.c_uint64(k), C.c_uint64(max_iters), C.c_uint64(seed),
                                       C.c_int32(int(normalize)), _p(lab), C.byref(it), C.byref(cv)))
        return lab, it.value, bool(cv.value)

    def leader_follower(self, m: Matrix, tol: float):
        lab = np.zeros(m.n_features, np.int64)
        nc = C.c_uint64()
        self._check(self._fn("leader_follower")(m.h, C.c_double(tol), _p(lab), C.byref(nc)))
        return lab, nc.value

    def leader_follower_target(self, m: Matrix, target: int):
        lab = np.zeros(m.n_features, np.int64)
        nc, ex, tol = C.c_uint64(), C.c_int32(), C.c_double()
        self._check(self._fn("leader_follower_target")(m.h, C.c_uint64(target), _p(lab), C.byref(nc),
                                                       C.byref(ex), C.byref(tol)))
        return lab, nc.value, bool(ex.value), tol.value

    def coarsen(self, m: Matrix, labels, n_clusters: int, beta: float = 0.0) -> Matrix:
        lab = np.ascontiguousarray(labels, np.int64)
        h = self._fn("coarsen")(m.h, _p(lab), C.c_uint64(n_clusters), C.c_double(beta))
        if not h:
            self._check(1)
        return Matrix(self, h)

    def two_level_apply(self, m: Matrix, beta, labels, n_clusters, omega, r):
        lab = np.ascontiguousarray(labels, np.int64)
        r = np.ascontiguousarray(r, np.float64)
        z = np.zeros(m.n_features)
        self._check(self._fn("two_level_apply")(m.h, C.c_double(beta), _p(lab), C.c_uint64(n_clusters),
                                                C.c_double(omega), _p(r), _p(z)))
        return z

    # ------------------------------------------------------------ solve
    def solve(self, m: Matrix, beta: float, b, method="cg", levels=(), tol=1e-6, max_iters=1000,
              truncation=20) -> Solution:
        """PreparedMethod(x, beta, spec).solve(b) (krylov.cpp:617-668).

        ``levels`` is a sequence of dicts with LevelSpec field names; a
        ``labels`` entry (int64 array) imports the clustering for that level.
        """
        keep = []
        arr = (LevelSpec * max(1, len(levels)))()
        for i, lv in enumerate(levels):
            s = arr[i]
            s.clustering_kind = lv.get("clustering_kind", CLUSTER_KMEANS)
            s.tolerance = lv.get("tolerance", 1.0)
            s.target_size = lv.get("target_size", 0)
            s.seed = lv.get("seed", 0)
            s.kmeans_max_iters = lv.get("kmeans_max_iters", 100)
            s.normalize_columns = int(lv.get("normalize_columns", False))
            if lv.get("labels") is not None:
                lab = np.ascontiguousarray(lv["labels"], np.int64)
                keep.append(lab)
                s.labels = lab.ctypes.data
                s.n_clusters = int(lv["n_clusters"])
            s.coarse_kind = lv.get("coarse_kind", COARSE_DIRECT)
            s.coarse_tol = lv.get("coarse_tol", 1e-6)
            s.coarse_max_iters = lv.get("coarse_max_iters", 500)
            s.coarse_truncation = lv.get("coarse_truncation", 20)
            if lv.get("beta_override") is not None:
                s.has_beta_override = 1
                s.beta_override = lv["beta_override"]
        b = np.ascontiguousarray(b, np.float64)
        w = np.zeros(m.n_features)
        hist = np.zeros(max_iters + 1)
        inner = np.zeros(max_iters + 1, np.uint64)
        rep = SolveReport()
        rep.residual_history = hist.ctypes.data
        rep.residual_capacity = len(hist)
        rep.inner_iterations = inner.ctypes.data
        rep.inner_capacity = len(inner)
        cfg = SolverConfig(tol, max_iters, truncation)
        mk = METHODS[method] if isinstance(method, str) else int(method)
        self._check(self._fn("solve")(m.h, C.c_double(beta), C.c_int32(mk), arr, C.c_uint64(len(levels)),
                                      C.byref(cfg), _p(b), _p(w), C.byref(rep)))
        it = rep.iterations
        nl = rep.n_levels
        return Solution(w=w, iterations=it, converged=bool(rep.converged), wall_time_s=rep.wall_time_s,
                        residual_history=hist[:it].copy(),
                        inner_iterations=inner[:it].copy() if mk >= 2 else np.zeros(0, np.uint64),
                        omega=list(rep.omega[: max(0, nl - 1)]), level_sizes=list(rep.level_sizes[:nl]))


# ---------------------------------------------------------------- bench harness
def describe_clustering(level: dict, coarse_size: int) -> str:
    """describe_clustering (krylov.cpp:596-612) for a checker level dict."""
    kind = level.get("clustering_kind", CLUSTER_KMEANS)
    if level.get("labels") is not None:
        return f"imported(fc={coarse_size})"
    if kind == CLUSTER_LEADER_TOLERANCE:
        return f"lf(tol={level.get('tolerance', 1.0):g},fc={coarse_size})"
    if kind == CLUSTER_LEADER_TARGET:
        return f"lf(fc={coarse_size})"
    return f"km(k={coarse_size})"


def compare_methods(chk: Checker, m: Matrix, dataset: str, beta_grid, tol_grid, methods, n_repeats=1,
                    rhs_seed=42):
    """analysis.cpp:137-211 on a checker: for every (beta, tol) the plain-CG baseline
    (max_iters = max(20000, 4F)) and every method of `methods` -- (name, levels)
    pairs with checker level dicts -- solved for generate_rhs(x, rhs_seed).b, wall
    time averaged over n_repeats (the solver's own timer); rows as dicts in the
    reference's CSV schema (dataset, method, clustering, f_c, beta, tol, iterations,
    wall_time_s, speedup)."""
    if not beta_grid or not tol_grid:
        raise ValueError("compare_methods: beta and tol grids must be non-empty")
    if not methods:
        raise ValueError("compare_methods: method list must be non-empty")
    b, _ = chk.generate_rhs(m, rhs_seed)
    rows = []
    for beta in beta_grid:
        for tol in tol_grid:
            cg_t, cg = 0.0, None
            for _ in range(n_repeats):
                cg = chk.solve(m, beta, b, "cg", tol=tol, max_iters=max(20000, 4 * m.n_features))
                cg_t += cg.wall_time_s
            cg_t /= n_repeats
            for name, levels in methods:
                row = dict(dataset=dataset, method=name, clustering="", f_c=0, beta=beta, tol=tol)
                if name == "cg":
                    rows.append(dict(row, iterations=cg.iterations, wall_time_s=cg_t, speedup=1.0))
                    continue
                t, s = 0.0, None
                for _ in range(n_repeats):
                    s = chk.solve(m, beta, b, name, levels=levels, tol=tol)
                    t += s.wall_time_s
                t /= n_repeats
                fc = int(s.level_sizes[1]) if len(s.level_sizes) > 1 else 0
                rows.append(dict(row, clustering=describe_clustering(levels[0], fc) if levels else "", f_c=fc,
                                 iterations=s.iterations, wall_time_s=t, speedup=cg_t / t if t > 0 else 0.0))
    return rows
