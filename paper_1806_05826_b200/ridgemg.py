"""Python mirror of the reference's solver interface (proj/include/ridgemg),
backed by the B200 C ABI (include/ridgemg_b200.h).

Names, argument meanings and error types follow the reference:
``ValueError`` where it throws ``std::invalid_argument`` and ``RuntimeError``
where it throws ``std::runtime_error``; non-convergence is reported through
``SolveReport.converged``.  Every numerical call runs on the GPU; there is no
CPU code path here.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from typing import Optional, Sequence

import numpy as np

from . import _lib

# ---------------------------------------------------------------- enums (krylov.hpp)
CG, JACOBI_CG, FCG_TWOLEVEL, FCG_MULTILEVEL, FGMRES_TWOLEVEL, PCG_VCYCLE, PCG_VCYCLE_ADDITIVE = 0, 1, 2, 3, 4, 5, 6
METHOD_NAMES = {"cg": CG, "jacobi_cg": JACOBI_CG, "fcg_twolevel": FCG_TWOLEVEL, "fcg_multilevel": FCG_MULTILEVEL,
                "fgmres_twolevel": FGMRES_TWOLEVEL,
                "pcg_vcycle": PCG_VCYCLE,  # extension: symmetric Jacobi-smoothed V-cycle
                "pcg_vcycle_additive": PCG_VCYCLE_ADDITIVE}  # extension: additive finest level (§4.15)
LEADER_TOLERANCE, LEADER_TARGET, KMEANS, KMEANS_SKETCH, IMPORTED = 0, 1, 2, 3, 100
DIRECT_CHOLESKY, INNER_CG, INNER_FCG = 0, 1, 2


def method_from_string(s: str) -> int:
    """krylov.cpp:574-581 (fgmres_twolevel is out of scope here)."""
    if s not in METHOD_NAMES:
        raise ValueError(f"unknown method: '{s}'")
    return METHOD_NAMES[s]


def _ptr(a: Optional[np.ndarray]):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


# ---------------------------------------------------------------- data (sparse.hpp)
@dataclass
class FeatureMatrix:
    """CSR sample-by-feature matrix (sparse.hpp:24-32); values None = binary pattern."""

    n_samples: int
    n_features: int
    row_offsets: np.ndarray
    column_indices: np.ndarray
    values: Optional[np.ndarray] = None

    @property
    def nnz(self) -> int:
        return int(len(self.column_indices))

    def dense(self) -> np.ndarray:
        d = np.zeros((self.n_samples, self.n_features))
        rows = np.repeat(np.arange(self.n_samples), np.diff(self.row_offsets).astype(np.int64))
        d[rows, self.column_indices.astype(np.int64)] = 1.0 if self.values is None else self.values
        return d

    def value_array(self) -> np.ndarray:
        return np.ones(self.nnz) if self.values is None else self.values


def csr_from_triplets(n_samples: int, n_features: int, rows, cols, vals) -> FeatureMatrix:
    """sparse.cpp:27-73: validate, sort by (row, col), sum duplicates in input order."""
    rows = np.asarray(rows, np.int64)
    cols = np.asarray(cols, np.int64)
    vals = np.asarray(vals, np.float64)
    if len(rows) and (rows.min() < 0 or rows.max() >= n_samples or cols.min() < 0 or cols.max() >= n_features):
        raise ValueError(f"csr_from_triplets: entry outside {n_samples}x{n_features}")
    if not np.all(np.isfinite(vals)):
        raise ValueError("csr_from_triplets: non-finite value")
    order = np.lexsort((cols, rows))  # stable: duplicates keep input order
    r, c, v = rows[order], cols[order], vals[order]
    keep_c, keep_v, keep_r = [], [], []
    for i in range(len(r)):
        if keep_r and keep_r[-1] == r[i] and keep_c[-1] == c[i]:
            keep_v[-1] += v[i]
        else:
            keep_r.append(r[i])
            keep_c.append(c[i])
            keep_v.append(v[i])
    rp = np.zeros(n_samples + 1, np.uint64)
    np.add.at(rp, np.asarray(keep_r, np.int64) + 1, 1)
    rp = np.cumsum(rp).astype(np.uint64)
    return FeatureMatrix(n_samples, n_features, rp, np.asarray(keep_c, np.uint64), np.asarray(keep_v, np.float64))


def from_dense(a: np.ndarray) -> FeatureMatrix:
    a = np.asarray(a, np.float64)
    r, c = np.nonzero(a)
    rp = np.zeros(a.shape[0] + 1, np.uint64)
    np.add.at(rp, r + 1, 1)
    return FeatureMatrix(a.shape[0], a.shape[1], np.cumsum(rp).astype(np.uint64), c.astype(np.uint64),
                         a[r, c].copy())


def read_matrix_market(path: str) -> FeatureMatrix:
    """matrix_market.cpp:34-148 (coordinate / array; real / integer / pattern; general /
    symmetric), parsed by the library (rmg_read_matrix_market); RuntimeError on
    malformed input, like the reference."""
    lib = _lib.load()
    h, nnz = C.c_void_p(), C.c_uint64()
    _lib.check(lib.rmg_read_matrix_market(path.encode(), C.byref(h), C.byref(nnz)))
    n, f = C.c_uint64(), C.c_uint64()
    _lib.check(lib.rmg_host_csr_shape(h, C.byref(n), C.byref(f), None, None))
    return _host_csr_to_matrix(h, n.value, f.value, nnz.value, False)


def _host_handle(x: FeatureMatrix):
    lib = _lib.load()
    rp = np.ascontiguousarray(x.row_offsets, np.uint64)
    ci = np.ascontiguousarray(x.column_indices, np.uint64)
    v = None if x.values is None else np.ascontiguousarray(x.values, np.float64)
    h = C.c_void_p()
    _lib.check(lib.rmg_host_csr_create(x.n_samples, x.n_features, _ptr(rp), _ptr(ci), _ptr(v), C.byref(h)))
    return h


def csr_sha256(x: FeatureMatrix) -> str:
    """SHA-256 of (uint64 row offsets, uint64 column indices, fp64 values or 1.0)."""
    lib = _lib.load()
    h = _host_handle(x)
    out = C.create_string_buffer(65)
    try:
        _lib.check(lib.rmg_host_csr_sha256(h, out))
    finally:
        lib.rmg_host_csr_destroy(h)
    return out.value.decode()


def save_csr(x: FeatureMatrix, path: str) -> str:
    """The binary CSR cache (ingest.cpp); returns the SHA-256 stamped into it."""
    lib = _lib.load()
    h = _host_handle(x)
    out = C.create_string_buffer(65)
    try:
        _lib.check(lib.rmg_host_csr_save(h, path.encode()))
        _lib.check(lib.rmg_host_csr_sha256(h, out))
    finally:
        lib.rmg_host_csr_destroy(h)
    return out.value.decode()


def load_csr(path: str, verify: bool = True) -> tuple:
    """(FeatureMatrix, SHA-256) from a binary CSR cache; verify re-hashes the arrays."""
    lib = _lib.load()
    h, nnz = C.c_void_p(), C.c_uint64()
    sha = C.create_string_buffer(65)
    _lib.check(lib.rmg_host_csr_load(path.encode(), int(verify), C.byref(h), C.byref(nnz), sha))
    n, f, hv = C.c_uint64(), C.c_uint64(), C.c_int32()
    _lib.check(lib.rmg_host_csr_shape(h, C.byref(n), C.byref(f), None, C.byref(hv)))
    return _host_csr_to_matrix(h, n.value, f.value, nnz.value, not hv.value), sha.value.decode()


def _host_csr_to_matrix(h, n: int, f: int, nnz: int, pattern: bool) -> FeatureMatrix:
    lib = _lib.load()
    rp = np.zeros(n + 1, np.uint64)
    ci = np.zeros(nnz, np.uint64)
    v = None if pattern else np.zeros(nnz, np.float64)
    try:
        _lib.check(lib.rmg_host_csr_export(h, _ptr(rp), _ptr(ci), None if v is None else _ptr(v)))
    finally:
        lib.rmg_host_csr_destroy(h)
    return FeatureMatrix(n, f, rp, ci, v)


def synth_dense_clustered(n: int, f: int, groups: int = 50, noise: float = 0.1, seed: int = 0) -> FeatureMatrix:
    """BASELINE cfg 1 generator."""
    lib = _lib.load()
    h, nnz = C.c_void_p(), C.c_uint64()
    _lib.check(lib.rmg_synth_dense_clustered(n, f, groups, noise, seed, C.byref(h), C.byref(nnz)))
    return _host_csr_to_matrix(h, n, f, nnz.value, False)


def synth_sparse_zipf(n: int, f: int, mean_nnz: float, zipf_s: float, abs_normal_values: bool = False,
                      seed: int = 0, row_streams: bool = False) -> FeatureMatrix:
    """BASELINE cfg 2/3/5 generator.  row_streams=True: same
    distribution, one RNG stream per row, threaded (large measurement shards)."""
    lib = _lib.load()
    h, nnz = C.c_void_p(), C.c_uint64()
    fn = lib.rmg_synth_sparse_zipf_rows if row_streams else lib.rmg_synth_sparse_zipf
    _lib.check(fn(n, f, mean_nnz, zipf_s, int(abs_normal_values), seed, C.byref(h), C.byref(nnz)))
    return _host_csr_to_matrix(h, n, f, nnz.value, not abs_normal_values)


def synth_sparse_zipf_row_range(n: int, f: int, mean_nnz: float, zipf_s: float, abs_normal_values: bool, seed: int,
                                row0: int, row1: int) -> FeatureMatrix:
    """Rows [row0, row1) of synth_sparse_zipf(..., row_streams=True) (same bytes), as a
    (row1 - row0)-row matrix: per-rank generation of a row-sharded input."""
    lib = _lib.load()
    h, nnz = C.c_void_p(), C.c_uint64()
    _lib.check(lib.rmg_synth_sparse_zipf_row_range(n, f, mean_nnz, zipf_s, int(abs_normal_values), seed, row0, row1,
                                                   C.byref(h), C.byref(nnz)))
    return _host_csr_to_matrix(h, row1 - row0, f, nnz.value, not abs_normal_values)


def rng_normals(seed: int, n: int) -> np.ndarray:
    out = np.zeros(n)
    _lib.check(_lib.load().rmg_rng_normals(seed, n, _ptr(out)))
    return out


# ---------------------------------------------------------------- device objects
class Context:
    """One GPU and one stream (rmg_context)."""

    def __init__(self, device: int = 0):
        self.lib = _lib.load()
        self.h = C.c_void_p()
        _lib.check(self.lib.rmg_context_create(device, C.byref(self.h)))
        self.device = device

    def set_stream(self, cuda_stream: int) -> None:
        _lib.check(self.lib.rmg_context_set_stream(self.h, C.c_void_p(cuda_stream)))

    def synchronize(self) -> None:
        _lib.check(self.lib.rmg_context_synchronize(self.h))

    def close(self) -> None:
        if self.h:
            self.lib.rmg_context_destroy(self.h)
            self.h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


_default_ctx: Optional[Context] = None


def default_context() -> Context:
    global _default_ctx
    if _default_ctx is None:
        _default_ctx = Context(0)
    return _default_ctx


def shard_rows(row_offsets, nranks: int) -> np.ndarray:
    """nnz-balanced contiguous row blocks (host only): bounds[r]..bounds[r+1]."""
    rp = np.ascontiguousarray(row_offsets, np.uint64)
    out = np.zeros(nranks + 1, np.uint64)
    _lib.check(_lib.load().rmg_shard_rows(_ptr(rp), len(rp) - 1, nranks, _ptr(out)))
    return out


class Comm:
    """NCCL communicator (rmg_comm) for row-sharded operators.  `unique_id` is
    the 128-byte id from Comm.new_unique_id() on rank 0, broadcast by the caller."""

    @staticmethod
    def new_unique_id() -> bytes:
        buf = (C.c_uint8 * 128)()
        _lib.check(_lib.load().rmg_comm_unique_id(buf))
        return bytes(buf)

    def __init__(self, ctx: Context, nranks: int, rank: int, unique_id: bytes):
        self.lib = ctx.lib
        self.h = C.c_void_p()
        idb = (C.c_uint8 * 128).from_buffer_copy(unique_id)
        _lib.check(self.lib.rmg_comm_create(ctx.h, nranks, rank, idb, C.byref(self.h)))
        self.nranks, self.rank = nranks, rank

    @classmethod
    def host_staged(cls, ctx: Context, nranks: int, rank: int, allreduce) -> "Comm":
        """A host-staged communicator (rmg_comm_create_host): `allreduce(buf)` gets a
        float64 numpy view of the staged vector and must replace it in place by the
        sum over all ranks (e.g. a gloo all-reduce).  Several ranks may share one GPU."""
        self = cls.__new__(cls)
        self.lib = ctx.lib
        self.h = C.c_void_p()

        def fn(user, buf, count):
            try:
                allreduce(np.ctypeslib.as_array(C.cast(buf, C.POINTER(C.c_double)), shape=(count,)))
                return 0
            except Exception:  # reported to the library as a failed collective
                return 1

        self._cb = _HOST_ALLREDUCE(fn)  # kept alive with the communicator
        _lib.check(self.lib.rmg_comm_create_host(ctx.h, nranks, rank, C.cast(self._cb, C.c_void_p), None,
                                                 C.byref(self.h)))
        self.nranks, self.rank = nranks, rank
        return self

    def close(self):
        if self.h:
            self.lib.rmg_comm_destroy(self.h)
            self.h = C.c_void_p()


_HOST_ALLREDUCE = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_void_p, C.c_uint64)


class DeviceMatrix:
    """X and X^T resident in HBM (rmg_matrix).  Mirrors the FeatureMatrix-level
    free functions of the reference: spmv, spmv_transpose, RidgeOperator::apply,
    gram_diagonal, estimate_lambda_max(GramOperator).  With `comm`, only this
    rank's nnz-balanced row block lives on the device and X^T passes all-reduce."""

    def __init__(self, x: FeatureMatrix, ctx: Optional[Context] = None, detect_pattern: bool = True,
                 comm: Optional["Comm"] = None):
        self.ctx = ctx or default_context()
        self.lib = self.ctx.lib
        self.x = x
        self.comm = comm
        rp = np.ascontiguousarray(x.row_offsets, np.uint64)
        ci = np.ascontiguousarray(x.column_indices, np.uint64)
        v = None if x.values is None else np.ascontiguousarray(x.values, np.float64)
        self.h = C.c_void_p()
        if comm is None:
            _lib.check(self.lib.rmg_matrix_create_csr(self.ctx.h, x.n_samples, x.n_features, _ptr(rp), _ptr(ci),
                                                      _ptr(v), int(detect_pattern), C.byref(self.h)))
        else:
            _lib.check(self.lib.rmg_matrix_create_csr_sharded(self.ctx.h, comm.h, x.n_samples, x.n_features, _ptr(rp),
                                                              _ptr(ci), _ptr(v), int(detect_pattern),
                                                              C.byref(self.h)))
        self._query()

    @classmethod
    def from_rows(cls, x_local: FeatureMatrix, n_samples: int, row0: int, comm: "Comm",
                  ctx: Optional[Context] = None, detect_pattern: bool = True) -> "DeviceMatrix":
        """Per-rank input (rmg_matrix_create_csr_rows): this rank's rows [row0, row0 +
        x_local.n_samples) of an n_samples-row X; the hierarchy setup on it is sharded."""
        self = cls.__new__(cls)
        self.ctx = ctx or default_context()
        self.lib = self.ctx.lib
        self.x = x_local
        self.comm = comm
        rp = np.ascontiguousarray(x_local.row_offsets, np.uint64)
        ci = np.ascontiguousarray(x_local.column_indices, np.uint64)
        v = None if x_local.values is None else np.ascontiguousarray(x_local.values, np.float64)
        self.h = C.c_void_p()
        _lib.check(self.lib.rmg_matrix_create_csr_rows(self.ctx.h, comm.h, n_samples, row0, x_local.n_samples,
                                                       x_local.n_features, _ptr(rp), _ptr(ci), _ptr(v),
                                                       int(detect_pattern), C.byref(self.h)))
        self._query()
        return self

    @classmethod
    def from_dense_rows(cls, a_local, n_samples: int, row0: int, comm: "Comm",
                        ctx: Optional[Context] = None) -> "DeviceMatrix":
        """Per-rank dense input (rmg_matrix_create_dense_rows): this rank's rows [row0,
        row0 + len(a_local)) of a dense n_samples-row X; hierarchy setup sharded."""
        a = np.asarray(a_local)
        fp32 = a.dtype == np.float32
        a = np.ascontiguousarray(a, np.float32 if fp32 else np.float64)
        self = cls.__new__(cls)
        self.ctx = ctx or default_context()
        self.lib = self.ctx.lib
        self.x = None
        self.comm = comm
        self.h = C.c_void_p()
        nl, f = a.shape
        _lib.check(self.lib.rmg_matrix_create_dense_rows(self.ctx.h, comm.h, n_samples, row0, nl, f, _ptr(a), f,
                                                         int(fp32), C.byref(self.h)))
        self._query()
        return self

    @classmethod
    def from_dense(cls, a, ctx: Optional[Context] = None, comm: Optional["Comm"] = None) -> "DeviceMatrix":
        """Dense X (row-major, float64 or float32 storage; arithmetic stays fp64):
        the operator is one fused sweep over X.  n_features <= 1024."""
        a = np.asarray(a)
        if a.ndim != 2:
            raise ValueError("from_dense: a must be 2-D (samples x features)")
        fp32 = a.dtype == np.float32
        a = np.ascontiguousarray(a, np.float32 if fp32 else np.float64)
        self = cls.__new__(cls)
        self.ctx = ctx or default_context()
        self.lib = self.ctx.lib
        self.x = None
        self.comm = comm
        self.h = C.c_void_p()
        n, f = a.shape
        if comm is None:
            _lib.check(self.lib.rmg_matrix_create_dense(self.ctx.h, n, f, _ptr(a), f, int(fp32), C.byref(self.h)))
        else:
            _lib.check(self.lib.rmg_matrix_create_dense_sharded(self.ctx.h, comm.h, n, f, _ptr(a), f, int(fp32),
                                                                C.byref(self.h)))
        self._query()
        return self

    def is_dense(self) -> bool:
        d = C.c_int32()
        _lib.check(self.lib.rmg_matrix_is_dense(self.h, C.byref(d), None))
        return bool(d.value)

    def _query(self):
        r0, r1, nr, rk = C.c_uint64(), C.c_uint64(), C.c_int32(), C.c_int32()
        n, f, z, pat = C.c_uint64(), C.c_uint64(), C.c_uint64(), C.c_int32()
        _lib.check(self.lib.rmg_matrix_shape(self.h, C.byref(n), C.byref(f), C.byref(z), C.byref(pat)))
        _lib.check(self.lib.rmg_matrix_shard(self.h, C.byref(r0), C.byref(r1), C.byref(nr), C.byref(rk)))
        self.row_range = (r0.value, r1.value)
        self.n_samples, self.n_features, self.nnz, self.is_pattern = n.value, f.value, z.value, bool(pat.value)

    def close(self):
        if self.h:
            self.lib.rmg_matrix_destroy(self.h)
            self.h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _vec(self, a, n):
        a = np.ascontiguousarray(a, np.float64)
        if a.shape != (n,):
            raise ValueError(f"length {a.shape[0] if a.ndim else 0}, expected {n}")
        return a

    def ridge_apply_block(self, beta: float, v) -> np.ndarray:
        """X^T (X V) + beta V for V of shape (n_features, k), k <= 64 (cfg 3's block operator)."""
        v = np.ascontiguousarray(v, np.float64)
        if v.ndim != 2 or v.shape[0] != self.n_features:
            raise ValueError("ridge_apply_block: V must be (n_features, k)")
        out = np.zeros_like(v)
        _lib.check(self.lib.rmg_ridge_apply_block(self.h, beta, _ptr(v), _ptr(out), v.shape[1], 0))
        return out

    def hybrid_hot_features(self) -> int:
        """Hot features of the hybrid X^T pass (0: plain segmented pass)."""
        h = C.c_uint64()
        _lib.check(self.lib.rmg_matrix_hot_layout(self.h, C.byref(h), None, None))
        return int(h.value)

    def spmv(self, v) -> np.ndarray:
        v = self._vec(v, self.n_features)
        y = np.zeros(self.n_samples)
        _lib.check(self.lib.rmg_spmv(self.h, _ptr(v), _ptr(y), 0))
        return y

    def spmv_transpose(self, u) -> np.ndarray:
        u = self._vec(u, self.n_samples)
        y = np.zeros(self.n_features)
        _lib.check(self.lib.rmg_spmv_transpose(self.h, _ptr(u), _ptr(y), 0))
        return y

    def ridge_apply(self, beta: float, w) -> np.ndarray:
        w = self._vec(w, self.n_features)
        out = np.zeros(self.n_features)
        _lib.check(self.lib.rmg_ridge_apply(self.h, beta, _ptr(w), _ptr(out), 0))
        return out

    def gram_diagonal(self, beta: float) -> np.ndarray:
        out = np.zeros(self.n_features)
        _lib.check(self.lib.rmg_gram_diagonal(self.h, beta, _ptr(out), 0))
        return out

    def lambda_max(self, tol: float = 1e-4, max_iters: int = 200, seed: int = 0x5EED):
        v, it, cv = C.c_double(), C.c_uint64(), C.c_int32()
        _lib.check(self.lib.rmg_lambda_max(self.h, tol, max_iters, seed, C.byref(v), C.byref(it), C.byref(cv)))
        return v.value, it.value, bool(cv.value)


@dataclass
class RhsSample:
    b: np.ndarray
    rhs: np.ndarray


def generate_rhs(x: DeviceMatrix, seed: int) -> RhsSample:
    """analysis.cpp:225-232: b = CounterRng(seed) normals, rhs = X^T b."""
    b = np.zeros(x.n_samples)
    rhs = np.zeros(x.n_features)
    _lib.check(x.lib.rmg_generate_rhs(x.h, seed, _ptr(b), _ptr(rhs)))
    return RhsSample(b, rhs)


# ---------------------------------------------------------------- specs (krylov.hpp:16-23,135-218)
@dataclass
class SolverConfig:
    tol: float = 1e-6
    max_iters: int = 1000
    truncation: int = 20


@dataclass
class ClusteringChoice:
    kind: int = LEADER_TOLERANCE
    tolerance: float = 1.0
    target_size: int = 0
    seed: int = 0
    kmeans_max_iters: int = 100
    normalize_columns: bool = False  # BASELINE cfg 2 extension
    labels: Optional[np.ndarray] = None  # IMPORTED
    n_clusters: int = 0
    sketch_dim: int = 32  # KMEANS_SKETCH


@dataclass
class CoarseSolveChoice:
    kind: int = DIRECT_CHOLESKY
    tol: float = 1e-6
    max_iters: int = 500
    truncation: int = 20


@dataclass
class LevelSpec:
    clustering: ClusteringChoice = field(default_factory=ClusteringChoice)
    solver: CoarseSolveChoice = field(default_factory=CoarseSolveChoice)
    beta_override: Optional[float] = None
    omega_override: Optional[float] = None  # parity runs
    additive: bool = False  # pcg_vcycle_additive: this level enters additively too


@dataclass
class MethodSpec:
    kind: int = CG
    levels: Sequence[LevelSpec] = ()
    solver: SolverConfig = field(default_factory=SolverConfig)


@dataclass
class SolveReport:
    iterations: int = 0
    residual_history: np.ndarray = field(default_factory=lambda: np.zeros(0))
    converged: bool = False
    wall_time_s: float = 0.0
    inner_iterations: np.ndarray = field(default_factory=lambda: np.zeros(0, np.uint64))
    kernel_launches: int = 0


def _level_array(levels: Sequence[LevelSpec]):
    arr = (_lib.LevelSpecC * max(1, len(levels)))()
    keep = []
    for i, lv in enumerate(levels):
        s = arr[i]
        c = lv.clustering
        s.clustering_kind = c.kind
        s.tolerance = c.tolerance
        s.target_size = c.target_size
        s.seed = c.seed
        s.kmeans_max_iters = c.kmeans_max_iters
        s.normalize_columns = int(c.normalize_columns)
        s.sketch_dim = c.sketch_dim
        s.additive = int(lv.additive)
        if c.kind == IMPORTED:
            if c.labels is None:
                raise ValueError("imported clustering without labels")
            lab = np.ascontiguousarray(c.labels, np.int64)
            keep.append(lab)
            s.labels = lab.ctypes.data
            s.n_clusters = int(c.n_clusters if c.n_clusters else lab.max() + 1)
        s.coarse_kind = lv.solver.kind
        s.coarse_tol = lv.solver.tol
        s.coarse_max_iters = lv.solver.max_iters
        s.coarse_truncation = lv.solver.truncation
        if lv.beta_override is not None:
            s.has_beta_override, s.beta_override = 1, lv.beta_override
        if lv.omega_override is not None:
            s.has_omega_override, s.omega_override = 1, lv.omega_override
    return arr, keep


class PreparedMethod:
    """krylov.hpp:222-242: setup in the constructor, then solve(b) for any b."""

    def __init__(self, x: DeviceMatrix, beta: float, spec: MethodSpec):
        self.x, self.beta, self.spec = x, beta, spec
        self.lib = x.lib
        arr, self._keep = _level_array(spec.levels)
        cfg = _lib.SolverConfigC(spec.solver.tol, spec.solver.max_iters, spec.solver.truncation)
        self.h = C.c_void_p()
        _lib.check(self.lib.rmg_method_prepare(x.h, beta, spec.kind, arr, len(spec.levels), C.byref(cfg),
                                               C.byref(self.h)))
        nl, cs = C.c_uint64(), C.c_uint64()
        _lib.check(self.lib.rmg_method_info(self.h, C.byref(nl), C.byref(cs)))
        self.n_levels, self._coarse_size = nl.value, cs.value

    def close(self):
        if self.h:
            self.lib.rmg_method_destroy(self.h)
            self.h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def set_beta(self, beta: float) -> None:
        """A new regularization over the same hierarchy (cfg 3's beta sweep)."""
        _lib.check(self.lib.rmg_method_set_beta(self.h, beta))
        self.beta = beta

    def coarse_size(self) -> int:
        return self._coarse_size

    def _report(self):
        cap = self.spec.solver.max_iters + 1
        hist = np.zeros(cap)
        inner = np.zeros(cap, np.uint64)
        rep = _lib.SolveReportC()
        rep.residual_history, rep.residual_capacity = hist.ctypes.data, cap
        rep.inner_iterations, rep.inner_capacity = inner.ctypes.data, cap
        return rep, hist, inner

    def _finish(self, rep, hist, inner) -> SolveReport:
        it = rep.iterations
        nh = it if it else (1 if rep.converged else 0)
        flexible = self.spec.kind in (FCG_TWOLEVEL, FCG_MULTILEVEL, FGMRES_TWOLEVEL)
        return SolveReport(iterations=it, residual_history=hist[:nh].copy(), converged=bool(rep.converged),
                           wall_time_s=rep.wall_time_s,
                           inner_iterations=inner[:it].copy() if flexible else np.zeros(0, np.uint64),
                           kernel_launches=rep.kernel_launches)

    def solve(self, b) -> tuple[np.ndarray, SolveReport]:
        """PreparedMethod::solve (krylov.cpp:651-668): rhs = X^T b, then the Krylov solve."""
        b = np.ascontiguousarray(b, np.float64)
        if b.shape != (self.x.n_samples,):
            raise ValueError("PreparedMethod::solve: b length != n_samples")
        w = np.zeros(self.x.n_features)
        rep, hist, inner = self._report()
        _lib.check(self.lib.rmg_method_solve(self.h, _ptr(b), _ptr(w), C.byref(rep), 0))
        return w, self._finish(rep, hist, inner)

    def solve_batch(self, B) -> tuple[np.ndarray, list]:
        """k right-hand sides, B of shape (n_samples, k): W (n_features, k) and one
        SolveReport per column, each equal to solve(B[:, q])."""
        B = np.asarray(B, np.float64)
        if B.ndim != 2 or B.shape[0] != self.x.n_samples:
            raise ValueError("solve_batch: B must be (n_samples, k)")
        k = B.shape[1]
        bcol = np.ascontiguousarray(B.T)  # column-major block = row-major transpose
        wcol = np.zeros((k, self.x.n_features))
        parts = [self._report() for _ in range(k)]
        arr = (_lib.SolveReportC * max(1, k))()
        for q, (rep, _, _) in enumerate(parts):
            arr[q] = rep
        _lib.check(self.lib.rmg_method_solve_batch(self.h, _ptr(bcol), _ptr(wcol), k, arr, 0))
        reports = [self._finish(arr[q], parts[q][1], parts[q][2]) for q in range(k)]
        return np.ascontiguousarray(wcol.T), reports

    def solve_batch_device(self, b_ptr: int, w_ptr: int, k: int, on_device: bool = True) -> list:
        """rmg_method_solve_batch on raw pointers: column-major b (n_samples x k) and
        w (n_features x k) in device memory (on_device) or host memory."""
        parts = [self._report() for _ in range(k)]
        arr = (_lib.SolveReportC * max(1, k))()
        for q, (rep, _, _) in enumerate(parts):
            arr[q] = rep
        _lib.check(self.lib.rmg_method_solve_batch(self.h, C.c_void_p(b_ptr), C.c_void_p(w_ptr), k, arr,
                                                   int(on_device)))
        return [self._finish(arr[q], parts[q][1], parts[q][2]) for q in range(k)]

    def solve_rhs(self, rhs) -> tuple[np.ndarray, SolveReport]:
        rhs = np.ascontiguousarray(rhs, np.float64)
        if rhs.shape != (self.x.n_features,):
            raise ValueError("fcg: rhs length != operator dimension")
        w = np.zeros(self.x.n_features)
        rep, hist, inner = self._report()
        _lib.check(self.lib.rmg_method_solve_rhs(self.h, _ptr(rhs), _ptr(w), C.byref(rep), 0))
        return w, self._finish(rep, hist, inner)

    def solve_device(self, b_ptr: int, w_ptr: int, from_rhs: bool = False) -> SolveReport:
        """Device-pointer solve (inputs already resident in HBM)."""
        rep, hist, inner = self._report()
        fn = self.lib.rmg_method_solve_rhs if from_rhs else self.lib.rmg_method_solve
        _lib.check(fn(self.h, C.c_void_p(b_ptr), C.c_void_p(w_ptr), C.byref(rep), 1))
        return self._finish(rep, hist, inner)

    def precondition(self, r) -> np.ndarray:
        """two_level_apply (krylov.cpp:422-426) with the level-0 preconditioner."""
        r = np.ascontiguousarray(r, np.float64)
        z = np.zeros(self.x.n_features)
        _lib.check(self.lib.rmg_method_precondition(self.h, _ptr(r), _ptr(z), 0))
        return z

    def level(self, k: int) -> dict:
        nf, nnz, beta, omega = C.c_uint64(), C.c_uint64(), C.c_double(), C.c_double()
        _lib.check(self.lib.rmg_method_level(self.h, k, C.byref(nf), C.byref(nnz), C.byref(beta), C.byref(omega)))
        return {"n_features": nf.value, "nnz": nnz.value, "beta": beta.value, "omega": omega.value}

    def labels(self, k: int) -> np.ndarray:
        out = np.zeros(self.level(k)["n_features"], np.int64)
        _lib.check(self.lib.rmg_method_level_labels(self.h, k, _ptr(out)))
        return out

    def level_matrix(self, k: int) -> FeatureMatrix:
        info = self.level(k)
        n = self.x.n_samples
        rp = np.zeros(n + 1, np.uint64)
        ci = np.zeros(info["nnz"], np.uint64)
        v = np.zeros(info["nnz"])
        _lib.check(self.lib.rmg_method_level_matrix(self.h, k, _ptr(rp), _ptr(ci), _ptr(v)))
        return FeatureMatrix(n, info["n_features"], rp, ci, v)

    def set_profiling(self, on: bool = True) -> None:
        _lib.check(self.lib.rmg_method_set_profiling(self.h, int(on)))

    def profile(self, level: int):
        """(applications, ms in K1, ms in K2) accumulated by in-situ profiling."""
        n, k1, k2 = C.c_uint64(), C.c_double(), C.c_double()
        _lib.check(self.lib.rmg_method_profile(self.h, level, C.byref(n), C.byref(k1), C.byref(k2)))
        return n.value, k1.value, k2.value

    def time_operator(self, level: int = 0, reps: int = 20, flush_l2: bool = True):
        t, k1, k2 = C.c_double(), C.c_double(), C.c_double()
        _lib.check(self.lib.rmg_method_time_operator(self.h, level, reps, int(flush_l2), C.byref(t), C.byref(k1),
                                                     C.byref(k2)))
        return t.value, k1.value, k2.value


@dataclass
class SystemSolution:
    w: np.ndarray
    report: SolveReport
    coarse_size: int = 0


def solve_system(x: DeviceMatrix, beta: float, b, spec: MethodSpec) -> SystemSolution:
    """krylov.cpp:670-679: setup plus a single solve."""
    pm = PreparedMethod(x, beta, spec)
    try:
        w, rep = pm.solve(b)
        return SystemSolution(w, rep, pm.coarse_size())
    finally:
        pm.close()


# ---------------------------------------------------------------- bench harness (analysis.cpp:137-223)
METHOD_STRINGS = {v: k for k, v in METHOD_NAMES.items()}


def clustering_description(spec: "MethodSpec", coarse_size: int) -> str:
    """describe_clustering (krylov.cpp:596-612); C++ ostream default formatting."""
    if not spec.levels:
        return ""
    c = spec.levels[0].clustering
    if c.kind == LEADER_TOLERANCE:
        return f"lf(tol={c.tolerance:g},fc={coarse_size})"
    if c.kind == LEADER_TARGET:
        return f"lf(fc={coarse_size})"
    if c.kind == KMEANS:
        return f"km(k={coarse_size})"
    if c.kind == KMEANS_SKETCH:  # extension
        return f"kms(d={c.sketch_dim},k={coarse_size})"
    return f"imported(fc={coarse_size})"


@dataclass
class BenchRow:
    """analysis.hpp BenchRow: one (method, beta, tol) measurement."""
    dataset: str
    method: str
    clustering: str = ""
    f_c: int = 0
    beta: float = 0.0
    tol: float = 0.0
    iterations: int = 0
    wall_time_s: float = 0.0
    speedup: float = 0.0


def compare_methods(x: DeviceMatrix, dataset_name: str, beta_grid, tol_grid, methods, n_repeats: int = 1,
                    rhs_seed: int = 42) -> list:
    """compare_methods (analysis.cpp:137-198): for every (beta, tol), CG is always
    measured (max_iters = max(20000, 4 F)) as the speed-up denominator; each method
    is prepared once and solved n_repeats times for the rhs of generate_rhs(rhs_seed);
    times are the solver's own wall_time_s (setup excluded), averaged."""
    beta_grid, tol_grid, methods = list(beta_grid), list(tol_grid), list(methods)
    if not beta_grid or not tol_grid:
        raise ValueError("compare_methods: beta and tol grids must be non-empty")
    if not methods:
        raise ValueError("compare_methods: method list must be non-empty")
    if n_repeats < 1:
        raise ValueError("compare_methods: n_repeats must be >= 1")
    b = generate_rhs(x, rhs_seed).b
    rows = []
    for beta in beta_grid:
        for tol in tol_grid:
            base = MethodSpec(kind=CG, solver=SolverConfig(tol, max(20000, x.n_features * 4)))
            pcg = PreparedMethod(x, beta, base)
            cg_time, cg_rep = 0.0, None
            for _ in range(n_repeats):
                _, cg_rep = pcg.solve(b)
                cg_time += cg_rep.wall_time_s
            cg_time /= n_repeats
            pcg.close()
            for m in methods:
                spec = MethodSpec(kind=m.kind, levels=m.levels,
                                  solver=SolverConfig(tol, m.solver.max_iters, m.solver.truncation))
                row = BenchRow(dataset_name, METHOD_STRINGS[spec.kind], beta=beta, tol=tol)
                if spec.kind == CG:
                    row.iterations, row.wall_time_s, row.speedup = cg_rep.iterations, cg_time, 1.0
                    rows.append(row)
                    continue
                pm = PreparedMethod(x, beta, spec)
                t, rep = 0.0, None
                for _ in range(n_repeats):
                    _, rep = pm.solve(b)
                    t += rep.wall_time_s
                t /= n_repeats
                row.clustering = clustering_description(spec, pm.coarse_size())
                row.f_c = pm.coarse_size()
                row.iterations = rep.iterations
                row.wall_time_s = t
                row.speedup = cg_time / t if t > 0.0 else 0.0
                pm.close()
                rows.append(row)
    return rows


def to_csv(rows) -> str:
    """to_csv (analysis.cpp:200-212): the reference's header, ostream precision 12."""
    out = ["dataset,method,clustering,f_c,beta,tol,iterations,wall_time_s,speedup"]
    for r in rows:
        out.append(f"{r.dataset},{r.method},{r.clustering},{r.f_c},{r.beta:.12g},{r.tol:.12g},{r.iterations},"
                   f"{r.wall_time_s:.12g},{r.speedup:.12g}")
    return "\n".join(out) + "\n"
