"""ctypes binding of libridgemg_b200.so (include/ridgemg_b200.h).

The product path has no CPU fallback: if the shared library (built for
sm_100a) is missing or no CUDA device is present, calls fail loudly.
"""
from __future__ import annotations

import ctypes as C
import os

PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(PKG, "libridgemg_b200.so")

RMG_OK, RMG_ERR_INVALID_ARGUMENT, RMG_ERR_RUNTIME, RMG_ERR_CUDA, RMG_ERR_INTERNAL = 0, 1, 2, 3, 4


class RmgCudaError(RuntimeError):
    """A CUDA / device failure inside libridgemg_b200 (no CPU fallback exists)."""


class LevelSpecC(C.Structure):
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
        ("has_omega_override", C.c_int32),
        ("omega_override", C.c_double),
        ("sketch_dim", C.c_uint64),
        ("additive", C.c_int32),
    ]


class SolverConfigC(C.Structure):
    _fields_ = [("tol", C.c_double), ("max_iters", C.c_uint64), ("truncation", C.c_uint64)]


class SolveReportC(C.Structure):
    _fields_ = [
        ("iterations", C.c_uint64),
        ("converged", C.c_int32),
        ("wall_time_s", C.c_double),
        ("final_relative_residual", C.c_double),
        ("residual_history", C.c_void_p),
        ("residual_capacity", C.c_uint64),
        ("inner_iterations", C.c_void_p),
        ("inner_capacity", C.c_uint64),
        ("kernel_launches", C.c_uint64),
    ]


_P = C.c_void_p
_U64 = C.c_uint64
_I32 = C.c_int32
_D = C.c_double
_PP = C.POINTER(C.c_void_p)

# name -> argtypes (all return int status unless noted)
SIGNATURES = {
    "rmg_version": [_P, _P],
    "rmg_context_create": [_I32, _PP],
    "rmg_context_destroy": [_P],
    "rmg_context_set_stream": [_P, _P],
    "rmg_context_synchronize": [_P],
    "rmg_matrix_create_csr": [_P, _U64, _U64, _P, _P, _P, _I32, _PP],
    "rmg_matrix_destroy": [_P],
    "rmg_matrix_shape": [_P, _P, _P, _P, _P],
    "rmg_matrix_hot_layout": [_P, _P, _P, _P],
    "rmg_matrix_create_dense": [_P, _U64, _U64, _P, _U64, _I32, _PP],
    "rmg_matrix_create_dense_sharded": [_P, _P, _U64, _U64, _P, _U64, _I32, _PP],
    "rmg_matrix_is_dense": [_P, _P, _P],
    "rmg_spmv": [_P, _P, _P, _I32],
    "rmg_spmv_transpose": [_P, _P, _P, _I32],
    "rmg_ridge_apply": [_P, _D, _P, _P, _I32],
    "rmg_ridge_apply_block": [_P, _D, _P, _P, _U64, _I32],
    "rmg_gram_diagonal": [_P, _D, _P, _I32],
    "rmg_lambda_max": [_P, _D, _U64, _U64, _P, _P, _P],
    "rmg_generate_rhs": [_P, _U64, _P, _P],
    "rmg_rng_normals": [_U64, _U64, _P],
    "rmg_synth_dense_clustered": [_U64, _U64, _U64, _D, _U64, _PP, _P],
    "rmg_synth_sparse_zipf": [_U64, _U64, _D, _D, _I32, _U64, _PP, _P],
    "rmg_synth_sparse_zipf_rows": [_U64, _U64, _D, _D, _I32, _U64, _PP, _P],
    "rmg_host_csr_export": [_P, _P, _P, _P],
    "rmg_host_csr_destroy": [_P],
    "rmg_method_prepare": [_P, _D, _I32, _P, _U64, _P, _PP],
    "rmg_method_destroy": [_P],
    "rmg_method_set_beta": [_P, _D],
    "rmg_method_solve": [_P, _P, _P, _P, _I32],
    "rmg_method_solve_rhs": [_P, _P, _P, _P, _I32],
    "rmg_method_precondition": [_P, _P, _P, _I32],
    "rmg_method_solve_batch": [_P, _P, _P, _U64, _P, _I32],
    "rmg_method_info": [_P, _P, _P],
    "rmg_method_level": [_P, _U64, _P, _P, _P, _P],
    "rmg_method_level_labels": [_P, _U64, _P],
    "rmg_method_level_matrix": [_P, _U64, _P, _P, _P],
    "rmg_solve_system": [_P, _D, _I32, _P, _U64, _P, _P, _P, _P, _P],
    "rmg_method_time_operator": [_P, _U64, _U64, _I32, _P, _P, _P],
    "rmg_comm_unique_id": [_P],
    "rmg_comm_create": [_P, _I32, _I32, _P, _PP],
    "rmg_comm_destroy": [_P],
    "rmg_comm_create_host": [_P, _I32, _I32, _P, _P, _PP],
    "rmg_read_matrix_market": [C.c_char_p, _PP, _P],
    "rmg_host_csr_create": [_U64, _U64, _P, _P, _P, _PP],
    "rmg_host_csr_shape": [_P, _P, _P, _P, _P],
    "rmg_host_csr_sha256": [_P, C.c_char_p],
    "rmg_host_csr_save": [_P, C.c_char_p],
    "rmg_host_csr_load": [C.c_char_p, _I32, _PP, _P, C.c_char_p],
    "rmg_matrix_create_from_host": [_P, _P, _I32, _PP],
    "rmg_matrix_create_csr_rows": [_P, _P, _U64, _U64, _U64, _U64, _P, _P, _P, _I32, _PP],
    "rmg_matrix_create_dense_rows": [_P, _P, _U64, _U64, _U64, _U64, _P, _U64, _I32, _PP],
    "rmg_synth_sparse_zipf_row_range": [_U64, _U64, _D, _D, _I32, _U64, _U64, _U64, _PP, _P],
    "rmg_matrix_create_csr_sharded": [_P, _P, _U64, _U64, _P, _P, _P, _I32, _PP],
    "rmg_matrix_shard": [_P, _P, _P, _P, _P],
    "rmg_shard_rows": [_P, _U64, _I32, _P],
    "rmg_method_set_profiling": [_P, _I32],
    "rmg_method_profile": [_P, _U64, _P, _P, _P],
}

_lib = None


def load() -> C.CDLL:
    """Load the in-tree shared library (never a fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} is missing: run `python -m paper_1806_05826_b200.build` "
                          "(the solve path has no CPU fallback)")
    override = os.environ.get("RMG_LIB_PATH")  # diagnostics: A/B another build of the library
    lib = C.CDLL(override or LIB_PATH)
    lib.rmg_last_error.restype = C.c_char_p
    lib.rmg_last_error.argtypes = []
    for name, args in SIGNATURES.items():
        if override and not hasattr(lib, name):
            continue
        fn = getattr(lib, name)
        fn.argtypes = args
        fn.restype = C.c_int
    _lib = lib
    return lib


def check(rc: int) -> None:
    if rc == RMG_OK:
        return
    msg = load().rmg_last_error().decode(errors="replace")
    if rc == RMG_ERR_INVALID_ARGUMENT:
        raise ValueError(msg)
    if rc == RMG_ERR_CUDA:
        raise RmgCudaError(msg)
    raise RuntimeError(msg)


def exported_symbols() -> list[str]:
    return ["rmg_last_error", *SIGNATURES.keys()]
