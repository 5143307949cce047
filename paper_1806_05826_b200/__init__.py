"""ridgemg_b200: B200-native (sm_100a) solve path for the clustering-based
multilevel preconditioner of (X^T X + beta I) w = X^T b (arXiv:1806.05826).

The product is the C-ABI library ``libridgemg_b200.so`` (include/ridgemg_b200.h);
this package is its ctypes binding plus a Python mirror of the reference's
``ridgemg::`` interface (``ridgemg.py``).
"""
from ._lib import LIB_PATH, RmgCudaError, load  # noqa: F401
from .ridgemg import (  # noqa: F401
    CG, DIRECT_CHOLESKY, FCG_MULTILEVEL, FCG_TWOLEVEL, FGMRES_TWOLEVEL, IMPORTED, INNER_CG, INNER_FCG, JACOBI_CG, KMEANS,
    KMEANS_SKETCH, PCG_VCYCLE, PCG_VCYCLE_ADDITIVE,
    LEADER_TARGET, LEADER_TOLERANCE, ClusteringChoice, CoarseSolveChoice, Comm, Context, DeviceMatrix, FeatureMatrix,
    LevelSpec, MethodSpec, PreparedMethod, RhsSample, SolveReport, SolverConfig, SystemSolution, csr_from_triplets,
    default_context, from_dense, generate_rhs, method_from_string, read_matrix_market, rng_normals, shard_rows,
    solve_system, synth_dense_clustered, synth_sparse_zipf, synth_sparse_zipf_row_range, BenchRow, compare_methods,
    to_csv, clustering_description, csr_sha256, save_csr, load_csr)

__all__ = [n for n in dir() if not n.startswith("_")]
