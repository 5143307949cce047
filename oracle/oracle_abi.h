/* TEST INFRASTRUCTURE ONLY — never linked into the product library.
 *
 * Shared plain-C structs for the two CPU checkers under oracle/:
 *   - oracle/_ref/libridgemg_ref.so : the reference's own sources
 *     (/root/reference/proj/src/*.cpp) compiled verbatim + ref_capi.cpp glue;
 *   - oracle/_build/libridgemg_oracle.so : this repo's CPU restatement
 *     (oracle/restatement.cpp).
 * Both export the same entry points with prefixes `ref_` and `orc_` so the
 * pytest suite can run one check against either.
 */
#ifndef RIDGEMG_ORACLE_ABI_H
#define RIDGEMG_ORACLE_ABI_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* krylov.hpp:135-146 ClusteringChoice::Kind */
enum { OR_CLUSTER_LEADER_TOLERANCE = 0, OR_CLUSTER_LEADER_TARGET = 1, OR_CLUSTER_KMEANS = 2 };
/* krylov.hpp:154-160 CoarseSolveChoice::Kind */
enum { OR_COARSE_DIRECT = 0, OR_COARSE_INNER_CG = 1, OR_COARSE_INNER_FCG = 2 };
/* krylov.hpp:207 MethodKind */
enum { OR_METHOD_CG = 0, OR_METHOD_JACOBI_CG = 1, OR_METHOD_FCG_TWOLEVEL = 2,
       OR_METHOD_FCG_MULTILEVEL = 3, OR_METHOD_FGMRES_TWOLEVEL = 4 };

typedef struct {
  /* clustering (used when labels == NULL) */
  int32_t clustering_kind;
  double tolerance;
  uint64_t target_size;
  uint64_t seed;
  uint64_t kmeans_max_iters;
  int32_t normalize_columns; /* BASELINE cfg 2 extension: cluster x_j/||x_j|| */
  /* imported labels (parity runs): membership per fine feature, or NULL */
  const int64_t* labels;
  uint64_t n_clusters;
  /* coarse solve */
  int32_t coarse_kind;
  double coarse_tol;
  uint64_t coarse_max_iters;
  uint64_t coarse_truncation;
  int32_t has_beta_override;
  double beta_override;
} or_level_spec;

typedef struct {
  double tol;
  uint64_t max_iters;
  uint64_t truncation;
} or_solver_config;

typedef struct {
  uint64_t iterations;
  int32_t converged;
  double wall_time_s;
  double* residual_history;       /* caller buffer or NULL */
  uint64_t residual_capacity;
  uint64_t* inner_iterations;     /* caller buffer or NULL */
  uint64_t inner_capacity;
  double omega[8];                /* per-level omega actually used */
  uint64_t level_sizes[8];        /* F_k per level (level 0 = fine) */
  uint64_t n_levels;
} or_solve_report;

#ifdef __cplusplus
}
#endif
#endif
