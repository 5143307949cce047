/* ridgemg_b200 — B200-native (sm_100a) solve path for the clustering-based
 * multilevel preconditioner of (X^T X + beta I) w = X^T b  (arXiv:1806.05826).
 *
 * Plain C ABI: opaque handles, plain pointers and sizes, int status codes.
 * Every entry point replaces one piece of the reference's C++ interface in
 * /root/reference/proj/include/ridgemg (cited per function).  The C++ mirror
 * of that interface over this ABI is include/ridgemg_b200.hpp; the ctypes
 * binding is paper_1806_05826_b200/_lib.py.
 *
 * Error model (mirrors the reference's exception types):
 *   RMG_OK                     success
 *   RMG_ERR_INVALID_ARGUMENT   where the reference throws std::invalid_argument
 *   RMG_ERR_RUNTIME            where it throws std::runtime_error (breakdown,
 *                              indefinite coarse factorization)
 *   RMG_ERR_CUDA               CUDA / device failure (no CPU fallback exists)
 *   RMG_ERR_INTERNAL           anything else
 * rmg_last_error() returns the thread-local message of the last failure.
 * Non-convergence is not an error: report->converged == 0.
 *
 * Pointers flagged `on_device` are CUDA device pointers on the context's
 * device; otherwise host pointers (pinned or pageable), copied inside the call.
 */
#ifndef RIDGEMG_B200_H
#define RIDGEMG_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define RMG_OK 0
#define RMG_ERR_INVALID_ARGUMENT 1
#define RMG_ERR_RUNTIME 2
#define RMG_ERR_CUDA 3
#define RMG_ERR_INTERNAL 4

#define RMG_MAX_LEVELS 8

typedef struct rmg_context rmg_context;
typedef struct rmg_matrix rmg_matrix;
typedef struct rmg_method rmg_method;

/* krylov.hpp:207 MethodKind */
typedef enum {
  RMG_METHOD_CG = 0,
  RMG_METHOD_JACOBI_CG = 1,
  RMG_METHOD_FCG_TWOLEVEL = 2,
  RMG_METHOD_FCG_MULTILEVEL = 3,
  RMG_METHOD_FGMRES_TWOLEVEL = 4, /* krylov.cpp:229-328 + :628-635, full (unrestarted) */
  /* extension (BASELINE cfg 1's "Jacobi smoothing, 1 pre- and 1 post-sweep"; north-star (2);
   * no reference counterpart): plain PCG with a symmetric V-cycle over the
   * same hierarchy, damped-Jacobi pre- and post-smoothing at every level above the coarsest,
   * the coarsest level solved directly */
  RMG_METHOD_PCG_VCYCLE = 5,
  /* extension: PCG with the same hierarchy entered additively at the finest
   * level -- z = D_0^-1 r + P_0 V_1(P_0^T r), V_1 the symmetric V-cycle of levels >= 1 (dense
   * coarse Grams where they are smaller than the level's sweep), so an iteration costs one
   * fine-level operator application instead of three.  SPD, so plain PCG applies. */
  RMG_METHOD_PCG_VCYCLE_ADDITIVE = 6
} rmg_method_kind;

/* krylov.hpp:135-146 ClusteringChoice::Kind (+ imported labels for parity runs) */
typedef enum {
  RMG_CLUSTER_LEADER_TOLERANCE = 0,
  RMG_CLUSTER_LEADER_TARGET = 1,
  RMG_CLUSTER_KMEANS = 2,
  /* extension for levels too large for the reference's k-means (BASELINE cfg 3 / 5,
   * SURVEY App. A.8): the reference k-means on a sign sketch of the columns
   * (d = sketch_dim <= 32 rows).  Not the reference's clustering. */
  RMG_CLUSTER_KMEANS_SKETCH = 3,
  RMG_CLUSTER_IMPORTED = 100
} rmg_clustering_kind;

/* krylov.hpp:154-160 CoarseSolveChoice::Kind */
typedef enum {
  RMG_COARSE_DIRECT_CHOLESKY = 0,
  RMG_COARSE_INNER_CG = 1,
  RMG_COARSE_INNER_FCG = 2
} rmg_coarse_kind;

/* krylov.hpp:16-23 SolverConfig (omega_* of the reference is a dead knob,
 * SURVEY.md App. A.9; per-level omega overrides live in rmg_level_spec). */
typedef struct {
  double tol;          /* relative residual ||r|| / ||rhs||, default 1e-6 */
  uint64_t max_iters;  /* default 1000 */
  uint64_t truncation; /* FCG history bound m, default 20 */
} rmg_solver_config;

/* krylov.hpp:162-167 LevelSpec (+ ClusteringChoice :135-146, CoarseSolveChoice :154-160) */
typedef struct {
  int32_t clustering_kind;    /* rmg_clustering_kind */
  double tolerance;           /* leader_tolerance */
  uint64_t target_size;       /* leader_target / kmeans */
  uint64_t seed;              /* kmeans++ seed */
  uint64_t kmeans_max_iters;  /* default 100 */
  int32_t normalize_columns;  /* BASELINE cfg 2: cluster x_j/||x_j|| (extension) */
  const int64_t* labels;      /* RMG_CLUSTER_IMPORTED: membership per feature (host) */
  uint64_t n_clusters;        /* RMG_CLUSTER_IMPORTED: number of clusters */
  int32_t coarse_kind;        /* rmg_coarse_kind */
  double coarse_tol;          /* default 1e-6 */
  uint64_t coarse_max_iters;  /* default 500 */
  uint64_t coarse_truncation; /* default 20 */
  int32_t has_beta_override;
  double beta_override;
  int32_t has_omega_override; /* parity runs: import the oracle's omega_k */
  double omega_override;
  uint64_t sketch_dim;        /* RMG_CLUSTER_KMEANS_SKETCH: rows of the sketch (0: 32) */
  int32_t additive;           /* RMG_METHOD_PCG_VCYCLE_ADDITIVE only: the level this spec coarsens
                               * (level i for levels[i]) enters additively, z = D^-1 r + P V(P^T r),
                               * with no operator application of its own; level 0 always does
                               * (DESIGN.md section 4.15).  0 elsewhere. */
} rmg_level_spec;

/* krylov.hpp:25-31 SolveReport; history arrays are caller buffers (may be NULL). */
typedef struct {
  uint64_t iterations;
  int32_t converged;
  double wall_time_s;            /* Krylov loop only, like krylov.cpp:163,225 */
  double final_relative_residual;
  double* residual_history;      /* out: relative residual after each iteration */
  uint64_t residual_capacity;
  uint64_t* inner_iterations;    /* out: inner iterations per outer step */
  uint64_t inner_capacity;
  uint64_t kernel_launches;      /* kernels this solve launched (diagnostics) */
} rmg_solve_report;

/* ---------------------------------------------------------------- context */
const char* rmg_last_error(void);
int rmg_version(int32_t* major, int32_t* minor);
/* device ordinal on this process; creates a private stream */
int rmg_context_create(int32_t device, rmg_context** out);
int rmg_context_destroy(rmg_context* ctx);
/* run subsequent work on an external cudaStream_t (e.g. torch's current stream) */
int rmg_context_set_stream(rmg_context* ctx, void* cuda_stream);
int rmg_context_synchronize(rmg_context* ctx);

/* ---------------------------------------------------------------- matrix
 * FeatureMatrix (sparse.hpp:24-32): canonical CSR, size_t offsets/indices,
 * strictly increasing columns per row.  values == NULL (or all-ones with
 * detect_pattern != 0) selects the binary-pattern storage (4 B/nnz).
 * Uploads X and its transpose (X^T as CSR) to HBM with int32 indices.     */
int rmg_matrix_create_csr(rmg_context* ctx, uint64_t n_samples, uint64_t n_features,
                          const uint64_t* row_offsets, const uint64_t* column_indices,
                          const double* values, int32_t detect_pattern, rmg_matrix** out);
int rmg_matrix_destroy(rmg_matrix* m);
/* Dense X (north-star (1): row-major dense for dense inputs; no reference
 * counterpart -- the reference stores every input as FeatureMatrix CSR, which a
 * dense array becomes via csr_from_triplets, sparse.hpp:55-56).  data: host,
 * row-major n x f with leading dimension ld elements, fp64 (fp32 = 0) or fp32
 * storage (fp32 = 1; arithmetic stays fp64).  f <= 1024.  The operator is one
 * fused sweep over X.  No host CSR is kept: the hierarchy setup
 * (k-means, X_c = X P, coarse Gram) runs on the device with the same arithmetic as
 * the CSR path; the sharded variant keeps the host CSR setup. */
int rmg_matrix_create_dense(rmg_context* ctx, uint64_t n_samples, uint64_t n_features, const void* data,
                            uint64_t ld, int32_t fp32, rmg_matrix** out);
int rmg_matrix_is_dense(const rmg_matrix* m, int32_t* dense, int32_t* fp32);
int rmg_matrix_shape(const rmg_matrix* m, uint64_t* n_samples, uint64_t* n_features,
                     uint64_t* nnz, int32_t* is_pattern);
/* Diagnostics (no reference counterpart): layout of the hybrid X^T pass --
 * hot features summed per sample block from SMEM; zeros when
 * the matrix uses the plain segmented pass. */
int rmg_matrix_hot_layout(const rmg_matrix* m, uint64_t* hot_features, uint64_t* sample_blocks,
                          uint64_t* block_samples);

/* y = X v            (sparse.hpp:61, sparse.cpp:127-144)   */
int rmg_spmv(rmg_matrix* m, const double* v, double* y, int32_t on_device);
/* y = X^T u          (sparse.hpp:66, sparse.cpp:152-176)   */
int rmg_spmv_transpose(rmg_matrix* m, const double* u, double* y, int32_t on_device);
/* out = X^T X w + beta w   (RidgeOperator::apply, ridge.cpp:16-24) */
int rmg_ridge_apply(rmg_matrix* m, double beta, const double* w, double* out, int32_t on_device);
/* k right-hand sides at once (BASELINE cfg 3's block operator, no reference
 * counterpart: the reference applies RidgeOperator once per vector):
 * out = X^T (X V) + beta V with V, out row-major n_features x k, 1 <= k <= 64;
 * column q equals rmg_ridge_apply of column q up to summation order.  Single-GPU
 * matrices: CSR (record-streaming gather passes) or dense, where the
 * operator is the dense contraction (X^T X) V + beta V on the FP64 tensor cores --
 * G = X^T X is formed once by a DMMA SYRK on the first call and kept. */
int rmg_ridge_apply_block(rmg_matrix* m, double beta, const double* v, double* out, uint64_t k, int32_t on_device);
/* d_j = beta + ||X(:,j)||^2 (gram_diagonal, ridge.cpp:30-37) */
int rmg_gram_diagonal(rmg_matrix* m, double beta, double* out, int32_t on_device);
/* largest eigenvalue of X^T X by power iteration (estimate_lambda_max, krylov.cpp:62-92) */
int rmg_lambda_max(rmg_matrix* m, double tol, uint64_t max_iters, uint64_t seed, double* value,
                   uint64_t* iterations, int32_t* converged);

/* ---------------------------------------------------------------- multi-GPU
 * Row sharding of X across the GPUs of one node (one process per GPU,
 * SURVEY.md §8(e)): each rank keeps an nnz-balanced contiguous block of rows
 * of X (and its transpose) on its device; every X^T pass all-reduces the
 * F-vector with NCCL over NVLink before the epilogue.  Krylov vectors and the
 * coarse levels are replicated.  Rank 0 creates the unique id, the caller
 * broadcasts it (e.g. torch.distributed), every rank creates its communicator. */
typedef struct rmg_comm rmg_comm;
#define RMG_UNIQUE_ID_BYTES 128
int rmg_comm_unique_id(uint8_t* id_out);
int rmg_comm_create(rmg_context* ctx, int32_t nranks, int32_t rank, const uint8_t* id, rmg_comm** out);
/* Dense X row-sharded over the communicator (north-star (e), cfg 4): each rank
 * keeps its nnz-balanced (= row-balanced) block; see rmg_matrix_create_dense. */
int rmg_matrix_create_dense_sharded(rmg_context* ctx, rmg_comm* comm, uint64_t n_samples, uint64_t n_features,
                                    const void* data, uint64_t ld, int32_t fp32, rmg_matrix** out);
int rmg_comm_destroy(rmg_comm* comm);
/* A host-staged communicator: every all-reduce copies the vector to pinned host
 * memory, calls fn(user, buf, count) -- which must replace buf by the sum over
 * all ranks, in rank order, and return 0 -- and copies it back.  For several
 * ranks on ONE device (NCCL refuses duplicate devices): tests and single-GPU
 * rehearsals of the sharded path (e.g. fn = a gloo all-reduce). */
typedef int (*rmg_host_allreduce_fn)(void* user, double* buf, uint64_t count);
int rmg_comm_create_host(rmg_context* ctx, int32_t nranks, int32_t rank, rmg_host_allreduce_fn fn, void* user,
                         rmg_comm** out);
/* Per-rank input (no rank needs the whole matrix): this rank's contiguous block of
 * rows [row0, row0 + n_local) of an n_samples x n_features X, row offsets rebased
 * to 0 (n_local + 1 entries).  Blocks must tile [0, n_samples) in rank order.
 * Hierarchy setup on such a matrix is sharded too: coarse levels X_k = X P are
 * coarsened row-locally (X_k keeps the same row blocks), their Gram matrices and
 * Jacobi diagonals are all-reduced, and clustering must be kmeans_sketch (the
 * sketch S = G^T X is all-reduced) or imported labels. */
int rmg_matrix_create_csr_rows(rmg_context* ctx, rmg_comm* comm, uint64_t n_samples, uint64_t row0,
                               uint64_t n_local, uint64_t n_features, const uint64_t* row_offsets,
                               const uint64_t* column_indices, const double* values, int32_t detect_pattern,
                               rmg_matrix** out);
/* Per-rank dense input (cfg 4 sharded): this rank's rows [row0, row0 + n_local) of a
 * dense n_samples x n_features X (row-major, leading dimension ld, fp32 or fp64
 * storage); no CSR is ever built.  The hierarchy is set up sharded on the device:
 * kmeans_sketch (S all-reduced, columns normalised by the all-reduced norms) or
 * imported labels, X_k = X P on every rank's rows, all-reduced coarse Grams. */
int rmg_matrix_create_dense_rows(rmg_context* ctx, rmg_comm* comm, uint64_t n_samples, uint64_t row0,
                                 uint64_t n_local, uint64_t n_features, const void* data, uint64_t ld, int32_t fp32,
                                 rmg_matrix** out);
/* Replicated-setup variant: every rank passes the FULL matrix (the hierarchy is then
 * built unsharded on every rank); only this rank's nnz-balanced row block is
 * uploaded. */
int rmg_matrix_create_csr_sharded(rmg_context* ctx, rmg_comm* comm, uint64_t n_samples, uint64_t n_features,
                                  const uint64_t* row_offsets, const uint64_t* column_indices,
                                  const double* values, int32_t detect_pattern, rmg_matrix** out);
int rmg_matrix_shard(const rmg_matrix* m, uint64_t* row0, uint64_t* row1, int32_t* nranks, int32_t* rank);
/* The partition itself (host only): bounds_out[r]..bounds_out[r+1] for rank r. */
int rmg_shard_rows(const uint64_t* row_offsets, uint64_t n_samples, int32_t nranks, uint64_t* bounds_out);

/* ---------------------------------------------------------------- host helpers
 * generate_rhs (analysis.cpp:225-232): b_i = CounterRng(seed) normals
 * (rng.hpp:25-72, glibc libm), rhs = X^T b on the device.  rhs may be NULL. */
int rmg_generate_rhs(rmg_matrix* m, uint64_t seed, double* b_out, double* rhs_out);
/* n standard normals of CounterRng(seed) (rng.hpp:50-61) */
int rmg_rng_normals(uint64_t seed, uint64_t n, double* out);

/* BASELINE.json synthetic inputs, generated on the host with
 * CounterRng + glibc libm so every arm sees identical bytes.  Two-step:
 * rmg_synth_* returns an opaque host CSR and its sizes; rmg_host_csr_export
 * copies it into caller arrays (values may be NULL for binary patterns). */
typedef struct rmg_host_csr rmg_host_csr;
/* cfg 1: X[:,j] = Z[:, j mod groups] + noise * N(0,1), Z ~ N(0,1) (N x groups) */
int rmg_synth_dense_clustered(uint64_t n, uint64_t f, uint64_t groups, double noise, uint64_t seed,
                              rmg_host_csr** out, uint64_t* nnz);
/* cfg 2/3/5: nnz per row max(1, Poisson(mean)), Zipf(s) column popularity over a
 * seeded permutation, without replacement per row; values 1.0 or |N(0,1)| */
int rmg_synth_sparse_zipf(uint64_t n, uint64_t f, double mean_nnz, double zipf_s, int32_t abs_normal_values,
                          uint64_t seed, rmg_host_csr** out, uint64_t* nnz);
/* Same distribution with one RNG stream per row, generated by all host threads
 * (large measurement shards, e.g. cfg5 per-GPU); not the reference's stream */
int rmg_synth_sparse_zipf_rows(uint64_t n, uint64_t f, double mean_nnz, double zipf_s, int32_t abs_normal_values,
                               uint64_t seed, rmg_host_csr** out, uint64_t* nnz);
/* Rows [row0, row1) of the matrix rmg_synth_sparse_zipf_rows generates (the same
 * bytes): per-rank generation of a row-sharded input. */
int rmg_synth_sparse_zipf_row_range(uint64_t n, uint64_t f, double mean_nnz, double zipf_s,
                                    int32_t abs_normal_values, uint64_t seed, uint64_t row0, uint64_t row1,
                                    rmg_host_csr** out, uint64_t* nnz);
int rmg_host_csr_export(const rmg_host_csr* h, uint64_t* row_offsets, uint64_t* column_indices, double* values);
int rmg_host_csr_destroy(rmg_host_csr* h);

/* ---------------------------------------------------------------- ingest
 * read_matrix_market (matrix_market.cpp:34-148; same variants and errors) into a host
 * CSR, csr_from_triplets semantics (sparse.cpp:27-73); a binary CSR cache stamped
 * with the SHA-256 of its arrays (uint64 offsets, uint64 indices, fp64 values with 1.0
 * for a binary pattern: the bytes bench.py and the fixtures hash); upload straight
 * from a host CSR.  sha_hex: 65 bytes (64 hex digits + NUL). */
int rmg_read_matrix_market(const char* path, rmg_host_csr** out, uint64_t* nnz);
int rmg_host_csr_create(uint64_t n, uint64_t f, const uint64_t* row_offsets, const uint64_t* column_indices,
                        const double* values, rmg_host_csr** out);
int rmg_host_csr_shape(const rmg_host_csr* h, uint64_t* n, uint64_t* f, uint64_t* nnz, int32_t* has_values);
int rmg_host_csr_sha256(const rmg_host_csr* h, char* sha_hex);
int rmg_host_csr_save(const rmg_host_csr* h, const char* path);
int rmg_host_csr_load(const char* path, int32_t verify, rmg_host_csr** out, uint64_t* nnz, char* sha_hex);
int rmg_matrix_create_from_host(rmg_context* ctx, const rmg_host_csr* h, int32_t detect_pattern, rmg_matrix** out);

/* ---------------------------------------------------------------- methods
 * PreparedMethod(x, beta, spec) (krylov.hpp:222-242, krylov.cpp:617-649):
 * clustering, aggregation, coarse matrices, omegas and coarse factorization
 * all done here.  `levels` is ignored by cg / jacobi_cg.  The matrix must
 * outlive the method (ridge.hpp:37 lifetime contract).                  */
int rmg_method_prepare(rmg_matrix* m, double beta, int32_t method_kind,
                       const rmg_level_spec* levels, uint64_t n_levels,
                       const rmg_solver_config* solver, rmg_method** out);
/* Regularization sweep over a fixed hierarchy (BASELINE cfg 3; the reference
 * re-prepares per beta, analysis.cpp:157-196): keeps the clustering, P, the
 * coarse matrices and lambda_max, rebuilds the beta-dependent parts (level
 * betas, omega, coarsest inverse, dense inner levels, and the CUDA graph of
 * the batched solve loop when one was built).  Solves after it equal a fresh
 * rmg_method_prepare at this beta. */
int rmg_method_set_beta(rmg_method* pm, double beta);
int rmg_method_destroy(rmg_method* pm);
/* PreparedMethod::solve (krylov.cpp:651-668): rhs = X^T b, then the Krylov
 * solve; b has n_samples entries, w_out n_features.                     */
int rmg_method_solve(rmg_method* pm, const double* b, double* w_out, rmg_solve_report* report,
                     int32_t on_device);
/* Same solve from a prebuilt rhs = X^T b (the reference's timed region). */
int rmg_method_solve_rhs(rmg_method* pm, const double* rhs, double* w_out,
                         rmg_solve_report* report, int32_t on_device);
/* k right-hand sides (SURVEY §8(b) k_rhs): b is column-major n_samples x k, w_out
 * column-major n_features x k, reports[k] optional.  Column q equals
 * rmg_method_solve of column q to rounding.  For cg, jacobi_cg, pcg_vcycle and
 * pcg_vcycle_additive on a single-GPU matrix (CSR or dense) and 2 <= k <= 64 the k
 * columns run in LOCK STEP: rhs = X^T B is one block pass, every
 * operator application at every level is one block-operator call (rmg_ridge_
 * apply_block; dense coarse Grams as one skinny GEMM), reductions are per column
 * in a fixed order and a converged column freezes.  Other
 * methods (or RMG_BATCH_SEQ=1) solve the columns one after the other. */
int rmg_method_solve_batch(rmg_method* pm, const double* b, double* w_out, uint64_t k, rmg_solve_report* reports,
                           int32_t on_device);
/* Apply the level-0 preconditioner once: z = M^{-1} r (two_level_apply, krylov.cpp:379-425). */
int rmg_method_precondition(rmg_method* pm, const double* r, double* z, int32_t on_device);
/* PreparedMethod::coarse_size (krylov.hpp:229) and per-level introspection */
int rmg_method_info(const rmg_method* pm, uint64_t* n_levels, uint64_t* coarse_size);
int rmg_method_level(const rmg_method* pm, uint64_t level, uint64_t* n_features, uint64_t* nnz,
                     double* beta, double* omega);
/* labels of the aggregation from `level` to `level+1` (membership per feature) */
int rmg_method_level_labels(const rmg_method* pm, uint64_t level, int64_t* labels_out);
/* export the coarse matrix X_{level} (level >= 1) in CSR (for parity checks) */
int rmg_method_level_matrix(const rmg_method* pm, uint64_t level, uint64_t* row_offsets,
                            uint64_t* column_indices, double* values);

/* SystemSolution solve_system(x, beta, b, spec) (krylov.hpp:251-252) */
int rmg_solve_system(rmg_matrix* m, double beta, int32_t method_kind, const rmg_level_spec* levels,
                     uint64_t n_levels, const rmg_solver_config* solver, const double* b,
                     double* w_out, rmg_solve_report* report, uint64_t* coarse_size);

/* ---------------------------------------------------------------- profiling
 * Average device time (CUDA events on the context stream) of `reps`
 * applications of the level-`level` operator kernels, for the roofline. */
int rmg_method_time_operator(rmg_method* pm, uint64_t level, uint64_t reps, int32_t flush_l2,
                             double* ms_per_apply, double* ms_k1, double* ms_k2);
/* In-situ profiling: with `on`, every operator application of every level
 * inside real solves is bracketed by CUDA events (K1 = X v, K2 = X^T pass);
 * rmg_method_profile returns the accumulated applications and milliseconds
 * since profiling was (re)enabled. */
int rmg_method_set_profiling(rmg_method* pm, int32_t on);
int rmg_method_profile(const rmg_method* pm, uint64_t level, uint64_t* applications, double* ms_k1,
                       double* ms_k2);

#ifdef __cplusplus
}
#endif
#endif /* RIDGEMG_B200_H */
