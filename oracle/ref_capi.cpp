// TEST INFRASTRUCTURE ONLY — compiled into oracle/_ref/libridgemg_ref.so
// together with the reference's own, unmodified translation units
// (/root/reference/proj/src/{sparse,ridge,distance,clustering,coarsening,
// krylov,matrix_market}.cpp) by oracle/Makefile.  This file is glue: it turns
// the reference's C++ API (proj/include/ridgemg/*.hpp) into `extern "C"`
// entry points that pytest can load with ctypes.  It is never linked into,
// or called by, the product library.
//
// Two compositions below mirror reference code paths that take clustering
// as input rather than computing it, so the expensive reference k-means can
// be replaced by imported labels in parity runs (SURVEY.md §8(c) "cfg 2/3:
// imported labels"):
//   build_from_labels  mirrors build_hierarchy  (krylov.cpp:493-568)
//   ref_generate_rhs   mirrors generate_rhs     (analysis.cpp:225-232; the
//                      reference TU needs Eigen's EigenSolver, so the six
//                      lines are restated on top of the verbatim CounterRng
//                      and spmv_transpose).
#include <cmath>
#include <cstring>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "oracle_abi.h"
#include "synth.hpp"
#include "ridgemg/krylov.hpp"
#include "ridgemg/matrix_market.hpp"
#include "ridgemg/rng.hpp"

using namespace ridgemg;

namespace {

thread_local std::string g_err;

template <class F>
int guard(F&& f) {
  try {
    f();
    return 0;
  } catch (const std::invalid_argument& e) {
    g_err = e.what();
    return 1;
  } catch (const std::runtime_error& e) {
    g_err = e.what();
    return 2;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 3;
  }
}

FeatureMatrix* M(void* h) { return static_cast<FeatureMatrix*>(h); }

ClusterAssignment assignment_from_labels(const int64_t* labels, std::size_t f, std::size_t nc) {
  ClusterAssignment a;
  a.n_features = f;
  a.n_clusters = nc;
  a.membership.resize(f);
  a.sizes.assign(nc, 0);
  a.prototype_feature.assign(nc, ClusterAssignment::npos);
  for (std::size_t i = 0; i < f; ++i) {
    if (labels[i] < 0 || static_cast<std::size_t>(labels[i]) >= nc)
      throw std::invalid_argument("imported label out of range");
    const auto s = static_cast<std::size_t>(labels[i]);
    a.membership[i] = s;
    a.sizes[s] += 1;
    if (a.prototype_feature[s] == ClusterAssignment::npos) a.prototype_feature[s] = i;
  }
  return a;
}

// BASELINE cfg 2 extension: x_j / ||x_j||, norms accumulated in row order.
FeatureMatrix normalized_copy(const FeatureMatrix& x) {
  std::vector<double> sq(x.n_features, 0.0);
  for (std::size_t r = 0; r < x.n_samples; ++r)
    for (std::size_t k = x.row_offsets[r]; k < x.row_offsets[r + 1]; ++k)
      sq[x.column_indices[k]] += x.values[k] * x.values[k];
  for (double& v : sq) v = std::sqrt(v);
  FeatureMatrix y = x;
  for (std::size_t k = 0; k < y.values.size(); ++k) y.values[k] /= sq[y.column_indices[k]];
  return y;
}

ClusterAssignment cluster_level(const FeatureMatrix& current, const or_level_spec& s) {
  if (s.labels != nullptr) return assignment_from_labels(s.labels, current.n_features, s.n_clusters);
  const FeatureMatrix* src = &current;
  FeatureMatrix norm;
  if (s.normalize_columns) {
    norm = normalized_copy(current);
    src = &norm;
  }
  const CscMatrix cols = to_csc(*src);
  switch (s.clustering_kind) {
    case OR_CLUSTER_LEADER_TOLERANCE:
      return leader_follower(cols, s.tolerance, DistanceKind::euclidean, false);
    case OR_CLUSTER_LEADER_TARGET:
      return leader_follower_target(cols, s.target_size, DistanceKind::euclidean, false).assignment;
    case OR_CLUSTER_KMEANS:
      return kmeans(cols, s.target_size, s.kmeans_max_iters, s.seed).assignment;
  }
  throw std::invalid_argument("unknown clustering kind");
}

// Hierarchy assembled from the reference's public pieces in the order of
// build_hierarchy (krylov.cpp:493-568).
struct RefHierarchy {
  const FeatureMatrix* fine = nullptr;
  std::unique_ptr<RidgeOperator> fine_op;
  std::vector<std::unique_ptr<CoarseLevel>> coarse;
  std::vector<std::unique_ptr<GalerkinOperator>> ops;
  std::vector<std::unique_ptr<TwoLevelPreconditioner>> preconds;
  std::vector<double> omegas;

  const FeatureMatrix& level_matrix(std::size_t k) const {
    return k == 0 ? *fine : coarse[k - 1]->coarse_matrix;
  }
  const LinearOperator& level_op(std::size_t k) const {
    return k == 0 ? static_cast<const LinearOperator&>(*fine_op) : *ops[k - 1];
  }
};

std::unique_ptr<RefHierarchy> build_from_specs(const FeatureMatrix& x, double beta,
                                               const or_level_spec* specs, std::size_t n) {
  if (n == 0) throw std::invalid_argument("at least one level spec is required");
  for (std::size_t k = 0; k + 1 < n; ++k)
    if (specs[k].coarse_kind == OR_COARSE_DIRECT)
      throw std::invalid_argument("only the last level may use direct_cholesky");
  if (specs[n - 1].coarse_kind != OR_COARSE_DIRECT)
    throw std::invalid_argument("the coarsest level must use direct_cholesky");

  auto h = std::make_unique<RefHierarchy>();
  h->fine = &x;
  h->fine_op = std::make_unique<RidgeOperator>(x, beta);
  double level_beta = beta;
  for (std::size_t k = 0; k < n; ++k) {
    const FeatureMatrix& current = h->level_matrix(k);
    const double next_beta = specs[k].has_beta_override ? specs[k].beta_override : level_beta;
    ClusterAssignment a = cluster_level(current, specs[k]);
    if (a.n_clusters >= current.n_features)
      throw std::invalid_argument("level has no fewer clusters than features");
    h->coarse.push_back(
        std::make_unique<CoarseLevel>(coarsen(current, build_adjusted_average(a), next_beta)));
    h->ops.push_back(std::make_unique<GalerkinOperator>(*h->coarse.back()));
    level_beta = next_beta;
  }
  if (h->coarse.back()->coarse_matrix.n_features > kDirectSolveCap)
    throw std::invalid_argument("coarsest level above the direct-solve cap");
  for (std::size_t k = 0; k < n; ++k) {
    const GramOperator gram(h->level_matrix(k));
    const double lmax = estimate_lambda_max(gram, 1e-4, 200, 0x5eed + k).value;
    const double b = k == 0 ? beta : h->coarse[k - 1]->beta;
    h->omegas.push_back(2.0 / (b + lmax));
  }
  h->preconds.resize(n);
  for (std::size_t k = n; k-- > 0;) {
    TwoLevelPreconditioner::CoarseSolve solve;
    if (specs[k].coarse_kind == OR_COARSE_DIRECT) {
      solve = TwoLevelPreconditioner::DirectCoarse{};
    } else {
      TwoLevelPreconditioner::IterativeCoarse it;
      it.flexible = specs[k].coarse_kind == OR_COARSE_INNER_FCG;
      it.config.tol = specs[k].coarse_tol;
      it.config.max_iters = specs[k].coarse_max_iters;
      it.config.truncation = specs[k].coarse_truncation;
      it.preconditioner = it.flexible ? h->preconds[k + 1].get() : nullptr;
      solve = it;
    }
    h->preconds[k] = std::make_unique<TwoLevelPreconditioner>(h->level_op(k), *h->coarse[k],
                                                              h->omegas[k], solve);
  }
  return h;
}

void fill_report(const SolveReport& r, or_solve_report* out) {
  if (!out) return;
  out->iterations = r.iterations;
  out->converged = r.converged ? 1 : 0;
  out->wall_time_s = r.wall_time_s;
  if (out->residual_history) {
    const std::size_t n = std::min<std::size_t>(out->residual_capacity, r.residual_history.size());
    std::memcpy(out->residual_history, r.residual_history.data(), n * sizeof(double));
  }
  if (out->inner_iterations) {
    const std::size_t n = std::min<std::size_t>(out->inner_capacity, r.inner_iterations.size());
    for (std::size_t i = 0; i < n; ++i) out->inner_iterations[i] = r.inner_iterations[i];
  }
}

}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

int ref_set_num_threads(unsigned t) {
  return guard([&] { set_num_threads(t); });
}

void* ref_matrix_from_csr(uint64_t n, uint64_t f, uint64_t nnz, const uint64_t* rp,
                          const uint64_t* ci, const double* v) {
  auto* m = new FeatureMatrix;
  m->n_samples = n;
  m->n_features = f;
  m->row_offsets.assign(rp, rp + n + 1);
  m->column_indices.assign(ci, ci + nnz);
  if (v) {
    m->values.assign(v, v + nnz);
  } else {
    m->values.assign(nnz, 1.0);
  }
  return m;
}

void* ref_matrix_from_triplets(uint64_t n, uint64_t f, uint64_t nt, const uint64_t* rows,
                               const uint64_t* cols, const double* vals) {
  FeatureMatrix* out = nullptr;
  const int rc = guard([&] {
    std::vector<Triplet> ts(nt);
    for (uint64_t i = 0; i < nt; ++i) ts[i] = {rows[i], cols[i], vals[i]};
    out = new FeatureMatrix(csr_from_triplets(n, f, ts));
  });
  return rc == 0 ? out : nullptr;
}

void* ref_read_matrix_market(const char* path) {
  FeatureMatrix* out = nullptr;
  const int rc = guard([&] { out = new FeatureMatrix(read_matrix_market(std::filesystem::path(path))); });
  return rc == 0 ? out : nullptr;
}

// BASELINE synthetic inputs (oracle/synth.hpp) drawn from the reference's own
// CounterRng (rng.hpp:25-72): the reference arm builds its X without the
// product library.  The CSR is filled directly (csr_from_triplets would need
// ~3x the memory at cfg 3 / cfg 5 scale).
void* ref_synth_sparse_zipf(uint64_t n, uint64_t f, double mean, double s, int32_t values, uint64_t seed,
                            int32_t row_streams) {
  auto g = oracle_synth::sparse_zipf<CounterRng>(static_cast<int64_t>(n), static_cast<int64_t>(f), mean, s,
                                                 values != 0, seed, row_streams != 0);
  auto* m = new FeatureMatrix;
  m->n_samples = n;
  m->n_features = f;
  m->row_offsets = std::move(g.ptr);
  m->column_indices.assign(g.idx.begin(), g.idx.end());
  std::vector<uint64_t>().swap(g.idx);
  if (values)
    m->values = std::move(g.val);
  else
    m->values.assign(m->column_indices.size(), 1.0);
  return m;
}
void* ref_synth_dense_clustered(uint64_t n, uint64_t f, uint64_t groups, double noise, uint64_t seed) {
  auto g = oracle_synth::dense_clustered<CounterRng>(static_cast<int64_t>(n), static_cast<int64_t>(f),
                                                     static_cast<int64_t>(groups), noise, seed);
  return ref_matrix_from_csr(n, f, g.idx.size(), g.ptr.data(), g.idx.data(), g.val.data());
}

void ref_matrix_free(void* h) { delete M(h); }

int ref_matrix_shape(void* h, uint64_t* n, uint64_t* f, uint64_t* nnz) {
  *n = M(h)->n_samples;
  *f = M(h)->n_features;
  *nnz = M(h)->nnz();
  return 0;
}

int ref_matrix_export(void* h, uint64_t* rp, uint64_t* ci, double* v) {
  const FeatureMatrix& m = *M(h);
  std::memcpy(rp, m.row_offsets.data(), (m.n_samples + 1) * sizeof(uint64_t));
  std::memcpy(ci, m.column_indices.data(), m.nnz() * sizeof(uint64_t));
  std::memcpy(v, m.values.data(), m.nnz() * sizeof(double));
  return 0;
}

int ref_spmv(void* h, const double* v, double* y) {
  return guard([&] {
    spmv(*M(h), std::span<const double>(v, M(h)->n_features), std::span<double>(y, M(h)->n_samples));
  });
}

int ref_spmv_transpose(void* h, const double* u, double* y) {
  return guard([&] {
    spmv_transpose(*M(h), std::span<const double>(u, M(h)->n_samples),
                   std::span<double>(y, M(h)->n_features));
  });
}

int ref_ridge_apply(void* h, double beta, const double* w, double* out) {
  return guard([&] {
    const RidgeOperator op(*M(h), beta);
    op.apply(std::span<const double>(w, M(h)->n_features), std::span<double>(out, M(h)->n_features));
  });
}

int ref_gram_diagonal(void* h, double beta, double* out) {
  return guard([&] {
    const RidgeOperator op(*M(h), beta);
    const DenseVector d = gram_diagonal(op);
    std::memcpy(out, d.data(), d.size() * sizeof(double));
  });
}

int ref_lambda_max(void* h, double tol, uint64_t max_iters, uint64_t seed, double* value,
                   uint64_t* iters, int32_t* converged) {
  return guard([&] {
    const GramOperator g(*M(h));
    const PowerIterationResult r = estimate_lambda_max(g, tol, max_iters, seed);
    *value = r.value;
    *iters = r.iterations;
    *converged = r.converged ? 1 : 0;
  });
}

int ref_normals(uint64_t seed, uint64_t n, double* out) {
  CounterRng rng(seed);
  for (uint64_t i = 0; i < n; ++i) out[i] = rng.next_normal();
  return 0;
}

int ref_generate_rhs(void* h, uint64_t seed, double* b, double* rhs) {
  return guard([&] {
    CounterRng rng(seed);
    DenseVector bv(M(h)->n_samples);
    for (double& v : bv) v = rng.next_normal();
    const DenseVector r = spmv_transpose(*M(h), bv);
    std::memcpy(b, bv.data(), bv.size() * sizeof(double));
    if (rhs) std::memcpy(rhs, r.data(), r.size() * sizeof(double));
  });
}

int ref_kmeanspp_seed(void* h, uint64_t k, uint64_t seed, int64_t* chosen) {
  return guard([&] {
    const auto c = kmeanspp_seed(to_csc(*M(h)), k, seed);
    for (std::size_t i = 0; i < c.size(); ++i) chosen[i] = static_cast<int64_t>(c[i]);
  });
}

int ref_kmeans(void* h, uint64_t k, uint64_t max_iters, uint64_t seed, int32_t normalize,
               int64_t* labels, uint64_t* iters, int32_t* converged) {
  return guard([&] {
    const FeatureMatrix src = normalize ? normalized_copy(*M(h)) : *M(h);
    const KmeansResult r = kmeans(to_csc(src), k, max_iters, seed);
    for (std::size_t i = 0; i < r.assignment.n_features; ++i)
      labels[i] = static_cast<int64_t>(r.assignment.membership[i]);
    *iters = r.iterations;
    *converged = r.converged ? 1 : 0;
  });
}

int ref_leader_follower(void* h, double tol, int64_t* labels, uint64_t* n_clusters) {
  return guard([&] {
    const ClusterAssignment a = leader_follower(to_csc(*M(h)), tol, DistanceKind::euclidean);
    for (std::size_t i = 0; i < a.n_features; ++i) labels[i] = static_cast<int64_t>(a.membership[i]);
    *n_clusters = a.n_clusters;
  });
}

int ref_leader_follower_target(void* h, uint64_t target, int64_t* labels, uint64_t* n_clusters,
                               int32_t* exact, double* tol) {
  return guard([&] {
    const LeaderTargetResult r = leader_follower_target(to_csc(*M(h)), target, DistanceKind::euclidean);
    for (std::size_t i = 0; i < r.assignment.n_features; ++i)
      labels[i] = static_cast<int64_t>(r.assignment.membership[i]);
    *n_clusters = r.assignment.n_clusters;
    *exact = r.exact ? 1 : 0;
    *tol = r.tolerance;
  });
}

void* ref_coarsen(void* h, const int64_t* labels, uint64_t n_clusters, double beta) {
  FeatureMatrix* out = nullptr;
  guard([&] {
    const ClusterAssignment a = assignment_from_labels(labels, M(h)->n_features, n_clusters);
    CoarseLevel lvl = coarsen(*M(h), build_adjusted_average(a), beta);
    out = new FeatureMatrix(std::move(lvl.coarse_matrix));
  });
  return out;
}

int ref_two_level_apply(void* h, double beta, const int64_t* labels, uint64_t n_clusters,
                        double omega, const double* r, double* z) {
  return guard([&] {
    const FeatureMatrix& x = *M(h);
    const RidgeOperator a(x, beta);
    const CoarseLevel level =
        coarsen(x, build_adjusted_average(assignment_from_labels(labels, x.n_features, n_clusters)), beta);
    const TwoLevelPreconditioner m(a, level, omega, TwoLevelPreconditioner::DirectCoarse{});
    m.apply(std::span<const double>(r, x.n_features), std::span<double>(z, x.n_features));
  });
}

// PreparedMethod::solve (krylov.cpp:651-668) for cg / jacobi_cg, and the
// build_hierarchy-ordered composition above for the (F)CG hierarchy methods.
int ref_solve(void* h, double beta, int32_t method, const or_level_spec* levels, uint64_t n_levels,
              const or_solver_config* cfg, const double* b, double* w, or_solve_report* rep) {
  return guard([&] {
    const FeatureMatrix& x = *M(h);
    SolverConfig sc;
    sc.tol = cfg->tol;
    sc.max_iters = cfg->max_iters;
    sc.truncation = cfg->truncation;
    const DenseVector bv(b, b + x.n_samples);
    if (method == OR_METHOD_CG || method == OR_METHOD_JACOBI_CG) {
      MethodSpec spec;
      spec.kind = method == OR_METHOD_CG ? MethodKind::cg : MethodKind::jacobi_cg;
      spec.solver = sc;
      const PreparedMethod pm(x, beta, spec);
      auto [sol, report] = pm.solve(bv);
      std::memcpy(w, sol.data(), sol.size() * sizeof(double));
      fill_report(report, rep);
      if (rep) {
        rep->n_levels = 1;
        rep->level_sizes[0] = x.n_features;
      }
      return;
    }
    std::vector<or_level_spec> specs(levels, levels + n_levels);
    if (method == OR_METHOD_FCG_TWOLEVEL || method == OR_METHOD_FGMRES_TWOLEVEL) {  // krylov.cpp:628-635
      specs.resize(1);
      specs[0].coarse_kind = OR_COARSE_DIRECT;
    }
    auto hier = build_from_specs(x, beta, specs.data(), specs.size());
    const DenseVector rhs = spmv_transpose(x, bv);  // krylov.cpp:655
    auto [sol, report] = method == OR_METHOD_FGMRES_TWOLEVEL ? fgmres(*hier->fine_op, rhs, sc, *hier->preconds[0])
                                                             : fcg(*hier->fine_op, rhs, sc, *hier->preconds[0]);
    std::memcpy(w, sol.data(), sol.size() * sizeof(double));
    fill_report(report, rep);
    if (rep) {
      rep->n_levels = specs.size() + 1;
      for (std::size_t k = 0; k < specs.size() && k < 8; ++k) rep->omega[k] = hier->omegas[k];
      for (std::size_t k = 0; k <= specs.size() && k < 8; ++k)
        rep->level_sizes[k] = hier->level_matrix(k).n_features;
    }
  });
}

}  // extern "C"
