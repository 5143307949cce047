// ridgemg_b200.hpp — the reference's C++ solver interface (proj/include/ridgemg:
// sparse.hpp, ridge.hpp, krylov.hpp, analysis.hpp), re-created header-only over
// the B200 C ABI (ridgemg_b200.h).  A reference user replaces
//     #include "ridgemg/krylov.hpp"      with   #include "ridgemg_b200.hpp"
//     namespace ridgemg                  with   namespace ridgemg::b200
// and links libridgemg_b200.so.  Names, fields, defaults and exception types
// follow the reference: std::invalid_argument for dimension/spec errors,
// std::runtime_error for numerical breakdown; non-convergence is reported in
// SolveReport::converged.  There is no CPU fallback.
#pragma once

#include <cstdint>
#include <memory>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "ridgemg_b200.h"

namespace ridgemg::b200 {

using DenseVector = std::vector<double>;  // sparse.hpp:9

// sparse.hpp:24-32
struct FeatureMatrix {
  std::size_t n_samples = 0;
  std::size_t n_features = 0;
  std::vector<std::size_t> row_offsets;
  std::vector<std::size_t> column_indices;
  std::vector<double> values;
  [[nodiscard]] std::size_t nnz() const { return values.size(); }
};

// Status -> the reference's exception types.
inline void check(int rc) {
  if (rc == RMG_OK) return;
  const std::string msg = rmg_last_error();
  if (rc == RMG_ERR_INVALID_ARGUMENT) throw std::invalid_argument(msg);
  throw std::runtime_error(msg);
}

// krylov.hpp:16-23 (omega_mode/omega_fixed are dead in the reference; see LevelSpec::omega_override)
struct SolverConfig {
  double tol = 1e-6;
  std::size_t max_iters = 1000;
  std::size_t truncation = 20;
};

// krylov.hpp:25-31
struct SolveReport {
  std::size_t iterations = 0;
  std::vector<double> residual_history;
  bool converged = false;
  double wall_time_s = 0.0;
  std::vector<std::size_t> inner_iterations;
};

// krylov.hpp:135-146 (+ imported labels for parity runs)
struct ClusteringChoice {
  enum class Kind { leader_tolerance = RMG_CLUSTER_LEADER_TOLERANCE, leader_target = RMG_CLUSTER_LEADER_TARGET,
                    kmeans = RMG_CLUSTER_KMEANS, kmeans_sketch = RMG_CLUSTER_KMEANS_SKETCH,
                    imported = RMG_CLUSTER_IMPORTED };
  Kind kind = Kind::leader_tolerance;
  double tolerance = 1.0;
  std::size_t target_size = 0;
  std::uint64_t seed = 0;
  std::size_t kmeans_max_iters = 100;
  bool normalize_columns = false;
  std::vector<std::int64_t> labels;  // kind == imported
  std::size_t n_clusters = 0;
  std::size_t sketch_dim = 32;  // kind == kmeans_sketch (extension)
};

// krylov.hpp:154-160
struct CoarseSolveChoice {
  enum class Kind { direct_cholesky = RMG_COARSE_DIRECT_CHOLESKY, inner_cg = RMG_COARSE_INNER_CG,
                    inner_fcg = RMG_COARSE_INNER_FCG };
  Kind kind = Kind::direct_cholesky;
  double tol = 1e-6;
  std::size_t max_iters = 500;
  std::size_t truncation = 20;
};

// krylov.hpp:162-167
struct LevelSpec {
  ClusteringChoice clustering;
  CoarseSolveChoice solver;
  bool has_beta_override = false;
  double beta_override = 0.0;
  bool has_omega_override = false;
  double omega_override = 0.0;
  bool additive = false;  // pcg_vcycle_additive: this level enters additively too (extension)
};

// krylov.hpp:207-218
enum class MethodKind { cg = RMG_METHOD_CG, jacobi_cg = RMG_METHOD_JACOBI_CG, fcg_twolevel = RMG_METHOD_FCG_TWOLEVEL,
                        fcg_multilevel = RMG_METHOD_FCG_MULTILEVEL, fgmres_twolevel = RMG_METHOD_FGMRES_TWOLEVEL,
                        pcg_vcycle = RMG_METHOD_PCG_VCYCLE /* extension */,
                        pcg_vcycle_additive = RMG_METHOD_PCG_VCYCLE_ADDITIVE /* extension */ };

inline MethodKind method_from_string(const std::string& s) {  // krylov.cpp:574-581
  if (s == "cg") return MethodKind::cg;
  if (s == "jacobi_cg") return MethodKind::jacobi_cg;
  if (s == "fcg_twolevel") return MethodKind::fcg_twolevel;
  if (s == "fcg_multilevel") return MethodKind::fcg_multilevel;
  if (s == "fgmres_twolevel") return MethodKind::fgmres_twolevel;
  if (s == "pcg_vcycle") return MethodKind::pcg_vcycle;
  if (s == "pcg_vcycle_additive") return MethodKind::pcg_vcycle_additive;
  throw std::invalid_argument("unknown method: '" + s + "'");
}

struct MethodSpec {
  MethodKind kind = MethodKind::cg;
  std::vector<LevelSpec> levels;
  SolverConfig solver;
};

// One device + stream; the reference has process-global state instead, so a
// default context (device 0) is used when none is given.
class Context {
 public:
  explicit Context(int device = 0) { check(rmg_context_create(device, &h_)); }
  ~Context() { rmg_context_destroy(h_); }
  Context(const Context&) = delete;
  Context& operator=(const Context&) = delete;
  rmg_context* get() const { return h_; }
  static Context& default_context() {
    static Context ctx(0);
    return ctx;
  }

 private:
  rmg_context* h_ = nullptr;
};

// X and X^T resident in HBM (rmg_matrix); the FeatureMatrix may be released after upload.
class DeviceMatrix {
 public:
  explicit DeviceMatrix(const FeatureMatrix& x, Context& ctx = Context::default_context())
      : n_(x.n_samples), f_(x.n_features) {
    static_assert(sizeof(std::size_t) == sizeof(std::uint64_t), "size_t must be 64-bit");
    check(rmg_matrix_create_csr(ctx.get(), x.n_samples, x.n_features,
                                reinterpret_cast<const std::uint64_t*>(x.row_offsets.data()),
                                reinterpret_cast<const std::uint64_t*>(x.column_indices.data()),
                                x.values.empty() ? nullptr : x.values.data(), 1, &h_));
  }
  ~DeviceMatrix() { rmg_matrix_destroy(h_); }
  DeviceMatrix(const DeviceMatrix&) = delete;
  DeviceMatrix& operator=(const DeviceMatrix&) = delete;
  rmg_matrix* get() const { return h_; }
  std::size_t n_samples() const { return n_; }
  std::size_t n_features() const { return f_; }

  DenseVector spmv(const DenseVector& v) const {  // sparse.hpp:61
    if (v.size() != f_) throw std::invalid_argument("spmv: input length != n_features");
    DenseVector y(n_);
    check(rmg_spmv(h_, v.data(), y.data(), 0));
    return y;
  }
  DenseVector spmv_transpose(const DenseVector& u) const {  // sparse.hpp:66
    if (u.size() != n_) throw std::invalid_argument("spmv_transpose: input length != n_samples");
    DenseVector y(f_);
    check(rmg_spmv_transpose(h_, u.data(), y.data(), 0));
    return y;
  }
  DenseVector ridge_apply(double beta, const DenseVector& w) const {  // ridge.cpp:16-24
    if (w.size() != f_) throw std::invalid_argument("RidgeOperator::apply: dimension mismatch");
    DenseVector out(f_);
    check(rmg_ridge_apply(h_, beta, w.data(), out.data(), 0));
    return out;
  }
  DenseVector gram_diagonal(double beta) const {  // ridge.cpp:30-37
    DenseVector out(f_);
    check(rmg_gram_diagonal(h_, beta, out.data(), 0));
    return out;
  }

 private:
  rmg_matrix* h_ = nullptr;
  std::size_t n_ = 0, f_ = 0;
};

// analysis.hpp:71-75
struct RhsSample {
  DenseVector b;
  DenseVector rhs;
};
inline RhsSample generate_rhs(const DeviceMatrix& x, std::uint64_t seed) {
  RhsSample s{DenseVector(x.n_samples()), DenseVector(x.n_features())};
  check(rmg_generate_rhs(x.get(), seed, s.b.data(), s.rhs.data()));
  return s;
}

namespace detail {
inline std::vector<rmg_level_spec> to_c(const std::vector<LevelSpec>& levels) {
  std::vector<rmg_level_spec> out(levels.size());
  for (std::size_t i = 0; i < levels.size(); ++i) {
    const LevelSpec& l = levels[i];
    rmg_level_spec& s = out[i];
    s = rmg_level_spec{};
    s.clustering_kind = static_cast<int32_t>(l.clustering.kind);
    s.tolerance = l.clustering.tolerance;
    s.target_size = l.clustering.target_size;
    s.seed = l.clustering.seed;
    s.kmeans_max_iters = l.clustering.kmeans_max_iters;
    s.normalize_columns = l.clustering.normalize_columns ? 1 : 0;
    s.labels = l.clustering.labels.empty() ? nullptr : l.clustering.labels.data();
    s.n_clusters = l.clustering.n_clusters;
    s.sketch_dim = l.clustering.sketch_dim;
    s.coarse_kind = static_cast<int32_t>(l.solver.kind);
    s.coarse_tol = l.solver.tol;
    s.coarse_max_iters = l.solver.max_iters;
    s.coarse_truncation = l.solver.truncation;
    s.has_beta_override = l.has_beta_override ? 1 : 0;
    s.beta_override = l.beta_override;
    s.additive = l.additive ? 1 : 0;
    s.has_omega_override = l.has_omega_override ? 1 : 0;
    s.omega_override = l.omega_override;
  }
  return out;
}
}  // namespace detail

// krylov.hpp:222-242: setup in the constructor (clustering, hierarchy, omegas,
// coarsest factorization), then solve(b) for any b.  The DeviceMatrix must
// outlive the method (ridge.hpp:37 lifetime contract).
class PreparedMethod {
 public:
  PreparedMethod(const DeviceMatrix& x, double beta, MethodSpec spec) : x_(&x), spec_(std::move(spec)) {
    const auto lv = detail::to_c(spec_.levels);
    const rmg_solver_config cfg{spec_.solver.tol, spec_.solver.max_iters, spec_.solver.truncation};
    check(rmg_method_prepare(x.get(), beta, static_cast<int32_t>(spec_.kind), lv.empty() ? nullptr : lv.data(),
                             lv.size(), &cfg, &h_));
    std::uint64_t nl = 0, cs = 0;
    check(rmg_method_info(h_, &nl, &cs));
    coarse_size_ = cs;
  }
  ~PreparedMethod() { rmg_method_destroy(h_); }
  PreparedMethod(const PreparedMethod&) = delete;
  PreparedMethod& operator=(const PreparedMethod&) = delete;

  // krylov.cpp:651-668
  [[nodiscard]] std::pair<DenseVector, SolveReport> solve(const DenseVector& b) const {
    if (b.size() != x_->n_samples()) throw std::invalid_argument("PreparedMethod::solve: b length != n_samples");
    DenseVector w(x_->n_features());
    std::vector<double> hist(spec_.solver.max_iters + 1);
    std::vector<std::uint64_t> inner(spec_.solver.max_iters + 1);
    rmg_solve_report rep{};
    rep.residual_history = hist.data();
    rep.residual_capacity = hist.size();
    rep.inner_iterations = inner.data();
    rep.inner_capacity = inner.size();
    check(rmg_method_solve(h_, b.data(), w.data(), &rep, 0));
    SolveReport r;
    r.iterations = rep.iterations;
    r.converged = rep.converged != 0;
    r.wall_time_s = rep.wall_time_s;
    const std::size_t nh = rep.iterations ? rep.iterations : (rep.converged ? 1 : 0);
    r.residual_history.assign(hist.begin(), hist.begin() + nh);
    if (spec_.kind != MethodKind::cg && spec_.kind != MethodKind::jacobi_cg)
      r.inner_iterations.assign(inner.begin(), inner.begin() + rep.iterations);
    return {std::move(w), std::move(r)};
  }

  [[nodiscard]] std::size_t coarse_size() const { return coarse_size_; }
  [[nodiscard]] const MethodSpec& spec() const { return spec_; }
  rmg_method* get() const { return h_; }

 private:
  const DeviceMatrix* x_;
  MethodSpec spec_;
  rmg_method* h_ = nullptr;
  std::size_t coarse_size_ = 0;
};

// krylov.hpp:244-252
struct SystemSolution {
  DenseVector w;
  SolveReport report;
  std::size_t coarse_size = 0;
};

inline SystemSolution solve_system(const DeviceMatrix& x, double beta, const DenseVector& b, const MethodSpec& spec) {
  const PreparedMethod prepared(x, beta, spec);
  auto [w, report] = prepared.solve(b);
  return SystemSolution{std::move(w), std::move(report), prepared.coarse_size()};
}

}  // namespace ridgemg::b200
