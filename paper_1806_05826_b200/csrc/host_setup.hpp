// Host-side (C++) setup of the ridgemg_b200 path: the pieces of hierarchy
// construction that must reproduce the reference's floating-point order bit
// for bit (labels, aggregation weights, X_c values; SURVEY.md §2.1,
// Appendix B), plus the portable RNG and the BASELINE synthetic generators.
#pragma once

#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

namespace rmg {

struct InvalidArgument : std::invalid_argument {
  using std::invalid_argument::invalid_argument;
};
struct RuntimeError : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct CudaError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

// CounterRng (rng.hpp:25-72): splitmix64 over seed + k * 0x9E3779B97F4A7C15,
// Box-Muller normals with the sine variate cached.  glibc libm on the host.
class CounterRng {
 public:
  explicit CounterRng(uint64_t seed) : seed_(seed) {}
  uint64_t next_u64();
  double next_double();       // [0,1)
  double next_double_open();  // (0,1]
  double next_normal();
  uint64_t next_index(uint64_t n);

 private:
  uint64_t seed_, k_ = 0;
  double cached_ = 0.0;
  bool has_cached_ = false;
};

// Host CSR in the reference's FeatureMatrix shape (sparse.hpp:24-32).
struct HostCsr {
  int64_t n = 0, f = 0;
  std::vector<int64_t> ptr, idx;
  std::vector<double> val;
  int64_t nnz() const { return static_cast<int64_t>(idx.size()); }
};

// Validates the FeatureMatrix invariants (sparse.hpp:19-23).
void validate_csr(const HostCsr& m);
HostCsr transpose(const HostCsr& m);  // to_csc (sparse.cpp:75-99) as a CSR of X^T
HostCsr normalized_columns(const HostCsr& m);

// Clustering restatements (clustering.cpp), labels identical to the reference.
struct Clustering {
  std::vector<int64_t> labels;
  int64_t n_clusters = 0;
  uint64_t iterations = 0;
  bool converged = false;
  bool exact = true;
  double tolerance = 0.0;
};
Clustering kmeans(const HostCsr& xt, int64_t k, uint64_t max_iters, uint64_t seed, unsigned threads);
std::vector<int64_t> kmeanspp_seed(const HostCsr& xt, int64_t k, uint64_t seed, unsigned threads);
Clustering leader_follower(const HostCsr& xt, double tol);
Clustering leader_follower_target(const HostCsr& xt, int64_t target);

// Adjusted-average aggregation (coarsening.cpp:82-106) and X_c = X P
// (coarsening.cpp:112-148).
struct Aggregation {
  int64_t n_fine = 0, n_coarse = 0;
  std::vector<int32_t> label;     // fine -> cluster
  std::vector<double> weight;     // 1/sqrt(n_S)
  std::vector<int32_t> mptr, members;  // cluster -> sorted fine members
};
Aggregation make_aggregation(const std::vector<int64_t>& labels, int64_t n_clusters);
HostCsr coarsen(const HostCsr& x, const Aggregation& p);

// Coarsest level: dense A_c = sum_rows x_c x_c^T + beta I (krylov.cpp:350-365),
// Cholesky (throws RuntimeError when indefinite, krylov.cpp:367-375), and
// the explicit inverse used by the device GEMV.
std::vector<double> coarse_gram(const HostCsr& xc, double beta);
std::vector<double> spd_inverse(const std::vector<double>& a, int64_t n, const std::string& context);

// BASELINE.json synthetic generators (DESIGN.md §6 documents the recipes).
HostCsr synth_dense_clustered(int64_t n, int64_t f, int64_t groups, double noise, uint64_t seed);
HostCsr synth_sparse_zipf(int64_t n, int64_t f, double mean_nnz, double zipf_s, bool abs_normal_values,
                          uint64_t seed);
// Same distribution, one RNG stream per row (threaded): large measurement shards.
// rows [row0, row1) only (row1 < 0: all): per-rank generation of a row-sharded input
HostCsr synth_sparse_zipf_rows(int64_t n, int64_t f, double mean_nnz, double zipf_s, bool abs_normal_values,
                               uint64_t seed, int64_t row0 = 0, int64_t row1 = -1);

}  // namespace rmg
