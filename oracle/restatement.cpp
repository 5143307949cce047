// TEST INFRASTRUCTURE ONLY — the CPU oracle.  Built into
// oracle/_build/libridgemg_oracle.so by oracle/Makefile.  Only tests/,
// __graft_entry__.smoke() and bench.py's cpu_baseline leg may load it; the
// product library never links or calls it.
//
// A sequential CPU restatement of the reference solve path
// (/root/reference/proj), written against plain arrays, that keeps the
// reference's floating-point evaluation order so it can be pinned bit for
// bit against the verbatim reference build in oracle/_ref (see
// tests/test_oracle_pin.py).  Each routine cites the reference lines it
// restates.  Differences from the reference are only in data structures:
//   * int64 indices instead of size_t vectors;
//   * k-means keeps prototypes transposed (N x K, cluster-contiguous) and
//     evaluates features on worker threads; every (feature, prototype) sum
//     is still accumulated sequentially in the reference's order, so the
//     labels are identical;
//   * the dense coarsest factorization is an unblocked Cholesky (Eigen's
//     blocked LLT is not pinned by the reference tests).
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <limits>
#include <memory>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include "oracle_abi.h"
#include "synth.hpp"

namespace {

thread_local std::string g_err;
using Vec = std::vector<double>;

// ---------------------------------------------------------------- RNG
// rng.hpp:25-72: splitmix64 over seed + k * golden, Box-Muller with a cached
// sine variate.
struct Rng {
  uint64_t seed, ctr = 0;
  bool spare_ok = false;
  double spare = 0.0;
  explicit Rng(uint64_t s) : seed(s) {}
  uint64_t u64() {
    uint64_t z = seed + (++ctr) * 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
  }
  double unit() { return static_cast<double>(u64() >> 11) * 0x1.0p-53; }
  double unit_open() { return (static_cast<double>(u64() >> 11) + 1.0) * 0x1.0p-53; }
  double normal() {
    if (spare_ok) {
      spare_ok = false;
      return spare;
    }
    const double a = unit_open(), b = unit();
    const double rad = std::sqrt(-2.0 * std::log(a));
    const double th = 2.0 * 3.141592653589793238462643383279502884 * b;
    spare = rad * std::sin(th);
    spare_ok = true;
    return rad * std::cos(th);
  }
  uint64_t index(uint64_t n) {
    const auto v = static_cast<uint64_t>(unit() * static_cast<double>(n));
    return v >= n ? n - 1 : v;
  }
  // the reference's method names (rng.hpp:36-69), for oracle/synth.hpp
  double next_double() { return unit(); }
  double next_normal() { return normal(); }
  uint64_t next_index(uint64_t n) { return index(n); }
};

// ---------------------------------------------------------------- CSR
struct Csr {  // sparse.hpp:24-32 (samples x features)
  int64_t n = 0, f = 0;
  std::vector<int64_t> ptr, idx;
  Vec val;
  int64_t nnz() const { return static_cast<int64_t>(val.size()); }
};

struct Csc {  // sparse.hpp:36-50, built like to_csc (sparse.cpp:75-99)
  int64_t n = 0, f = 0;
  std::vector<int64_t> ptr, row;
  Vec val;
};

Csc transpose_of(const Csr& m) {
  Csc c;
  c.n = m.n;
  c.f = m.f;
  c.ptr.assign(m.f + 1, 0);
  c.row.resize(m.nnz());
  c.val.resize(m.nnz());
  for (int64_t k = 0; k < m.nnz(); ++k) c.ptr[m.idx[k] + 1]++;
  for (int64_t j = 0; j < m.f; ++j) c.ptr[j + 1] += c.ptr[j];
  std::vector<int64_t> fill(c.ptr.begin(), c.ptr.end() - 1);
  for (int64_t r = 0; r < m.n; ++r)
    for (int64_t k = m.ptr[r]; k < m.ptr[r + 1]; ++k) {
      const int64_t d = fill[m.idx[k]]++;
      c.row[d] = r;
      c.val[d] = m.val[k];
    }
  return c;
}

int env_int(const char* name) {
  const char* e = std::getenv(name);
  return e == nullptr ? 0 : std::atoi(e);
}

// ORC_K1_POP=1 (envelope diagnostics): every row summed in descending column
// popularity (the GPU's SELL-32 element order)
const std::vector<int64_t>& popularity_order(const Csr& m) {
  static thread_local const Csr* key = nullptr;
  static thread_local std::vector<int64_t> perm;  // entries of each row, most popular column first
  if (key == &m && perm.size() == static_cast<size_t>(m.ptr[m.n])) return perm;
  std::vector<int64_t> cnt(m.f, 0);
  for (int64_t k = 0; k < m.ptr[m.n]; ++k) ++cnt[m.idx[k]];
  std::vector<int64_t> order(m.f), rank(m.f);
  for (int64_t j = 0; j < m.f; ++j) order[j] = j;
  std::stable_sort(order.begin(), order.end(), [&](int64_t a, int64_t b) { return cnt[a] > cnt[b]; });
  for (int64_t j = 0; j < m.f; ++j) rank[order[j]] = j;
  perm.resize(m.ptr[m.n]);
  for (int64_t r = 0; r < m.n; ++r) {
    for (int64_t k = m.ptr[r]; k < m.ptr[r + 1]; ++k) perm[k] = k;
    std::sort(perm.begin() + m.ptr[r], perm.begin() + m.ptr[r + 1],
              [&](int64_t a, int64_t b) { return rank[m.idx[a]] < rank[m.idx[b]]; });
  }
  key = &m;
  return perm;
}

// sparse.cpp:103-112 — per row, sequential in stored (increasing column) order
void mul(const Csr& m, const double* v, double* y) {
  static const bool pop = env_int("ORC_K1_POP") != 0;
  if (pop) {
    const std::vector<int64_t>& perm = popularity_order(m);
    for (int64_t r = 0; r < m.n; ++r) {
      double s = 0.0;
      for (int64_t k = m.ptr[r]; k < m.ptr[r + 1]; ++k) s += m.val[perm[k]] * v[m.idx[perm[k]]];
      y[r] = s;
    }
    return;
  }
  for (int64_t r = 0; r < m.n; ++r) {
    double s = 0.0;
    for (int64_t k = m.ptr[r]; k < m.ptr[r + 1]; ++k) s += m.val[k] * v[m.idx[k]];
    y[r] = s;
  }
}

// sparse.cpp:152-158,114-123 — zero fill, then scatter rows in order, skipping u_r == 0
void mul_t(const Csr& m, const double* u, double* y) {
  // ORC_XT_SEG=s (envelope diagnostics): every column summed in row segments of s
  // rows, the segment sums added in order (the GPU's segmented X^T pass class)
  static const int64_t seg = env_int("ORC_XT_SEG");
  // ORC_XT_SEGNNZ=c: every column summed in segments of c of its own entries (row
  // order), the segment sums added in order -- the GPU's segmented X^T schedule
  static const int64_t segnnz = env_int("ORC_XT_SEGNNZ");
  if (segnnz > 0) {
    std::vector<int64_t> cnt(m.f, 0), done(m.f, 0);
    for (int64_t k = 0; k < m.ptr[m.n]; ++k) ++cnt[m.idx[k]];
    Vec part(m.f, 0.0);
    std::fill(y, y + m.f, 0.0);
    for (int64_t r = 0; r < m.n; ++r) {
      const double ur = u[r];
      for (int64_t k = m.ptr[r]; k < m.ptr[r + 1]; ++k) {
        const int64_t j = m.idx[k];
        if (cnt[j] > segnnz) {  // long column: segment partials
          if (ur != 0.0) part[j] += m.val[k] * ur;
          if (++done[j] % segnnz == 0 || done[j] == cnt[j]) {
            y[j] += part[j];
            part[j] = 0.0;
          }
        } else if (ur != 0.0) {
          y[j] += m.val[k] * ur;
        }
      }
    }
    return;
  }
  if (seg > 0 && m.n > seg) {
    std::fill(y, y + m.f, 0.0);
    Vec part(m.f);
    for (int64_t r0 = 0; r0 < m.n; r0 += seg) {
      std::fill(part.begin(), part.end(), 0.0);
      for (int64_t r = r0; r < std::min(m.n, r0 + seg); ++r) {
        const double ur = u[r];
        if (ur == 0.0) continue;
        for (int64_t k = m.ptr[r]; k < m.ptr[r + 1]; ++k) part[m.idx[k]] += m.val[k] * ur;
      }
      for (int64_t j = 0; j < m.f; ++j) y[j] += part[j];
    }
    return;
  }
  std::fill(y, y + m.f, 0.0);
  for (int64_t r = 0; r < m.n; ++r) {
    const double ur = u[r];
    if (ur == 0.0) continue;
    for (int64_t k = m.ptr[r]; k < m.ptr[r + 1]; ++k) y[m.idx[k]] += m.val[k] * ur;
  }
}

// Rounding-envelope diagnostics (never set by the tests' pinned
// runs): ORC_DOT_TREE=1 sums dot products pairwise in blocks of 256 (the GPU's
// order class), ORC_OMEGA_ULP=k moves every omega_k by k ulps, ORC_COARSE_INV=1
// applies the coarsest level through its explicit inverse (the GPU's choice).

// sparse.cpp:184-191
double dotp(const double* a, const double* b, int64_t n) {
  static const int tree = env_int("ORC_DOT_TREE");
  if (tree == 2) {  // fully pairwise (the GPU's grid reduction is of this accuracy class)
    std::vector<double> part(static_cast<size_t>(n));
    for (int64_t i = 0; i < n; ++i) part[i] = a[i] * b[i];
    for (int64_t w = 1; w < n; w *= 2)
      for (int64_t i = 0; i + w < n; i += 2 * w) part[i] += part[i + w];
    return n > 0 ? part[0] : 0.0;
  }
  if (tree) {
    double total = 0.0;
    for (int64_t b0 = 0; b0 < n; b0 += 256) {
      double part[256];
      const int64_t m = std::min<int64_t>(256, n - b0);
      for (int64_t i = 0; i < m; ++i) part[i] = a[b0 + i] * b[b0 + i];
      for (int64_t w = 1; w < m; w *= 2)
        for (int64_t i = 0; i + w < m; i += 2 * w) part[i] += part[i + w];
      total += part[0];
    }
    return total;
  }
  double s = 0.0;
  for (int64_t i = 0; i < n; ++i) s += a[i] * b[i];
  return s;
}
double nrm(const double* a, int64_t n) { return std::sqrt(dotp(a, a, n)); }

// ---------------------------------------------------------------- operators
// ridge.cpp:16-24 (beta >= 0) and GalerkinOperator::apply, adjusted-average
// branch (coarsening.cpp:174-185): w -> X^T (X w) + beta w, beta added last.
struct Op {
  const Csr* x = nullptr;
  double beta = 0.0;
  bool add_beta = true;  // false: GramOperator (ridge.cpp:39-46)
  mutable Vec tmp;
  int64_t dim() const { return x->f; }
  void apply(const double* w, double* out) const {
    tmp.assign(x->n, 0.0);
    mul(*x, w, tmp.data());
    mul_t(*x, tmp.data(), out);
    if (add_beta)
      for (int64_t j = 0; j < x->f; ++j) out[j] += beta * w[j];
  }
};

// ---------------------------------------------------------------- power iteration
// krylov.cpp:62-92
double lambda_max(const Op& a, double tol, uint64_t max_iters, uint64_t seed, uint64_t* iters,
                  bool* conv) {
  const int64_t n = a.dim();
  Rng rng(seed);
  Vec v(n), w(n, 0.0);
  for (auto& e : v) e = rng.normal();
  double nv = nrm(v.data(), n);
  if (nv == 0.0) nv = 1.0;
  for (auto& e : v) e /= nv;
  double prev = 0.0, lam = 0.0;
  *conv = false;
  *iters = 0;
  for (uint64_t it = 0; it < max_iters; ++it) {
    a.apply(v.data(), w.data());
    lam = nrm(w.data(), n);
    *iters = it + 1;
    if (lam == 0.0) {
      *conv = true;
      return lam;
    }
    for (int64_t i = 0; i < n; ++i) v[i] = w[i] / lam;
    if (it > 0 && std::abs(lam - prev) <= tol * lam) {
      *conv = true;
      return lam;
    }
    prev = lam;
  }
  return lam;
}

// ---------------------------------------------------------------- reports
struct Report {
  uint64_t iterations = 0;
  bool converged = false;
  double wall = 0.0;
  Vec hist;
  std::vector<uint64_t> inner;
};

using Clock = std::chrono::steady_clock;
double since(Clock::time_point t) { return std::chrono::duration<double>(Clock::now() - t).count(); }

void check_rhs(const Vec& rhs, int64_t n, const char* who) {  // krylov.cpp:23-31
  if (static_cast<int64_t>(rhs.size()) != n)
    throw std::invalid_argument(std::string(who) + ": rhs length != operator dimension");
  for (double v : rhs)
    if (!std::isfinite(v)) throw std::invalid_argument(std::string(who) + ": non-finite rhs");
}

// ---------------------------------------------------------------- CG
// krylov.cpp:94-157 (inv_diag != nullptr: Jacobi, krylov.cpp:41-51)
Vec cg(const Op& a, const Vec& rhs, double tol, uint64_t max_iters, const Vec* inv_diag, Report& rep) {
  check_rhs(rhs, a.dim(), "cg");
  const auto t0 = Clock::now();
  const int64_t n = a.dim();
  Vec x(n, 0.0);
  const double nb = nrm(rhs.data(), n);
  if (nb == 0.0) {
    rep.converged = true;
    rep.hist.push_back(0.0);
    rep.wall = since(t0);
    return x;
  }
  Vec r = rhs, z(n), p, ap(n, 0.0);
  auto precond = [&] {
    if (inv_diag)
      for (int64_t i = 0; i < n; ++i) z[i] = (*inv_diag)[i] * r[i];
    else
      z = r;
  };
  precond();
  p = z;
  double rz = dotp(r.data(), z.data(), n);
  for (uint64_t it = 0; it < max_iters; ++it) {
    a.apply(p.data(), ap.data());
    const double pap = dotp(p.data(), ap.data(), n);
    if (!(pap > 0.0))
      throw std::runtime_error("cg: <p, Ap> = " + std::to_string(pap) + " at iteration " +
                               std::to_string(it) + "; operator is not positive definite");
    const double alpha = rz / pap;
    for (int64_t i = 0; i < n; ++i) {
      x[i] += alpha * p[i];
      r[i] -= alpha * ap[i];
    }
    const double rel = nrm(r.data(), n) / nb;
    rep.hist.push_back(rel);
    rep.iterations = it + 1;
    if (rel <= tol) {
      rep.converged = true;
      break;
    }
    precond();
    const double rz2 = dotp(r.data(), z.data(), n);
    const double bcoef = rz2 / rz;
    rz = rz2;
    for (int64_t i = 0; i < n; ++i) p[i] = z[i] + bcoef * p[i];
  }
  rep.wall = since(t0);
  return x;
}

// ---------------------------------------------------------------- preconditioners
struct Precond {
  virtual ~Precond() = default;
  virtual uint64_t apply(const double* r, double* z) const = 0;
};

struct Level;  // one coarse level of the hierarchy

Vec fcg(const Op& a, const Vec& rhs, double tol, uint64_t max_iters, uint64_t truncation,
        const Precond& m, Report& rep);

// Dense SPD factor, lower triangle, row-major.
struct Chol {
  int64_t n = 0;
  Vec l;
  void factor(const Vec& a, int64_t dim) {
    n = dim;
    l.assign(n * n, 0.0);
    for (int64_t j = 0; j < n; ++j) {
      double d = a[j * n + j];
      for (int64_t k = 0; k < j; ++k) d -= l[j * n + k] * l[j * n + k];
      if (!(d > 0.0) || !std::isfinite(d))
        throw std::runtime_error(
            "coarse Cholesky factorization failed; the Galerkin operator is numerically "
            "indefinite - consider a larger beta or a smaller coarse level");
      const double ljj = std::sqrt(d);
      l[j * n + j] = ljj;
      for (int64_t i = j + 1; i < n; ++i) {
        double s = a[i * n + j];
        for (int64_t k = 0; k < j; ++k) s -= l[i * n + k] * l[j * n + k];
        l[i * n + j] = s / ljj;
      }
    }
  }
  Vec inv;  // ORC_COARSE_INV: explicit inverse (columns by the triangular solves below)
  void make_inverse() {
    inv.assign(n * n, 0.0);
    Vec e(n), col(n);
    for (int64_t j = 0; j < n; ++j) {
      std::fill(e.begin(), e.end(), 0.0);
      e[j] = 1.0;
      solve_tri(e.data(), col.data());
      for (int64_t i = 0; i < n; ++i) inv[i * n + j] = col[i];
    }
  }
  void solve(const double* b, double* x) const {
    if (!inv.empty()) {
      for (int64_t i = 0; i < n; ++i) {
        double s = 0.0;
        for (int64_t j = 0; j < n; ++j) s += inv[i * n + j] * b[j];
        x[i] = s;
      }
      return;
    }
    solve_tri(b, x);
  }
  void solve_tri(const double* b, double* x) const {
    Vec y(n);
    for (int64_t i = 0; i < n; ++i) {
      double s = b[i];
      for (int64_t k = 0; k < i; ++k) s -= l[i * n + k] * y[k];
      y[i] = s / l[i * n + i];
    }
    for (int64_t i = n; i-- > 0;) {
      double s = y[i];
      for (int64_t k = i + 1; k < n; ++k) s -= l[k * n + i] * x[k];
      x[i] = s / l[i * n + i];
    }
  }
};

// Adjusted-average aggregation P (coarsening.cpp:82-100): one weight
// 1/sqrt(n_S) per fine feature.
struct Agg {
  int64_t nf = 0, nc = 0;
  std::vector<int64_t> label;
  Vec weight;
  // coarsening.cpp:43-55: zero-fill, scatter, skip zero fine entries
  void restrict_(const double* fine, double* coarse) const {
    std::fill(coarse, coarse + nc, 0.0);
    for (int64_t i = 0; i < nf; ++i) {
      const double fi = fine[i];
      if (fi == 0.0) continue;
      coarse[label[i]] += weight[i] * fi;
    }
  }
  // coarsening.cpp:30-41: acc starts at 0.0
  void prolong(const double* coarse, double* fine) const {
    for (int64_t i = 0; i < nf; ++i) {
      double acc = 0.0;
      acc += weight[i] * coarse[label[i]];
      fine[i] = acc;
    }
  }
};

Agg make_agg(const std::vector<int64_t>& labels, int64_t nc) {
  // clustering.cpp:13-41 validation subset + coarsening.cpp:82-100
  Agg p;
  p.nf = static_cast<int64_t>(labels.size());
  p.nc = nc;
  p.label = labels;
  std::vector<int64_t> size(nc, 0);
  for (int64_t s : labels) {
    if (s < 0 || s >= nc) throw std::invalid_argument("ClusterAssignment: cluster id out of range");
    size[s]++;
  }
  for (int64_t s = 0; s < nc; ++s)
    if (size[s] == 0) throw std::invalid_argument("ClusterAssignment: empty cluster " + std::to_string(s));
  p.weight.resize(p.nf);
  for (int64_t i = 0; i < p.nf; ++i) p.weight[i] = 1.0 / std::sqrt(static_cast<double>(size[labels[i]]));
  return p;
}

// coarsening.cpp:112-148: X_c = X P row by row; per coarse column the value is
// the sequential sum over the row's fine nonzeros in column order; coarse
// columns sorted; exact zeros from cancellation kept.
Csr coarsen(const Csr& x, const Agg& p) {
  if (p.nf != x.f) throw std::invalid_argument("coarsen: prolongation / matrix feature mismatch");
  Csr c;
  c.n = x.n;
  c.f = p.nc;
  c.ptr.assign(x.n + 1, 0);
  Vec acc(p.nc, 0.0);
  std::vector<int64_t> seen(p.nc, -1), touched;
  for (int64_t r = 0; r < x.n; ++r) {
    touched.clear();
    for (int64_t k = x.ptr[r]; k < x.ptr[r + 1]; ++k) {
      const int64_t i = x.idx[k];
      const int64_t s = p.label[i];
      if (seen[s] != r) {
        seen[s] = r;
        touched.push_back(s);
      }
      acc[s] += x.val[k] * p.weight[i];
    }
    std::sort(touched.begin(), touched.end());
    for (int64_t s : touched) {
      c.idx.push_back(s);
      c.val.push_back(acc[s]);
      acc[s] = 0.0;
    }
    c.ptr[r + 1] = static_cast<int64_t>(c.val.size());
  }
  return c;
}

struct Level {
  Csr xc;
  Agg p;
  double beta = 0.0;
  Op op;  // GalerkinOperator (coarsening.cpp:174-194), adjusted-average branch
};

// krylov.cpp:334-420
struct TwoLevel final : Precond {
  const Op* fine = nullptr;
  const Level* coarse = nullptr;
  double omega = 0.0;
  int kind = OR_COARSE_DIRECT;
  double tol = 1e-6;
  uint64_t max_iters = 500, truncation = 20;
  const Precond* nested = nullptr;
  Chol chol;

  void setup() {
    if (!(omega > 0.0)) throw std::invalid_argument("TwoLevelPreconditioner: omega must be positive");
    if (coarse->p.nf != fine->dim())
      throw std::invalid_argument("TwoLevelPreconditioner: prolongation does not match fine level");
    if (kind != OR_COARSE_DIRECT) return;
    // krylov.cpp:350-365: dense A_c = sum over rows of outer products, + beta on the diagonal
    const Csr& xc = coarse->xc;
    const int64_t fc = xc.f;
    Vec ac(fc * fc, 0.0);
    for (int64_t r = 0; r < xc.n; ++r)
      for (int64_t a = xc.ptr[r]; a < xc.ptr[r + 1]; ++a)
        for (int64_t b = xc.ptr[r]; b < xc.ptr[r + 1]; ++b)
          ac[xc.idx[a] * fc + xc.idx[b]] += xc.val[a] * xc.val[b];
    for (int64_t i = 0; i < fc; ++i) ac[i * fc + i] += coarse->beta;
    chol.factor(ac, fc);
    if (env_int("ORC_COARSE_INV") != 0) chol.make_inverse();
  }

  uint64_t apply(const double* r, double* z) const override {
    const int64_t nf = fine->dim(), nc = coarse->p.nc;
    Vec rc(nc, 0.0), ec(nc, 0.0);
    coarse->p.restrict_(r, rc.data());
    uint64_t inner = 0;
    if (kind == OR_COARSE_DIRECT) {
      chol.solve(rc.data(), ec.data());
    } else {
      Report sub;
      if (kind == OR_COARSE_INNER_FCG) {
        if (!nested) throw std::runtime_error("TwoLevelPreconditioner: flexible coarse solve needs a nested preconditioner");
        ec = fcg(coarse->op, rc, tol, max_iters, truncation, *nested, sub);
      } else {
        ec = cg(coarse->op, rc, tol, max_iters, nullptr, sub);
      }
      inner = sub.iterations;
    }
    Vec z1(nf, 0.0), az1(nf, 0.0);
    coarse->p.prolong(ec.data(), z1.data());
    fine->apply(z1.data(), az1.data());
    for (int64_t i = 0; i < nf; ++i) z[i] = z1[i] + omega * (r[i] - az1[i]);
    return inner;
  }
};

// ---------------------------------------------------------------- FCG
// krylov.cpp:159-227 — truncation m_0 = 0, m_i = max(1, i mod (m+1)); classical
// Gram-Schmidt of z against the newest min(m_i, |history|) stored directions.
Vec fcg(const Op& a, const Vec& rhs, double tol, uint64_t max_iters, uint64_t truncation,
        const Precond& m, Report& rep) {
  check_rhs(rhs, a.dim(), "fcg");
  const auto t0 = Clock::now();
  const int64_t n = a.dim();
  const uint64_t keep = std::max<uint64_t>(truncation, 1);
  Vec x(n, 0.0);
  const double nb = nrm(rhs.data(), n);
  if (nb == 0.0) {
    rep.converged = true;
    rep.hist.push_back(0.0);
    rep.wall = since(t0);
    return x;
  }
  // history as a ring of `keep` slots; `head` = oldest, `count` = live entries
  std::vector<Vec> hp(keep), hap(keep);
  Vec hpap(keep, 0.0);
  uint64_t head = 0, count = 0;
  Vec r = rhs, z(n), p(n), ap(n);
  for (uint64_t it = 0; it < max_iters; ++it) {
    rep.inner.push_back(m.apply(r.data(), z.data()));
    const uint64_t mi = it == 0 ? 0 : std::max<uint64_t>(1, it % (keep + 1));
    p = z;
    const uint64_t use = std::min(mi, count);
    for (uint64_t q = count - use; q < count; ++q) {  // oldest -> newest of the last `use`
      const uint64_t slot = (head + q) % keep;
      const double c = dotp(z.data(), hap[slot].data(), n) / hpap[slot];
      const double* ph = hp[slot].data();
      for (int64_t i = 0; i < n; ++i) p[i] -= c * ph[i];
    }
    a.apply(p.data(), ap.data());
    const double pap = dotp(p.data(), ap.data(), n);
    if (pap == 0.0) throw std::runtime_error("fcg: breakdown, <p, Ap> = 0 at iteration " + std::to_string(it));
    if (pap < 0.0)
      throw std::runtime_error("fcg: <p, Ap> < 0 at iteration " + std::to_string(it) +
                               "; operator is not positive definite");
    const double alpha = dotp(p.data(), r.data(), n) / pap;
    for (int64_t i = 0; i < n; ++i) {
      x[i] += alpha * p[i];
      r[i] -= alpha * ap[i];
    }
    uint64_t slot;
    if (count < keep) {
      slot = (head + count) % keep;
      ++count;
    } else {  // deque push_back + pop_front
      slot = head;
      head = (head + 1) % keep;
    }
    hp[slot] = p;
    hap[slot] = ap;
    hpap[slot] = pap;
    const double rel = nrm(r.data(), n) / nb;
    rep.hist.push_back(rel);
    rep.iterations = it + 1;
    if (rel <= tol) {
      rep.converged = true;
      break;
    }
  }
  rep.wall = since(t0);
  return x;
}

// ---------------------------------------------------------------- FGMRES
// krylov.cpp:229-328 — full (unrestarted) flexible GMRES, right-preconditioned:
// modified Gram-Schmidt of w = A z_j against v_0..v_j, Givens rotations on the
// Hessenberg column, residual estimate |g_{j+1}| / ||rhs||, back substitution,
// x = sum_j y_j z_j.
Vec fgmres(const Op& a, const Vec& rhs, double tol, uint64_t max_iters, const Precond& m, Report& rep) {
  check_rhs(rhs, a.dim(), "fgmres");
  const auto t0 = Clock::now();
  const int64_t n = a.dim();
  Vec x(n, 0.0);
  const double nrhs = nrm(rhs.data(), n);
  if (nrhs == 0.0) {
    rep.converged = true;
    rep.hist.push_back(0.0);
    rep.wall = since(t0);
    return x;
  }
  std::vector<Vec> basis, pre, hess;
  Vec gc, gs, g;
  basis.push_back(rhs);
  for (double& v : basis[0]) v /= nrhs;
  g.push_back(nrhs);
  Vec z(n), w(n);
  uint64_t k = 0;
  for (uint64_t j = 0; j < max_iters; ++j) {
    rep.inner.push_back(m.apply(basis[j].data(), z.data()));
    pre.push_back(z);
    a.apply(z.data(), w.data());
    Vec h(j + 2, 0.0);
    for (uint64_t i = 0; i <= j; ++i) {
      h[i] = dotp(w.data(), basis[i].data(), n);
      for (int64_t t = 0; t < n; ++t) w[t] -= h[i] * basis[i][t];
    }
    const double h_next = nrm(w.data(), n);
    h[j + 1] = h_next;
    for (uint64_t i = 0; i < j; ++i) {
      const double tmp = gc[i] * h[i] + gs[i] * h[i + 1];
      h[i + 1] = -gs[i] * h[i] + gc[i] * h[i + 1];
      h[i] = tmp;
    }
    const double denom = std::hypot(h[j], h[j + 1]);
    const double c = denom == 0.0 ? 1.0 : h[j] / denom;
    const double sn = denom == 0.0 ? 0.0 : h[j + 1] / denom;
    gc.push_back(c);
    gs.push_back(sn);
    h[j] = denom;
    h[j + 1] = 0.0;
    g.push_back(-sn * g[j]);
    g[j] = c * g[j];
    hess.push_back(std::move(h));
    k = j + 1;
    const double rel = std::abs(g[j + 1]) / nrhs;
    rep.hist.push_back(rel);
    rep.iterations = k;
    if (rel <= tol || h_next == 0.0) {
      rep.converged = true;
      break;
    }
    basis.emplace_back(n);
    for (int64_t t = 0; t < n; ++t) basis[j + 1][t] = w[t] / h_next;
  }
  Vec y(k, 0.0);
  for (uint64_t i = k; i-- > 0;) {
    double acc = g[i];
    for (uint64_t jj = i + 1; jj < k; ++jj) acc -= hess[jj][i] * y[jj];
    if (hess[i][i] == 0.0)
      throw std::runtime_error("fgmres: rank-deficient Hessenberg system at column " + std::to_string(i));
    y[i] = acc / hess[i][i];
  }
  for (uint64_t jj = 0; jj < k; ++jj)
    for (int64_t t = 0; t < n; ++t) x[t] += y[jj] * pre[jj][t];
  rep.wall = since(t0);
  return x;
}

// ---------------------------------------------------------------- clustering
using Labels = std::vector<int64_t>;

// distance.cpp:27-67: euclidean over the merged supports in increasing row order
double col_dist(const Csc& c, int64_t i, int64_t j) {
  int64_t a = c.ptr[i], ae = c.ptr[i + 1], b = c.ptr[j], be = c.ptr[j + 1];
  double s = 0.0;
  while (a < ae && b < be) {
    double d;
    if (c.row[a] == c.row[b]) {
      d = c.val[a++] - c.val[b++];
    } else if (c.row[a] < c.row[b]) {
      d = c.val[a++] - 0.0;
    } else {
      d = 0.0 - c.val[b++];
    }
    s += d * d;
  }
  for (; a < ae; ++a) {
    const double d = c.val[a] - 0.0;
    s += d * d;
  }
  for (; b < be; ++b) {
    const double d = 0.0 - c.val[b];
    s += d * d;
  }
  return std::sqrt(s);
}

template <class F>
void parallel_for(int64_t n, unsigned threads, F&& body) {
  if (threads <= 1 || n < 256) {
    body(int64_t{0}, n);
    return;
  }
  std::vector<std::thread> ws;
  const int64_t chunk = (n + threads - 1) / threads;
  for (unsigned t = 0; t < threads; ++t) {
    const int64_t lo = std::min<int64_t>(n, t * chunk), hi = std::min<int64_t>(n, lo + chunk);
    if (lo >= hi) break;
    ws.emplace_back([&, lo, hi] { body(lo, hi); });
  }
  for (auto& w : ws) w.join();
}

unsigned g_threads = 1;

// clustering.cpp:189-255
std::vector<int64_t> kpp_seed(const Csc& c, int64_t k, uint64_t seed) {
  const int64_t f = c.f;
  if (k <= 0 || k > f) throw std::invalid_argument("kmeanspp_seed: k outside [1, F]");
  Rng rng(seed);
  std::vector<int64_t> chosen;
  std::vector<char> taken(f, 0);
  const auto first = static_cast<int64_t>(rng.index(f));
  chosen.push_back(first);
  taken[first] = 1;
  Vec best(f, std::numeric_limits<double>::infinity()), dist(f, 0.0);
  while (static_cast<int64_t>(chosen.size()) < k) {
    const int64_t last = chosen.back();
    parallel_for(f, g_threads, [&](int64_t lo, int64_t hi) {
      for (int64_t j = lo; j < hi; ++j)
        if (!taken[j]) dist[j] = col_dist(c, j, last);
    });
    double total = 0.0;
    for (int64_t j = 0; j < f; ++j) {
      if (taken[j]) {
        best[j] = 0.0;
        continue;
      }
      best[j] = std::min(best[j], dist[j] * dist[j]);
      total += best[j];
    }
    int64_t pick = f;
    if (total > 0.0) {
      const double u = rng.unit() * total;
      double acc = 0.0;
      for (int64_t j = 0; j < f; ++j) {
        if (taken[j] || best[j] == 0.0) continue;
        acc += best[j];
        if (u < acc) {
          pick = j;
          break;
        }
      }
      if (pick == f)
        for (int64_t j = f; j-- > 0;)
          if (!taken[j] && best[j] > 0.0) {
            pick = j;
            break;
          }
    }
    if (pick == f) {
      uint64_t idx = rng.index(static_cast<uint64_t>(f) - chosen.size());
      for (int64_t j = 0; j < f; ++j) {
        if (taken[j]) continue;
        if (idx-- == 0) {
          pick = j;
          break;
        }
      }
    }
    chosen.push_back(pick);
    taken[pick] = 1;
  }
  return chosen;
}

// clustering.cpp:257-355 with prototypes transposed: pt[r * k + s] = proto_s[r].
// Distances follow column_dense_sqdist (distance.cpp:93-105):
//   ||p||^2 + sum_{i in supp x, increasing} ((x_i - p_i)^2 - p_i^2), clamped at 0.
Labels kmeans(const Csc& c, int64_t k, uint64_t max_iters, uint64_t seed, uint64_t* iters_out,
              bool* conv_out) {
  const int64_t f = c.f, n = c.n;
  if (k <= 0 || k > f) throw std::invalid_argument("kmeans: k outside [1, F]");
  Vec pt(static_cast<size_t>(n) * k, 0.0);
  auto densify_into = [&](int64_t j, int64_t s) {
    for (int64_t r = 0; r < n; ++r) pt[r * k + s] = 0.0;
    for (int64_t t = c.ptr[j]; t < c.ptr[j + 1]; ++t) pt[c.row[t] * k + s] = c.val[t];
  };
  const auto seeds = kpp_seed(c, k, seed);
  for (int64_t s = 0; s < k; ++s) densify_into(seeds[s], s);

  Labels member(f, 0), prev;
  std::vector<int64_t> sizes(k, 0);
  Vec psq(k, 0.0), own(f, 0.0);
  *conv_out = false;
  *iters_out = 0;
  const uint64_t rounds = std::max<uint64_t>(max_iters, 1);
  for (uint64_t iter = 0; iter < rounds; ++iter) {
    std::fill(psq.begin(), psq.end(), 0.0);
    for (int64_t r = 0; r < n; ++r) {  // each psq[s] accumulates over r = 0..N-1 in order
      const double* row = &pt[r * k];
      for (int64_t s = 0; s < k; ++s) psq[s] += row[s] * row[s];
    }
    parallel_for(f, g_threads, [&](int64_t lo, int64_t hi) {
      Vec d(k);
      for (int64_t j = lo; j < hi; ++j) {
        std::copy(psq.begin(), psq.end(), d.begin());
        for (int64_t t = c.ptr[j]; t < c.ptr[j + 1]; ++t) {
          const double xv = c.val[t];
          const double* row = &pt[c.row[t] * k];
          for (int64_t s = 0; s < k; ++s) {
            const double pi = row[s];
            const double diff = xv - pi;
            d[s] += diff * diff - pi * pi;
          }
        }
        int64_t b = 0;
        double bsq = std::numeric_limits<double>::infinity();
        for (int64_t s = 0; s < k; ++s) {
          const double sq = std::max(d[s], 0.0);
          if (sq < bsq) {
            bsq = sq;
            b = s;
          }
        }
        member[j] = b;
        own[j] = bsq;
      }
    });
    std::fill(sizes.begin(), sizes.end(), 0);
    for (int64_t j = 0; j < f; ++j) sizes[member[j]]++;
    // empty-cluster repair (clustering.cpp:303-321)
    for (int64_t s = 0; s < k; ++s) {
      if (sizes[s] != 0) continue;
      int64_t far = f;
      double far_sq = -1.0;
      for (int64_t j = 0; j < f; ++j) {
        if (sizes[member[j]] <= 1) continue;
        if (own[j] > far_sq) {
          far_sq = own[j];
          far = j;
        }
      }
      if (far == f) break;
      sizes[member[far]]--;
      member[far] = s;
      sizes[s] = 1;
      densify_into(far, s);
      own[far] = 0.0;
    }
    *iters_out = iter + 1;
    if (!prev.empty() && prev == member) {
      *conv_out = true;
      break;
    }
    prev = member;
    // means: features in index order, then x (1/size) (clustering.cpp:331-344)
    std::fill(pt.begin(), pt.end(), 0.0);
    for (int64_t j = 0; j < f; ++j) {
      const int64_t s = member[j];
      for (int64_t t = c.ptr[j]; t < c.ptr[j + 1]; ++t) pt[c.row[t] * k + s] += c.val[t];
    }
    Vec inv(k);
    for (int64_t s = 0; s < k; ++s) inv[s] = 1.0 / static_cast<double>(sizes[s]);
    for (int64_t r = 0; r < n; ++r)
      for (int64_t s = 0; s < k; ++s) pt[r * k + s] *= inv[s];
  }
  return member;
}

// clustering.cpp:64-130, fixed leaders
Labels leader_follower(const Csc& c, double tol, int64_t* n_clusters) {
  if (!(tol > 0.0)) throw std::invalid_argument("leader_follower: tolerance must be positive");
  if (c.f == 0) throw std::invalid_argument("leader_follower: empty matrix");
  Labels member(c.f, 0);
  std::vector<int64_t> leaders;
  for (int64_t i = 0; i < c.f; ++i) {
    int64_t best = -1;
    double bd = std::numeric_limits<double>::infinity();
    for (size_t s = 0; s < leaders.size(); ++s) {
      const double d = col_dist(c, i, leaders[s]);
      if (d < bd) {
        bd = d;
        best = static_cast<int64_t>(s);
      }
    }
    if (best >= 0 && bd < tol) {
      member[i] = best;
    } else {
      member[i] = static_cast<int64_t>(leaders.size());
      leaders.push_back(i);
    }
  }
  *n_clusters = static_cast<int64_t>(leaders.size());
  return member;
}

// clustering.cpp:132-187
Labels leader_follower_target(const Csc& c, int64_t target, int64_t* nc_out, bool* exact, double* tol_out) {
  if (target <= 0 || target > c.f) throw std::invalid_argument("leader_follower_target: target outside [1, F]");
  struct Run {
    Labels l;
    int64_t n = 0;
  };
  auto run = [&](double t) {
    Run r;
    r.l = leader_follower(c, t, &r.n);
    return r;
  };
  double lo = 1e-12, hi = 1.0;
  Run at_lo = run(lo), at_hi = run(hi);
  size_t grow = 0;
  while (at_hi.n > target && grow++ < 64) {
    hi *= 2.0;
    at_hi = run(hi);
  }
  Run best = at_lo;
  double best_tol = lo;
  auto gap = [&](const Run& r) { return std::llabs(r.n - target); };
  auto consider = [&](const Run& r, double t) {
    if (gap(r) < gap(best) || (gap(r) == gap(best) && r.n > best.n)) {
      best = r;
      best_tol = t;
    }
  };
  consider(at_hi, hi);
  for (size_t probe = 0; probe < 200 && best.n != target; ++probe) {
    const double mid = 0.5 * (lo + hi);
    if (mid <= lo || mid >= hi) break;
    Run at_mid = run(mid);
    consider(at_mid, mid);
    if (at_mid.n > target)
      lo = mid;
    else
      hi = mid;
  }
  *nc_out = best.n;
  *exact = best.n == target;
  *tol_out = best_tol;
  return best.l;
}

Csr normalized(const Csr& x) {  // BASELINE cfg 2 extension, norms accumulated in row order
  Vec sq(x.f, 0.0);
  for (int64_t k = 0; k < x.nnz(); ++k) sq[x.idx[k]] += x.val[k] * x.val[k];
  for (auto& v : sq) v = std::sqrt(v);
  Csr y = x;
  for (int64_t k = 0; k < y.nnz(); ++k) y.val[k] /= sq[y.idx[k]];
  return y;
}

Labels cluster(const Csr& cur, const or_level_spec& s, int64_t* nc) {
  if (s.labels) {
    Labels l(s.labels, s.labels + cur.f);
    *nc = static_cast<int64_t>(s.n_clusters);
    return l;
  }
  const Csc c = transpose_of(s.normalize_columns ? normalized(cur) : cur);
  switch (s.clustering_kind) {
    case OR_CLUSTER_LEADER_TOLERANCE:
      return leader_follower(c, s.tolerance, nc);
    case OR_CLUSTER_LEADER_TARGET: {
      bool ex;
      double t;
      return leader_follower_target(c, static_cast<int64_t>(s.target_size), nc, &ex, &t);
    }
    case OR_CLUSTER_KMEANS: {
      uint64_t it;
      bool cv;
      *nc = static_cast<int64_t>(s.target_size);
      return kmeans(c, *nc, s.kmeans_max_iters, s.seed, &it, &cv);
    }
  }
  throw std::invalid_argument("unknown clustering kind");
}

// ---------------------------------------------------------------- hierarchy
// krylov.cpp:493-568
struct Hierarchy {
  const Csr* fine = nullptr;
  Op fine_op;
  std::vector<std::unique_ptr<Level>> lv;
  std::vector<std::unique_ptr<TwoLevel>> pc;
  Vec omega;
  const Csr& mat(size_t k) const { return k == 0 ? *fine : lv[k - 1]->xc; }
  const Op& op(size_t k) const { return k == 0 ? fine_op : lv[k - 1]->op; }
};

std::unique_ptr<Hierarchy> build(const Csr& x, double beta, const or_level_spec* sp, size_t n) {
  if (n == 0) throw std::invalid_argument("build_hierarchy: at least one level spec is required");
  for (size_t k = 0; k + 1 < n; ++k)
    if (sp[k].coarse_kind == OR_COARSE_DIRECT)
      throw std::invalid_argument("build_hierarchy: only the last level may use direct_cholesky");
  if (sp[n - 1].coarse_kind != OR_COARSE_DIRECT)
    throw std::invalid_argument("build_hierarchy: the coarsest level must use direct_cholesky");
  if (beta < 0.0) throw std::invalid_argument("RidgeOperator: beta must be nonnegative");
  auto h = std::make_unique<Hierarchy>();
  h->fine = &x;
  h->fine_op.x = &x;
  h->fine_op.beta = beta;
  double lb = beta;
  for (size_t k = 0; k < n; ++k) {
    const Csr& cur = h->mat(k);
    const double nb = sp[k].has_beta_override ? sp[k].beta_override : lb;
    int64_t nc = 0;
    const Labels l = cluster(cur, sp[k], &nc);
    if (nc >= cur.f) throw std::invalid_argument("build_hierarchy: level has no fewer clusters than features");
    auto L = std::make_unique<Level>();
    L->p = make_agg(l, nc);
    L->xc = coarsen(cur, L->p);
    L->beta = nb;
    h->lv.push_back(std::move(L));
    h->lv.back()->op.x = &h->lv.back()->xc;
    h->lv.back()->op.beta = nb;
    lb = nb;
  }
  if (h->lv.back()->xc.f > 4096) throw std::invalid_argument("build_hierarchy: coarsest level above the direct-solve cap");
  for (size_t k = 0; k < n; ++k) {
    Op gram;
    gram.x = &h->mat(k);
    gram.add_beta = false;
    uint64_t it;
    bool cv;
    const double lmax = lambda_max(gram, 1e-4, 200, 0x5eed + k, &it, &cv);
    const double b = k == 0 ? beta : h->lv[k - 1]->beta;
    double om = 2.0 / (b + lmax);
    for (int u = env_int("ORC_OMEGA_ULP"), i = 0; i < std::abs(u); ++i)
      om = std::nextafter(om, u > 0 ? 2.0 * om : 0.0);
    h->omega.push_back(om);
  }
  h->pc.resize(n);
  for (size_t k = n; k-- > 0;) {
    auto t = std::make_unique<TwoLevel>();
    t->fine = &h->op(k);
    t->coarse = h->lv[k].get();
    t->omega = h->omega[k];
    t->kind = sp[k].coarse_kind;
    t->tol = sp[k].coarse_tol;
    t->max_iters = sp[k].coarse_max_iters;
    t->truncation = sp[k].coarse_truncation;
    t->nested = t->kind == OR_COARSE_INNER_FCG ? h->pc[k + 1].get() : nullptr;
    t->setup();
    h->pc[k] = std::move(t);
  }
  return h;
}

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

Csr* H(void* h) { return static_cast<Csr*>(h); }

void fill(const Report& r, or_solve_report* o) {
  if (!o) return;
  o->iterations = r.iterations;
  o->converged = r.converged ? 1 : 0;
  o->wall_time_s = r.wall;
  if (o->residual_history)
    std::memcpy(o->residual_history, r.hist.data(), std::min<size_t>(o->residual_capacity, r.hist.size()) * sizeof(double));
  if (o->inner_iterations)
    for (size_t i = 0; i < std::min<size_t>(o->inner_capacity, r.inner.size()); ++i) o->inner_iterations[i] = r.inner[i];
}

}  // namespace

extern "C" {

const char* orc_last_error() { return g_err.c_str(); }
int orc_set_num_threads(unsigned t) {
  g_threads = t == 0 ? 1 : t;
  return 0;
}

void* orc_matrix_from_csr(uint64_t n, uint64_t f, uint64_t nnz, const uint64_t* rp, const uint64_t* ci,
                          const double* v) {
  auto* m = new Csr;
  m->n = static_cast<int64_t>(n);
  m->f = static_cast<int64_t>(f);
  m->ptr.assign(rp, rp + n + 1);
  m->idx.assign(ci, ci + nnz);
  if (v)
    m->val.assign(v, v + nnz);
  else
    m->val.assign(nnz, 1.0);
  return m;
}
// BASELINE synthetic inputs (oracle/synth.hpp) as a checker matrix
void* orc_synth_sparse_zipf(uint64_t n, uint64_t f, double mean, double s, int32_t values, uint64_t seed,
                            int32_t row_streams) {
  auto g = oracle_synth::sparse_zipf<Rng>(static_cast<int64_t>(n), static_cast<int64_t>(f), mean, s, values != 0,
                                          seed, row_streams != 0);
  return orc_matrix_from_csr(n, f, g.idx.size(), g.ptr.data(), g.idx.data(), values ? g.val.data() : nullptr);
}
void* orc_synth_dense_clustered(uint64_t n, uint64_t f, uint64_t groups, double noise, uint64_t seed) {
  auto g = oracle_synth::dense_clustered<Rng>(static_cast<int64_t>(n), static_cast<int64_t>(f),
                                              static_cast<int64_t>(groups), noise, seed);
  return orc_matrix_from_csr(n, f, g.idx.size(), g.ptr.data(), g.idx.data(), g.val.data());
}
void orc_matrix_free(void* h) { delete H(h); }
int orc_matrix_shape(void* h, uint64_t* n, uint64_t* f, uint64_t* nnz) {
  *n = H(h)->n;
  *f = H(h)->f;
  *nnz = H(h)->nnz();
  return 0;
}
int orc_matrix_export(void* h, uint64_t* rp, uint64_t* ci, double* v) {
  const Csr& m = *H(h);
  for (int64_t i = 0; i <= m.n; ++i) rp[i] = m.ptr[i];
  for (int64_t k = 0; k < m.nnz(); ++k) {
    ci[k] = m.idx[k];
    v[k] = m.val[k];
  }
  return 0;
}

int orc_spmv(void* h, const double* v, double* y) {
  mul(*H(h), v, y);
  return 0;
}
int orc_spmv_transpose(void* h, const double* u, double* y) {
  mul_t(*H(h), u, y);
  return 0;
}
int orc_ridge_apply(void* h, double beta, const double* w, double* out) {
  return guard([&] {
    if (beta < 0.0) throw std::invalid_argument("RidgeOperator: beta must be nonnegative");
    Op op;
    op.x = H(h);
    op.beta = beta;
    op.apply(w, out);
  });
}
// ridge.cpp:30-37: d starts at beta, += v*v in storage order
int orc_gram_diagonal(void* h, double beta, double* out) {
  const Csr& m = *H(h);
  std::fill(out, out + m.f, beta);
  for (int64_t k = 0; k < m.nnz(); ++k) out[m.idx[k]] += m.val[k] * m.val[k];
  return 0;
}
int orc_lambda_max(void* h, double tol, uint64_t max_iters, uint64_t seed, double* value, uint64_t* iters,
                   int32_t* converged) {
  Op g;
  g.x = H(h);
  g.add_beta = false;
  bool cv;
  *value = lambda_max(g, tol, max_iters, seed, iters, &cv);
  *converged = cv ? 1 : 0;
  return 0;
}
int orc_normals(uint64_t seed, uint64_t n, double* out) {
  Rng r(seed);
  for (uint64_t i = 0; i < n; ++i) out[i] = r.normal();
  return 0;
}
// analysis.cpp:225-232
int orc_generate_rhs(void* h, uint64_t seed, double* b, double* rhs) {
  Rng r(seed);
  const Csr& m = *H(h);
  for (int64_t i = 0; i < m.n; ++i) b[i] = r.normal();
  if (rhs) mul_t(m, b, rhs);
  return 0;
}
int orc_kmeanspp_seed(void* h, uint64_t k, uint64_t seed, int64_t* chosen) {
  return guard([&] {
    const auto c = kpp_seed(transpose_of(*H(h)), static_cast<int64_t>(k), seed);
    std::copy(c.begin(), c.end(), chosen);
  });
}
int orc_kmeans(void* h, uint64_t k, uint64_t max_iters, uint64_t seed, int32_t normalize, int64_t* labels,
               uint64_t* iters, int32_t* converged) {
  return guard([&] {
    bool cv;
    const Labels l = kmeans(transpose_of(normalize ? normalized(*H(h)) : *H(h)), static_cast<int64_t>(k),
                            max_iters, seed, iters, &cv);
    std::copy(l.begin(), l.end(), labels);
    *converged = cv ? 1 : 0;
  });
}
int orc_leader_follower(void* h, double tol, int64_t* labels, uint64_t* n_clusters) {
  return guard([&] {
    int64_t nc;
    const Labels l = leader_follower(transpose_of(*H(h)), tol, &nc);
    std::copy(l.begin(), l.end(), labels);
    *n_clusters = static_cast<uint64_t>(nc);
  });
}
int orc_leader_follower_target(void* h, uint64_t target, int64_t* labels, uint64_t* n_clusters, int32_t* exact,
                               double* tol) {
  return guard([&] {
    int64_t nc;
    bool ex;
    const Labels l = leader_follower_target(transpose_of(*H(h)), static_cast<int64_t>(target), &nc, &ex, tol);
    std::copy(l.begin(), l.end(), labels);
    *n_clusters = static_cast<uint64_t>(nc);
    *exact = ex ? 1 : 0;
  });
}
void* orc_coarsen(void* h, const int64_t* labels, uint64_t n_clusters, double beta) {
  (void)beta;
  Csr* out = nullptr;
  guard([&] {
    const Agg p = make_agg(Labels(labels, labels + H(h)->f), static_cast<int64_t>(n_clusters));
    out = new Csr(coarsen(*H(h), p));
  });
  return out;
}
int orc_two_level_apply(void* h, double beta, const int64_t* labels, uint64_t n_clusters, double omega,
                        const double* r, double* z) {
  return guard([&] {
    const Csr& x = *H(h);
    Op fine;
    fine.x = &x;
    fine.beta = beta;
    Level L;
    L.p = make_agg(Labels(labels, labels + x.f), static_cast<int64_t>(n_clusters));
    L.xc = coarsen(x, L.p);
    L.beta = beta;
    L.op.x = &L.xc;
    L.op.beta = beta;
    TwoLevel t;
    t.fine = &fine;
    t.coarse = &L;
    t.omega = omega;
    t.kind = OR_COARSE_DIRECT;
    t.setup();
    t.apply(r, z);
  });
}
// PreparedMethod (krylov.cpp:617-668)
int orc_solve(void* h, double beta, int32_t method, const or_level_spec* levels, uint64_t n_levels,
              const or_solver_config* cfg, const double* b, double* w, or_solve_report* rep) {
  return guard([&] {
    const Csr& x = *H(h);
    Vec rhs(x.f);
    mul_t(x, b, rhs.data());  // krylov.cpp:655
    Report r;
    Vec sol;
    if (method == OR_METHOD_CG || method == OR_METHOD_JACOBI_CG) {
      if (beta < 0.0) throw std::invalid_argument("RidgeOperator: beta must be nonnegative");
      Op op;
      op.x = &x;
      op.beta = beta;
      Vec inv;
      if (method == OR_METHOD_JACOBI_CG) {
        inv.assign(x.f, beta);
        for (int64_t k = 0; k < x.nnz(); ++k) inv[x.idx[k]] += x.val[k] * x.val[k];
        for (auto& d : inv) {
          if (!(d > 0.0)) throw std::invalid_argument("JacobiPreconditioner: diagonal must be positive");
          d = 1.0 / d;
        }
      }
      sol = cg(op, rhs, cfg->tol, cfg->max_iters, method == OR_METHOD_JACOBI_CG ? &inv : nullptr, r);
      if (rep) {
        rep->n_levels = 1;
        rep->level_sizes[0] = x.f;
      }
    } else {
      std::vector<or_level_spec> sp(levels, levels + n_levels);
      if (method == OR_METHOD_FCG_TWOLEVEL || method == OR_METHOD_FGMRES_TWOLEVEL) {  // krylov.cpp:628-635
        if (sp.empty()) throw std::invalid_argument("two-level method requires one level spec");
        sp.resize(1);
        sp[0].coarse_kind = OR_COARSE_DIRECT;
      }
      auto hier = build(x, beta, sp.data(), sp.size());
      if (method == OR_METHOD_FGMRES_TWOLEVEL)
        sol = fgmres(hier->fine_op, rhs, cfg->tol, cfg->max_iters, *hier->pc[0], r);
      else
        sol = fcg(hier->fine_op, rhs, cfg->tol, cfg->max_iters, cfg->truncation, *hier->pc[0], r);
      if (rep) {
        rep->n_levels = sp.size() + 1;
        for (size_t k = 0; k < sp.size() && k < 8; ++k) rep->omega[k] = hier->omega[k];
        for (size_t k = 0; k <= sp.size() && k < 8; ++k) rep->level_sizes[k] = hier->mat(k).f;
      }
    }
    std::memcpy(w, sol.data(), sol.size() * sizeof(double));
    fill(r, rep);
  });
}

}  // extern "C"
