// Host-side setup of the ridgemg_b200 path.  See host_setup.hpp.
#include "host_setup.hpp"

#include <algorithm>
#include <cmath>
#include <limits>
#include <numeric>
#include <atomic>
#include <functional>
#include <thread>

namespace rmg {

// ------------------------------------------------------------------ RNG (rng.hpp:25-72)
uint64_t CounterRng::next_u64() {
  uint64_t z = seed_ + (++k_) * 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}
double CounterRng::next_double() { return static_cast<double>(next_u64() >> 11) * 0x1.0p-53; }
double CounterRng::next_double_open() { return (static_cast<double>(next_u64() >> 11) + 1.0) * 0x1.0p-53; }
double CounterRng::next_normal() {
  if (has_cached_) {
    has_cached_ = false;
    return cached_;
  }
  const double u1 = next_double_open();
  const double u2 = next_double();
  const double rad = std::sqrt(-2.0 * std::log(u1));
  const double ang = 2.0 * 3.141592653589793238462643383279502884 * u2;
  cached_ = rad * std::sin(ang);
  has_cached_ = true;
  return rad * std::cos(ang);
}
uint64_t CounterRng::next_index(uint64_t n) {
  const auto v = static_cast<uint64_t>(next_double() * static_cast<double>(n));
  return v >= n ? n - 1 : v;
}

// ------------------------------------------------------------------ CSR helpers
void validate_csr(const HostCsr& m) {
  if (m.n < 0 || m.f < 0) throw InvalidArgument("FeatureMatrix: negative shape");
  if (static_cast<int64_t>(m.ptr.size()) != m.n + 1) throw InvalidArgument("FeatureMatrix: row_offsets length != n_samples + 1");
  if (m.ptr[0] != 0 || m.ptr[m.n] != m.nnz()) throw InvalidArgument("FeatureMatrix: row_offsets do not span the nonzeros");
  if (!m.val.empty() && static_cast<int64_t>(m.val.size()) != m.nnz())
    throw InvalidArgument("FeatureMatrix: values length != nnz");
  // Row blocks on threads (cfg 5 validates four 1e9-entry levels); the error reported is the
  // sequential scan's: every block stops at its first, the lowest block's wins.
  const int64_t T = m.nnz() < (int64_t{1} << 22)
                        ? 1
                        : std::max<int64_t>(1, std::min<int64_t>(32, std::thread::hardware_concurrency()));
  std::vector<std::string> err(static_cast<size_t>(T));
  auto body = [&](int64_t t) {
    const int64_t ra = m.n * t / T, rb = m.n * (t + 1) / T;
    for (int64_t r = ra; r < rb; ++r) {
      if (m.ptr[r + 1] < m.ptr[r]) {
        err[t] = "FeatureMatrix: row_offsets decrease at row " + std::to_string(r);
        return;
      }
      if (m.ptr[r] < 0 || m.ptr[r + 1] > m.nnz()) {  // offsets that leave [0, nnz] must not index idx
        err[t] = "FeatureMatrix: row_offsets do not span the nonzeros";
        return;
      }
      for (int64_t k = m.ptr[r]; k < m.ptr[r + 1]; ++k) {
        const int64_t c = m.idx[k];
        if (c < 0 || c >= m.f) {
          err[t] = "FeatureMatrix: column index out of range in row " + std::to_string(r);
          return;
        }
        if (k > m.ptr[r] && c <= m.idx[k - 1]) {
          err[t] = "FeatureMatrix: column indices not strictly increasing in row " + std::to_string(r);
          return;
        }
        if (!m.val.empty() && !std::isfinite(m.val[k])) {
          err[t] = "FeatureMatrix: non-finite value";
          return;
        }
      }
    }
  };
  std::vector<std::thread> pool;
  for (int64_t t = 1; t < T; ++t) pool.emplace_back(body, t);
  body(0);
  for (auto& th : pool) th.join();
  for (const std::string& e : err)
    if (!e.empty()) throw InvalidArgument(e);
}

// X^T as CSR with the samples of every feature in increasing order.  Threaded over
// nnz-balanced row blocks: per-(block, column) counts, a prefix over (column, block),
// then every block scatters its rows in order at its own cursors -- the result is the
// sequential loop's, entry for entry (cfg 5: four 1e9-entry transposes per prepare).
HostCsr transpose(const HostCsr& m) {
  HostCsr t;
  t.n = m.f;
  t.f = m.n;
  t.ptr.assign(m.f + 1, 0);
  t.idx.resize(m.nnz());
  if (!m.val.empty()) t.val.resize(m.nnz());
  int64_t T = std::max<int64_t>(1, std::min<int64_t>(32, std::thread::hardware_concurrency()));
  if (m.nnz() < (int64_t{1} << 20) || m.f * T > (int64_t{1} << 28)) T = 1;  // small, or the count table would be large
  if (T == 1) {
    for (int64_t k = 0; k < m.nnz(); ++k) t.ptr[m.idx[k] + 1]++;
    for (int64_t j = 0; j < m.f; ++j) t.ptr[j + 1] += t.ptr[j];
    std::vector<int64_t> next(t.ptr.begin(), t.ptr.end() - 1);
    for (int64_t r = 0; r < m.n; ++r)
      for (int64_t k = m.ptr[r]; k < m.ptr[r + 1]; ++k) {
        const int64_t d = next[m.idx[k]]++;
        t.idx[d] = r;  // rows arrive in increasing order per column
        if (!m.val.empty()) t.val[d] = m.val[k];
      }
    return t;
  }
  std::vector<int64_t> rb(T + 1, m.n);  // row blocks of about nnz / T entries
  rb[0] = 0;
  for (int64_t b = 1; b < T; ++b)
    rb[b] = std::lower_bound(m.ptr.begin(), m.ptr.end(), m.nnz() / T * b) - m.ptr.begin();
  for (int64_t b = 1; b <= T; ++b) rb[b] = std::min<int64_t>(m.n, std::max(rb[b], rb[b - 1]));
  std::vector<std::vector<int64_t>> cur(T);
  auto run = [&](auto fn) {
    std::vector<std::thread> pool;
    for (int64_t b = 0; b < T; ++b) pool.emplace_back([&, b] { fn(b); });
    for (auto& th : pool) th.join();
  };
  run([&](int64_t b) {
    cur[b].assign(m.f, 0);
    for (int64_t k = m.ptr[rb[b]]; k < m.ptr[rb[b + 1]]; ++k) ++cur[b][m.idx[k]];
  });
  int64_t runsum = 0;
  for (int64_t j = 0; j < m.f; ++j) {  // counts -> each block's first slot in column j
    t.ptr[j] = runsum;
    for (int64_t b = 0; b < T; ++b) {
      const int64_t c = cur[b][j];
      cur[b][j] = runsum;
      runsum += c;
    }
  }
  t.ptr[m.f] = runsum;
  run([&](int64_t b) {
    std::vector<int64_t>& next = cur[b];
    for (int64_t r = rb[b]; r < rb[b + 1]; ++r)
      for (int64_t k = m.ptr[r]; k < m.ptr[r + 1]; ++k) {
        const int64_t d = next[m.idx[k]]++;
        t.idx[d] = r;
        if (!m.val.empty()) t.val[d] = m.val[k];
      }
  });
  return t;
}

HostCsr normalized_columns(const HostCsr& m) {
  std::vector<double> nrm(m.f, 0.0);
  for (int64_t k = 0; k < m.nnz(); ++k) {
    const double v = m.val.empty() ? 1.0 : m.val[k];
    nrm[m.idx[k]] += v * v;  // per column: increasing row order
  }
  for (double& v : nrm) v = std::sqrt(v);
  HostCsr y = m;
  y.val.resize(m.nnz());
  for (int64_t k = 0; k < m.nnz(); ++k) y.val[k] = (m.val.empty() ? 1.0 : m.val[k]) / nrm[m.idx[k]];
  return y;
}

namespace {

inline double value_at(const HostCsr& m, int64_t k) { return m.val.empty() ? 1.0 : m.val[k]; }

template <class F>
void parallel_ranges(int64_t n, unsigned threads, F&& body) {
  if (threads <= 1 || n < 512) {
    body(int64_t{0}, n);
    return;
  }
  std::vector<std::thread> pool;
  const int64_t step = (n + threads - 1) / threads;
  for (unsigned t = 0; t < threads; ++t) {
    const int64_t lo = std::min<int64_t>(n, t * step), hi = std::min<int64_t>(n, lo + step);
    if (lo < hi) pool.emplace_back([&, lo, hi] { body(lo, hi); });
  }
  for (auto& th : pool) th.join();
}

// Euclidean distance of two sparse columns over the merged supports in
// increasing row order (distance.cpp:27-67).  A row in one support only adds
// (x - 0)^2 = x^2 (exact operands), a shared row (x_i - x_j)^2, and (x - y)^2 ==
// (y - x)^2 exactly, so the lists may swap roles: the longer one is walked in
// runs between the shorter one's entries (binary search, then a branch-free
// sum).  Same terms, same order, same rounding as the element-wise merge.
double column_euclid(const HostCsr& xt, int64_t i, int64_t j) {
  int64_t a = xt.ptr[i], ae = xt.ptr[i + 1], b = xt.ptr[j], be = xt.ptr[j + 1];
  if (ae - a < be - b) {
    std::swap(a, b);
    std::swap(ae, be);
  }
  const int64_t* idx = xt.idx.data();
  const double* val = xt.val.empty() ? nullptr : xt.val.data();
  auto v = [&](int64_t q) { return val ? val[q] : 1.0; };
  double s = 0.0;
  for (; b < be; ++b) {
    const int64_t target = idx[b];
    const int64_t p = std::lower_bound(idx + a, idx + ae, target) - idx;
    for (; a < p; ++a) {
      const double x = v(a);
      s += x * x;
    }
    const double y = v(b);
    if (a < ae && idx[a] == target) {
      const double diff = v(a) - y;
      s += diff * diff;
      ++a;
    } else {
      s += y * y;
    }
  }
  for (; a < ae; ++a) {
    const double x = v(a);
    s += x * x;
  }
  return std::sqrt(s);
}

}  // namespace

// Persistent workers for loops issued many times in a row (k-means++ runs K
// parallel passes): threads are created once, each pass is handed out in
// dynamic chunks (Zipf-hot columns make static ranges uneven).  Which thread
// computes an element never changes the element's value.
class StepPool {
 public:
  explicit StepPool(unsigned threads) {
    for (unsigned t = 1; t < threads; ++t) workers_.emplace_back([this] { loop(); });
  }
  ~StepPool() {
    stop_.store(true);
    gen_.fetch_add(1);
    for (auto& w : workers_) w.join();
  }
  template <class F>
  void run(int64_t n, int64_t chunk, F&& body) {
    body_ = [&](int64_t lo, int64_t hi) { body(lo, hi); };
    n_ = n;
    chunk_ = chunk;
    next_.store(0);
    pending_.store(static_cast<int>(workers_.size()));
    gen_.fetch_add(1);
    work();
    while (pending_.load() != 0) std::this_thread::yield();
  }

 private:
  void work() {
    for (;;) {
      const int64_t lo = next_.fetch_add(chunk_);
      if (lo >= n_) return;
      body_(lo, std::min(n_, lo + chunk_));
    }
  }
  void loop() {
    int64_t seen = 0;
    for (;;) {
      while (gen_.load() == seen) std::this_thread::yield();
      seen = gen_.load();
      if (stop_.load()) return;
      work();
      pending_.fetch_sub(1);
    }
  }
  std::vector<std::thread> workers_;
  std::function<void(int64_t, int64_t)> body_;
  std::atomic<int64_t> gen_{0}, next_{0};
  std::atomic<int> pending_{0};
  std::atomic<bool> stop_{false};
  int64_t n_ = 0, chunk_ = 1;
};

// clustering.cpp:189-255
std::vector<int64_t> kmeanspp_seed(const HostCsr& xt, int64_t k, uint64_t seed, unsigned threads) {
  const int64_t f = xt.n;
  if (k <= 0 || k > f) throw InvalidArgument("kmeanspp_seed: k outside [1, F]");
  CounterRng rng(seed);
  std::vector<int64_t> chosen{static_cast<int64_t>(rng.next_index(f))};
  std::vector<char> used(f, 0);
  used[chosen[0]] = 1;
  std::vector<double> d2(f, std::numeric_limits<double>::infinity()), dist(f, 0.0);
  StepPool pool(f >= 512 ? std::max(1u, threads) : 1u);
  while (static_cast<int64_t>(chosen.size()) < k) {
    const int64_t last = chosen.back();
    pool.run(f, 64, [&](int64_t lo, int64_t hi) {
      for (int64_t j = lo; j < hi; ++j)
        if (!used[j]) dist[j] = column_euclid(xt, j, last);
    });
    double total = 0.0;
    for (int64_t j = 0; j < f; ++j) {
      if (used[j]) {
        d2[j] = 0.0;
        continue;
      }
      d2[j] = std::min(d2[j], dist[j] * dist[j]);
      total += d2[j];
    }
    int64_t pick = -1;
    if (total > 0.0) {
      const double u = rng.next_double() * total;
      double run = 0.0;
      for (int64_t j = 0; j < f && pick < 0; ++j) {
        if (used[j] || d2[j] == 0.0) continue;
        run += d2[j];
        if (u < run) pick = j;
      }
      for (int64_t j = f - 1; pick < 0 && j >= 0; --j)
        if (!used[j] && d2[j] > 0.0) pick = j;
    }
    if (pick < 0) {
      uint64_t idx = rng.next_index(static_cast<uint64_t>(f) - chosen.size());
      for (int64_t j = 0; j < f; ++j) {
        if (used[j]) continue;
        if (idx-- == 0) {
          pick = j;
          break;
        }
      }
    }
    chosen.push_back(pick);
    used[pick] = 1;
  }
  return chosen;
}

// clustering.cpp:257-355.  Prototypes are held transposed, proto[r * k + s];
// each (feature, prototype) distance still starts at ||p_s||^2 and adds
// ((x - p)^2 - p^2) over the feature's rows in increasing order
// (distance.cpp:93-105), so labels match the reference bit for bit.
Clustering kmeans(const HostCsr& xt, int64_t k, uint64_t max_iters, uint64_t seed, unsigned threads) {
  const int64_t f = xt.n, n = xt.f;
  if (k <= 0 || k > f) throw InvalidArgument("kmeans: k outside [1, F]");
  std::vector<double> proto(static_cast<size_t>(n) * k, 0.0);
  auto load_column = [&](int64_t j, int64_t s) {
    for (int64_t r = 0; r < n; ++r) proto[r * k + s] = 0.0;
    for (int64_t q = xt.ptr[j]; q < xt.ptr[j + 1]; ++q) proto[xt.idx[q] * k + s] = value_at(xt, q);
  };
  const std::vector<int64_t> seeds = kmeanspp_seed(xt, k, seed, threads);
  for (int64_t s = 0; s < k; ++s) load_column(seeds[s], s);

  Clustering out;
  std::vector<int64_t> member(f, 0), previous;
  std::vector<int64_t> size(k);
  std::vector<double> psq(k), own(f);
  for (uint64_t iter = 0; iter < std::max<uint64_t>(max_iters, 1); ++iter) {
    std::fill(psq.begin(), psq.end(), 0.0);
    for (int64_t r = 0; r < n; ++r)
      for (int64_t s = 0; s < k; ++s) psq[s] += proto[r * k + s] * proto[r * k + s];
    parallel_ranges(f, threads, [&](int64_t lo, int64_t hi) {
      std::vector<double> acc(k);
      for (int64_t j = lo; j < hi; ++j) {
        acc = psq;
        for (int64_t q = xt.ptr[j]; q < xt.ptr[j + 1]; ++q) {
          const double x = value_at(xt, q);
          const double* pr = &proto[xt.idx[q] * k];
          for (int64_t s = 0; s < k; ++s) {
            const double diff = x - pr[s];
            acc[s] += diff * diff - pr[s] * pr[s];
          }
        }
        int64_t best = 0;
        double best_sq = std::numeric_limits<double>::infinity();
        for (int64_t s = 0; s < k; ++s) {
          const double sq = std::max(acc[s], 0.0);
          if (sq < best_sq) {
            best_sq = sq;
            best = s;
          }
        }
        member[j] = best;
        own[j] = best_sq;
      }
    });
    std::fill(size.begin(), size.end(), 0);
    for (int64_t j = 0; j < f; ++j) size[member[j]]++;
    for (int64_t s = 0; s < k; ++s) {  // empty-cluster repair (clustering.cpp:303-321)
      if (size[s] != 0) continue;
      int64_t far = -1;
      double far_sq = -1.0;
      for (int64_t j = 0; j < f; ++j)
        if (size[member[j]] > 1 && own[j] > far_sq) {
          far_sq = own[j];
          far = j;
        }
      if (far < 0) break;
      size[member[far]]--;
      member[far] = s;
      size[s] = 1;
      load_column(far, s);
      own[far] = 0.0;
    }
    out.iterations = iter + 1;
    if (!previous.empty() && previous == member) {
      out.converged = true;
      break;
    }
    previous = member;
    std::fill(proto.begin(), proto.end(), 0.0);
    for (int64_t j = 0; j < f; ++j)
      for (int64_t q = xt.ptr[j]; q < xt.ptr[j + 1]; ++q) proto[xt.idx[q] * k + member[j]] += value_at(xt, q);
    std::vector<double> inv(k);
    for (int64_t s = 0; s < k; ++s) inv[s] = 1.0 / static_cast<double>(size[s]);
    for (int64_t r = 0; r < n; ++r)
      for (int64_t s = 0; s < k; ++s) proto[r * k + s] *= inv[s];
  }
  out.labels = std::move(member);
  out.n_clusters = k;
  return out;
}

// clustering.cpp:64-130 (fixed leaders)
Clustering leader_follower(const HostCsr& xt, double tol) {
  if (!(tol > 0.0)) throw InvalidArgument("leader_follower: tolerance must be positive");
  if (xt.n == 0) throw InvalidArgument("leader_follower: empty matrix");
  Clustering c;
  c.labels.assign(xt.n, 0);
  std::vector<int64_t> leaders;
  for (int64_t i = 0; i < xt.n; ++i) {
    int64_t best = -1;
    double bd = std::numeric_limits<double>::infinity();
    for (size_t s = 0; s < leaders.size(); ++s) {
      const double d = column_euclid(xt, i, leaders[s]);
      if (d < bd) {
        bd = d;
        best = static_cast<int64_t>(s);
      }
    }
    if (best >= 0 && bd < tol) {
      c.labels[i] = best;
    } else {
      c.labels[i] = static_cast<int64_t>(leaders.size());
      leaders.push_back(i);
    }
  }
  c.n_clusters = static_cast<int64_t>(leaders.size());
  c.tolerance = tol;
  return c;
}

// clustering.cpp:132-187 (bisection on the tolerance)
Clustering leader_follower_target(const HostCsr& xt, int64_t target) {
  if (target <= 0 || target > xt.n) throw InvalidArgument("leader_follower_target: target outside [1, F]");
  double lo = 1e-12, hi = 1.0;
  Clustering at_lo = leader_follower(xt, lo), at_hi = leader_follower(xt, hi);
  for (int grow = 0; at_hi.n_clusters > target && grow < 64; ++grow) {
    hi *= 2.0;
    at_hi = leader_follower(xt, hi);
  }
  Clustering best = at_lo;
  auto gap = [&](const Clustering& c) { return std::llabs(c.n_clusters - target); };
  auto consider = [&](const Clustering& c) {
    if (gap(c) < gap(best) || (gap(c) == gap(best) && c.n_clusters > best.n_clusters)) best = c;
  };
  consider(at_hi);
  for (int probe = 0; probe < 200 && best.n_clusters != target; ++probe) {
    const double mid = 0.5 * (lo + hi);
    if (mid <= lo || mid >= hi) break;
    Clustering at_mid = leader_follower(xt, mid);
    consider(at_mid);
    (at_mid.n_clusters > target ? lo : hi) = mid;
  }
  best.exact = best.n_clusters == target;
  return best;
}

// ------------------------------------------------------------------ aggregation
Aggregation make_aggregation(const std::vector<int64_t>& labels, int64_t nc) {
  Aggregation p;
  p.n_fine = static_cast<int64_t>(labels.size());
  p.n_coarse = nc;
  std::vector<int64_t> size(nc, 0);
  for (int64_t s : labels) {
    if (s < 0 || s >= nc) throw InvalidArgument("ClusterAssignment: cluster id out of range");
    size[s]++;
  }
  for (int64_t s = 0; s < nc; ++s)
    if (size[s] == 0) throw InvalidArgument("ClusterAssignment: empty cluster " + std::to_string(s));
  p.label.resize(p.n_fine);
  p.weight.resize(p.n_fine);
  p.mptr.assign(nc + 1, 0);
  for (int64_t i = 0; i < p.n_fine; ++i) {
    p.label[i] = static_cast<int32_t>(labels[i]);
    p.weight[i] = 1.0 / std::sqrt(static_cast<double>(size[labels[i]]));
    p.mptr[labels[i] + 1]++;
  }
  for (int64_t s = 0; s < nc; ++s) p.mptr[s + 1] += p.mptr[s];
  p.members.resize(p.n_fine);
  std::vector<int32_t> fill(p.mptr.begin(), p.mptr.end() - 1);
  for (int64_t i = 0; i < p.n_fine; ++i) p.members[fill[labels[i]]++] = static_cast<int32_t>(i);
  return p;
}

HostCsr coarsen(const HostCsr& x, const Aggregation& p) {
  if (p.n_fine != x.f) throw InvalidArgument("coarsen: prolongation does not match the matrix features");
  HostCsr c;
  c.n = x.n;
  c.f = p.n_coarse;
  c.ptr.assign(x.n + 1, 0);
  // rows are independent: contiguous row ranges per thread, concatenated in order
  // (each row exactly as the sequential loop builds it, coarsening.cpp:112-148)
  const unsigned T = x.nnz() < (1 << 20) ? 1u : std::max(1u, std::min(32u, std::thread::hardware_concurrency()));
  struct Part {
    std::vector<int64_t> idx;
    std::vector<double> val;
  };
  std::vector<Part> parts(T);
  auto body = [&](unsigned t) {
    const int64_t r0 = x.n * t / T, r1 = x.n * (t + 1) / T;
    Part& out = parts[t];
    std::vector<double> acc(p.n_coarse, 0.0);
    std::vector<int64_t> stamp(p.n_coarse, -1), hit;
    for (int64_t r = r0; r < r1; ++r) {
      hit.clear();
      for (int64_t k = x.ptr[r]; k < x.ptr[r + 1]; ++k) {
        const int64_t i = x.idx[k];
        const int32_t s = p.label[i];
        if (stamp[s] != r) {
          stamp[s] = r;
          hit.push_back(s);
        }
        acc[s] += value_at(x, k) * p.weight[i];
      }
      std::sort(hit.begin(), hit.end());
      for (int64_t s : hit) {
        out.idx.push_back(s);
        out.val.push_back(acc[s]);
        acc[s] = 0.0;
      }
      c.ptr[r + 1] = static_cast<int64_t>(hit.size());
    }
  };
  if (T == 1) {
    body(0);
  } else {
    std::vector<std::thread> pool;
    for (unsigned t = 0; t < T; ++t) pool.emplace_back(body, t);
    for (auto& th : pool) th.join();
  }
  for (int64_t r = 0; r < x.n; ++r) c.ptr[r + 1] += c.ptr[r];
  c.idx.resize(c.ptr[x.n]);
  c.val.resize(c.ptr[x.n]);
  {
    std::vector<std::thread> pool;
    int64_t off = 0;
    for (unsigned t = 0; t < T; ++t) {
      pool.emplace_back([&, t, off] {
        std::copy(parts[t].idx.begin(), parts[t].idx.end(), c.idx.begin() + off);
        std::copy(parts[t].val.begin(), parts[t].val.end(), c.val.begin() + off);
      });
      off += static_cast<int64_t>(parts[t].idx.size());
    }
    for (auto& th : pool) th.join();
  }
  return c;
}

std::vector<double> coarse_gram(const HostCsr& xc, double beta) {
  const int64_t n = xc.f;
  std::vector<double> a(static_cast<size_t>(n) * n, 0.0);
  for (int64_t r = 0; r < xc.n; ++r)
    for (int64_t p = xc.ptr[r]; p < xc.ptr[r + 1]; ++p) {
      const double vp = value_at(xc, p);
      double* row = &a[xc.idx[p] * n];
      for (int64_t q = xc.ptr[r]; q < xc.ptr[r + 1]; ++q) row[xc.idx[q]] += vp * value_at(xc, q);
    }
  for (int64_t i = 0; i < n; ++i) a[i * n + i] += beta;
  return a;
}

std::vector<double> spd_inverse(const std::vector<double>& a, int64_t n, const std::string& context) {
  std::vector<double> l(static_cast<size_t>(n) * n, 0.0);
  for (int64_t j = 0; j < n; ++j) {
    double d = a[j * n + j];
    for (int64_t k = 0; k < j; ++k) d -= l[j * n + k] * l[j * n + k];
    if (!(d > 0.0) || !std::isfinite(d))
      throw RuntimeError("coarse Cholesky factorization failed at " + context + " (coarse size " +
                         std::to_string(n) +
                         "); the Galerkin operator is numerically indefinite - consider a larger beta or a "
                         "smaller coarse level");
    const double ljj = std::sqrt(d);
    l[j * n + j] = ljj;
    for (int64_t i = j + 1; i < n; ++i) {
      double s = a[i * n + j];
      for (int64_t k = 0; k < j; ++k) s -= l[i * n + k] * l[j * n + k];
      l[i * n + j] = s / ljj;
    }
  }
  std::vector<double> inv(static_cast<size_t>(n) * n, 0.0);
  const unsigned threads = std::max(1u, std::min(16u, std::thread::hardware_concurrency()));
  parallel_ranges(n, n >= 256 ? threads : 1, [&](int64_t lo, int64_t hi) {
    std::vector<double> y(n), x(n);
    for (int64_t c = lo; c < hi; ++c) {
      for (int64_t i = 0; i < n; ++i) {
        double s = i == c ? 1.0 : 0.0;
        for (int64_t k = 0; k < i; ++k) s -= l[i * n + k] * y[k];
        y[i] = s / l[i * n + i];
      }
      for (int64_t i = n; i-- > 0;) {
        double s = y[i];
        for (int64_t k = i + 1; k < n; ++k) s -= l[k * n + i] * x[k];
        x[i] = s / l[i * n + i];
      }
      for (int64_t i = 0; i < n; ++i) inv[i * n + c] = x[i];
    }
  });
  return inv;
}

// ------------------------------------------------------------------ synthetic inputs
HostCsr synth_dense_clustered(int64_t n, int64_t f, int64_t groups, double noise, uint64_t seed) {
  if (n <= 0 || f <= 0 || groups <= 0) throw InvalidArgument("synth_dense_clustered: bad shape");
  CounterRng rng(seed);
  std::vector<double> z(static_cast<size_t>(n) * groups);  // column order
  for (int64_t g = 0; g < groups; ++g)
    for (int64_t r = 0; r < n; ++r) z[g * n + r] = rng.next_normal();
  std::vector<double> x(static_cast<size_t>(n) * f);  // column order
  for (int64_t j = 0; j < f; ++j) {
    const double* zc = &z[(j % groups) * n];
    for (int64_t r = 0; r < n; ++r) x[j * n + r] = zc[r] + noise * rng.next_normal();
  }
  HostCsr m;
  m.n = n;
  m.f = f;
  m.ptr.resize(n + 1);
  m.idx.reserve(n * f);
  m.val.reserve(n * f);
  for (int64_t r = 0; r < n; ++r) {
    m.ptr[r] = m.nnz();
    for (int64_t j = 0; j < f; ++j) {
      const double v = x[j * n + r];
      if (v == 0.0) continue;
      m.idx.push_back(j);
      m.val.push_back(v);
    }
  }
  m.ptr[n] = m.nnz();
  return m;
}

namespace {

struct ZipfTable {
  std::vector<int64_t> perm;
  std::vector<double> cdf;
  double total = 0.0;
  ZipfTable(int64_t f, double zipf_s, CounterRng& rng) : perm(f), cdf(f) {
    std::iota(perm.begin(), perm.end(), int64_t{0});
    for (int64_t i = f; i > 1; --i) std::swap(perm[i - 1], perm[rng.next_index(i)]);
    double run = 0.0;
    for (int64_t k = 0; k < f; ++k) {
      run += std::pow(static_cast<double>(k + 1), -zipf_s);
      cdf[k] = run;
    }
    total = run;
  }
};

// One row: k = max(1, Poisson(mean)) by inverse CDF (capped at F), then k
// distinct columns by Zipf rank (without replacement), sorted by column.
void zipf_row(CounterRng& rng, const ZipfTable& z, int64_t f, double mean_nnz, bool abs_normal_values,
              std::vector<int64_t>& row, std::vector<double>& rv, std::vector<int64_t>& idx_out,
              std::vector<double>& val_out) {
  const double u = rng.next_double();
  int64_t kk = 0;
  double pk = std::exp(-mean_nnz), cum = pk;
  while (u >= cum && kk < 20 * static_cast<int64_t>(mean_nnz) + 100) {
    ++kk;
    pk *= mean_nnz / static_cast<double>(kk);
    cum += pk;
  }
  kk = std::min<int64_t>(std::max<int64_t>(kk, 1), f);
  row.clear();
  rv.clear();
  while (static_cast<int64_t>(row.size()) < kk) {
    const double t = rng.next_double() * z.total;
    int64_t rank = std::upper_bound(z.cdf.begin(), z.cdf.end(), t) - z.cdf.begin();
    if (rank >= f) rank = f - 1;
    const int64_t col = z.perm[rank];
    if (std::find(row.begin(), row.end(), col) != row.end()) continue;
    row.push_back(col);
    if (abs_normal_values) rv.push_back(std::fabs(rng.next_normal()));
  }
  std::vector<size_t> order(row.size());
  std::iota(order.begin(), order.end(), size_t{0});
  std::sort(order.begin(), order.end(), [&](size_t a, size_t b) { return row[a] < row[b]; });
  for (size_t q : order) {
    idx_out.push_back(row[q]);
    if (abs_normal_values) val_out.push_back(rv[q]);
  }
}

}  // namespace

HostCsr synth_sparse_zipf(int64_t n, int64_t f, double mean_nnz, double zipf_s, bool abs_normal_values,
                          uint64_t seed) {
  if (n <= 0 || f <= 0 || !(mean_nnz > 0.0)) throw InvalidArgument("synth_sparse_zipf: bad shape");
  CounterRng rng(seed);
  const ZipfTable z(f, zipf_s, rng);
  HostCsr m;
  m.n = n;
  m.f = f;
  m.ptr.resize(n + 1);
  m.idx.reserve(static_cast<size_t>(n * mean_nnz * 1.05));
  if (abs_normal_values) m.val.reserve(m.idx.capacity());
  std::vector<int64_t> row;
  std::vector<double> rv;
  for (int64_t r = 0; r < n; ++r) {
    m.ptr[r] = m.nnz();
    zipf_row(rng, z, f, mean_nnz, abs_normal_values, row, rv, m.idx, m.val);
  }
  m.ptr[n] = m.nnz();
  return m;
}

// Same distribution with one RNG stream per row (seeded from (seed, row)), so
// rows are generated by all host threads: large measurement shards (cfg5).
HostCsr synth_sparse_zipf_rows(int64_t n_total, int64_t f, double mean_nnz, double zipf_s, bool abs_normal_values,
                               uint64_t seed, int64_t row0, int64_t row1) {
  if (row1 < 0) row1 = n_total;
  if (n_total <= 0 || f <= 0 || !(mean_nnz > 0.0)) throw InvalidArgument("synth_sparse_zipf: bad shape");
  if (row0 < 0 || row1 > n_total || row0 > row1) throw InvalidArgument("synth_sparse_zipf: row range outside [0, n)");
  const int64_t n = row1 - row0;  // rows [row0, row1) of the n_total-row matrix
  CounterRng table_rng(seed);
  const ZipfTable z(f, zipf_s, table_rng);
  const int64_t T = std::max<int64_t>(1, std::min<int64_t>(64, std::thread::hardware_concurrency()));
  const int64_t chunk = (n + T - 1) / T;
  std::vector<std::vector<int64_t>> idx(T), len(T);
  std::vector<std::vector<double>> val(T);
  std::vector<std::thread> pool;
  for (int64_t t = 0; t < T; ++t) {
    pool.emplace_back([&, t] {
      std::vector<int64_t> row;
      std::vector<double> rv;
      const int64_t r0 = t * chunk, r1 = std::min(n, r0 + chunk);
      if (r0 >= r1) return;
      idx[t].reserve(static_cast<size_t>((r1 - r0) * mean_nnz * 1.05));
      for (int64_t r = r0 + row0; r < r1 + row0; ++r) {  // global row numbers seed the streams
        uint64_t h = seed ^ (static_cast<uint64_t>(r) + 1) * 0xD1B54A32D192ED03ull;
        h = (h ^ (h >> 33)) * 0xFF51AFD7ED558CCDull;
        CounterRng rng(h ^ (h >> 29));
        const size_t before = idx[t].size();
        zipf_row(rng, z, f, mean_nnz, abs_normal_values, row, rv, idx[t], val[t]);
        len[t].push_back(static_cast<int64_t>(idx[t].size() - before));
      }
    });
  }
  for (auto& th : pool) th.join();
  HostCsr m;
  m.n = n;
  m.f = f;
  m.ptr.assign(n + 1, 0);
  size_t total = 0;
  for (auto& v : idx) total += v.size();
  m.idx.reserve(total);
  if (abs_normal_values) m.val.reserve(total);
  int64_t r = 0;
  for (int64_t t = 0; t < T; ++t) {
    for (int64_t l : len[t]) {
      m.ptr[r + 1] = m.ptr[r] + l;
      ++r;
    }
    m.idx.insert(m.idx.end(), idx[t].begin(), idx[t].end());
    if (abs_normal_values) m.val.insert(m.val.end(), val[t].begin(), val[t].end());
    std::vector<int64_t>().swap(idx[t]);
  }
  return m;
}

}  // namespace rmg
