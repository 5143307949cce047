// TEST INFRASTRUCTURE ONLY — the BASELINE.json synthetic inputs,
// restated for the two CPU checkers under oracle/ so that the reference arm of
// bench.py and the parity fixtures never load the product library to build
// their inputs ("feed it ... the oracle's own CounterRng
// generator").  Templated on the RNG so ref_capi.cpp instantiates it with the
// reference's own ridgemg::CounterRng (proj/include/ridgemg/rng.hpp:25-72) and
// restatement.cpp with its restated one.  tests/test_oracle_pin.py checks that
// both produce the same bytes as the product's generator (SHA-256 of the CSR).
//
// Recipe (cfg 2 / 3 / 5):
//   * a Zipf(s) popularity table over a seeded permutation of the F features
//     (Fisher-Yates with next_index, then cumulative k^-s);
//   * per row: k = max(1, Poisson(mean)) by inverse CDF (capped at F), then k
//     distinct columns drawn by inverse CDF over the table (without replacement),
//     each followed by |N(0,1)| when values are requested, then sorted by column.
//   * "row streams": row r draws from its own RNG seeded by a hash of (seed, r),
//     so many threads generate rows at once (large configs).
#pragma once

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <numeric>
#include <thread>
#include <vector>

namespace oracle_synth {

struct Csr64 {
  int64_t n = 0, f = 0;
  std::vector<uint64_t> ptr, idx;
  std::vector<double> val;  // empty for binary patterns
};

struct Popularity {
  std::vector<int64_t> perm;
  std::vector<double> cdf;
  double total = 0.0;
  template <class Rng>
  Popularity(int64_t f, double s, Rng& rng) : perm(f), cdf(f) {
    std::iota(perm.begin(), perm.end(), int64_t{0});
    for (int64_t i = f; i > 1; --i) std::swap(perm[i - 1], perm[rng.next_index(static_cast<uint64_t>(i))]);
    double run = 0.0;
    for (int64_t k = 0; k < f; ++k) {
      run += std::pow(static_cast<double>(k + 1), -s);
      cdf[k] = run;
    }
    total = run;
  }
};

template <class Rng>
void draw_row(Rng& rng, const Popularity& z, int64_t f, double mean, bool values, std::vector<uint64_t>& idx,
              std::vector<double>& val) {
  const double u = rng.next_double();
  int64_t k = 0;
  double pk = std::exp(-mean), cum = pk;
  const int64_t kmax = 20 * static_cast<int64_t>(mean) + 100;
  while (u >= cum && k < kmax) {
    ++k;
    pk *= mean / static_cast<double>(k);
    cum += pk;
  }
  k = std::min<int64_t>(std::max<int64_t>(k, 1), f);
  std::vector<std::pair<int64_t, double>> row;
  row.reserve(static_cast<size_t>(k));
  while (static_cast<int64_t>(row.size()) < k) {
    const double t = rng.next_double() * z.total;
    int64_t rank = std::upper_bound(z.cdf.begin(), z.cdf.end(), t) - z.cdf.begin();
    if (rank >= f) rank = f - 1;
    const int64_t col = z.perm[rank];
    bool seen = false;
    for (const auto& e : row) seen = seen || e.first == col;
    if (seen) continue;
    row.emplace_back(col, values ? std::fabs(rng.next_normal()) : 1.0);
  }
  std::sort(row.begin(), row.end(), [](const auto& a, const auto& b) { return a.first < b.first; });
  for (const auto& e : row) {
    idx.push_back(static_cast<uint64_t>(e.first));
    if (values) val.push_back(e.second);
  }
}

inline uint64_t row_seed(uint64_t seed, int64_t r) {
  uint64_t h = seed ^ (static_cast<uint64_t>(r) + 1) * 0xD1B54A32D192ED03ull;
  h = (h ^ (h >> 33)) * 0xFF51AFD7ED558CCDull;
  return h ^ (h >> 29);
}

template <class Rng>
Csr64 sparse_zipf(int64_t n, int64_t f, double mean, double s, bool values, uint64_t seed, bool row_streams) {
  Csr64 m;
  m.n = n;
  m.f = f;
  m.ptr.assign(static_cast<size_t>(n) + 1, 0);
  Rng table_rng(seed);
  const Popularity z(f, s, table_rng);
  if (!row_streams) {
    for (int64_t r = 0; r < n; ++r) {
      draw_row(table_rng, z, f, mean, values, m.idx, m.val);
      m.ptr[r + 1] = m.idx.size();
    }
    return m;
  }
  const int64_t T = std::max<int64_t>(1, std::min<int64_t>(64, std::thread::hardware_concurrency()));
  const int64_t chunk = (n + T - 1) / T;
  std::vector<std::vector<uint64_t>> idx(T), len(T);
  std::vector<std::vector<double>> val(T);
  std::vector<std::thread> pool;
  for (int64_t t = 0; t < T; ++t) {
    pool.emplace_back([&, t] {
      const int64_t r0 = std::min(n, t * chunk), r1 = std::min(n, r0 + chunk);
      for (int64_t r = r0; r < r1; ++r) {
        Rng rng(row_seed(seed, r));
        const size_t before = idx[t].size();
        draw_row(rng, z, f, mean, values, idx[t], val[t]);
        len[t].push_back(idx[t].size() - before);
      }
    });
  }
  for (auto& th : pool) th.join();
  size_t total = 0;
  for (const auto& v : idx) total += v.size();
  m.idx.reserve(total);
  if (values) m.val.reserve(total);
  int64_t r = 0;
  for (int64_t t = 0; t < T; ++t) {
    for (uint64_t l : len[t]) {
      m.ptr[r + 1] = m.ptr[r] + l;
      ++r;
    }
    m.idx.insert(m.idx.end(), idx[t].begin(), idx[t].end());
    if (values) m.val.insert(m.val.end(), val[t].begin(), val[t].end());
    std::vector<uint64_t>().swap(idx[t]);
    std::vector<double>().swap(val[t]);
  }
  return m;
}

// cfg 1: Z (N x groups normals, column order), then X[:,j] = Z[:, j mod groups] +
// noise * N(0,1) in column order; stored as CSR of the nonzero entries.
template <class Rng>
Csr64 dense_clustered(int64_t n, int64_t f, int64_t groups, double noise, uint64_t seed) {
  Rng rng(seed);
  std::vector<double> z(static_cast<size_t>(n) * groups), x(static_cast<size_t>(n) * f);
  for (int64_t g = 0; g < groups; ++g)
    for (int64_t r = 0; r < n; ++r) z[g * n + r] = rng.next_normal();
  for (int64_t j = 0; j < f; ++j)
    for (int64_t r = 0; r < n; ++r) x[j * n + r] = z[(j % groups) * n + r] + noise * rng.next_normal();
  Csr64 m;
  m.n = n;
  m.f = f;
  m.ptr.assign(static_cast<size_t>(n) + 1, 0);
  for (int64_t r = 0; r < n; ++r) {
    for (int64_t j = 0; j < f; ++j) {
      const double v = x[j * n + r];
      if (v == 0.0) continue;
      m.idx.push_back(static_cast<uint64_t>(j));
      m.val.push_back(v);
    }
    m.ptr[r + 1] = m.idx.size();
  }
  return m;
}

}  // namespace oracle_synth
