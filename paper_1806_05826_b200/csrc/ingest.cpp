// Ingest: the Matrix Market reader (matrix_market.cpp:34-148,
// same accepted variants and error cases), csr_from_triplets (sparse.cpp:27-73:
// sorted by (row, column), duplicates summed in input order) and a binary CSR
// cache stamped with the SHA-256 of its arrays, so a large synthetic or parsed
// input is built once and re-read at disk speed.
//
// Cache layout (little-endian): "RMGCSR01", n, f, nnz (uint64), has_values
// (uint64), the 32-byte SHA-256, then row offsets (uint64[n+1]), column indices
// (uint64[nnz]) and, if has_values, values (fp64[nnz]).  The digest covers the
// arrays as the checkers export them (uint64 offsets, uint64 indices, fp64 values
// with 1.0 for a binary pattern) -- the same bytes bench.py and the fixtures hash.
#include <algorithm>
#include <array>
#include <cctype>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <numeric>
#include <string>
#include <vector>

#include "host_setup.hpp"
#include "ingest.hpp"

namespace rmg {
namespace {

// ---------------------------------------------------------------- SHA-256 (FIPS 180-4)
struct Sha256 {
  uint32_t h[8] = {0x6a09e667u, 0xbb67ae85u, 0x3c6ef372u, 0xa54ff53au,
                   0x510e527fu, 0x9b05688cu, 0x1f83d9abu, 0x5be0cd19u};
  uint8_t buf[64];
  size_t used = 0;
  uint64_t bytes = 0;
  static uint32_t rotr(uint32_t x, int n) { return (x >> n) | (x << (32 - n)); }
  void block(const uint8_t* p) {
    static const uint32_t k[64] = {
        0x428a2f98u, 0x71374491u, 0xb5c0fbcfu, 0xe9b5dba5u, 0x3956c25bu, 0x59f111f1u, 0x923f82a4u, 0xab1c5ed5u,
        0xd807aa98u, 0x12835b01u, 0x243185beu, 0x550c7dc3u, 0x72be5d74u, 0x80deb1feu, 0x9bdc06a7u, 0xc19bf174u,
        0xe49b69c1u, 0xefbe4786u, 0x0fc19dc6u, 0x240ca1ccu, 0x2de92c6fu, 0x4a7484aau, 0x5cb0a9dcu, 0x76f988dau,
        0x983e5152u, 0xa831c66du, 0xb00327c8u, 0xbf597fc7u, 0xc6e00bf3u, 0xd5a79147u, 0x06ca6351u, 0x14292967u,
        0x27b70a85u, 0x2e1b2138u, 0x4d2c6dfcu, 0x53380d13u, 0x650a7354u, 0x766a0abbu, 0x81c2c92eu, 0x92722c85u,
        0xa2bfe8a1u, 0xa81a664bu, 0xc24b8b70u, 0xc76c51a3u, 0xd192e819u, 0xd6990624u, 0xf40e3585u, 0x106aa070u,
        0x19a4c116u, 0x1e376c08u, 0x2748774cu, 0x34b0bcb5u, 0x391c0cb3u, 0x4ed8aa4au, 0x5b9cca4fu, 0x682e6ff3u,
        0x748f82eeu, 0x78a5636fu, 0x84c87814u, 0x8cc70208u, 0x90befffau, 0xa4506cebu, 0xbef9a3f7u, 0xc67178f2u};
    uint32_t w[64];
    for (int t = 0; t < 16; ++t)
      w[t] = (uint32_t(p[4 * t]) << 24) | (uint32_t(p[4 * t + 1]) << 16) | (uint32_t(p[4 * t + 2]) << 8) |
             uint32_t(p[4 * t + 3]);
    for (int t = 16; t < 64; ++t) {
      const uint32_t s0 = rotr(w[t - 15], 7) ^ rotr(w[t - 15], 18) ^ (w[t - 15] >> 3);
      const uint32_t s1 = rotr(w[t - 2], 17) ^ rotr(w[t - 2], 19) ^ (w[t - 2] >> 10);
      w[t] = w[t - 16] + s0 + w[t - 7] + s1;
    }
    uint32_t a = h[0], b = h[1], c = h[2], d = h[3], e = h[4], f = h[5], g = h[6], hh = h[7];
    for (int t = 0; t < 64; ++t) {
      const uint32_t t1 = hh + (rotr(e, 6) ^ rotr(e, 11) ^ rotr(e, 25)) + ((e & f) ^ (~e & g)) + k[t] + w[t];
      const uint32_t t2 = (rotr(a, 2) ^ rotr(a, 13) ^ rotr(a, 22)) + ((a & b) ^ (a & c) ^ (b & c));
      hh = g;
      g = f;
      f = e;
      e = d + t1;
      d = c;
      c = b;
      b = a;
      a = t1 + t2;
    }
    h[0] += a;
    h[1] += b;
    h[2] += c;
    h[3] += d;
    h[4] += e;
    h[5] += f;
    h[6] += g;
    h[7] += hh;
  }
  void update(const void* data, size_t n) {
    const uint8_t* p = static_cast<const uint8_t*>(data);
    bytes += n;
    if (used) {
      const size_t take = std::min(n, 64 - used);
      std::memcpy(buf + used, p, take);
      used += take;
      p += take;
      n -= take;
      if (used == 64) {
        block(buf);
        used = 0;
      }
    }
    for (; n >= 64; n -= 64, p += 64) block(p);
    if (n) {
      std::memcpy(buf, p, n);
      used = n;
    }
  }
  std::array<uint8_t, 32> finish() {
    const uint64_t bits = bytes * 8;
    const uint8_t one = 0x80, zero = 0;
    update(&one, 1);
    while (used != 56) update(&zero, 1);
    uint8_t len[8];
    for (int i = 0; i < 8; ++i) len[i] = static_cast<uint8_t>(bits >> (56 - 8 * i));
    update(len, 8);
    std::array<uint8_t, 32> out{};
    for (int i = 0; i < 8; ++i)
      for (int j = 0; j < 4; ++j) out[4 * i + j] = static_cast<uint8_t>(h[i] >> (24 - 8 * j));
    return out;
  }
};

// the exported arrays in fixed-size pieces (uint64 / fp64, little-endian hosts)
template <class F>
void for_each_export_chunk(const HostCsr& m, F&& fn) {
  std::vector<uint64_t> u;
  std::vector<double> d;
  constexpr size_t kChunk = size_t(1) << 20;
  for (size_t a = 0; a < m.ptr.size(); a += kChunk) {
    const size_t b = std::min(m.ptr.size(), a + kChunk);
    u.assign(m.ptr.begin() + a, m.ptr.begin() + b);
    fn(u.data(), u.size() * 8);
  }
  for (size_t a = 0; a < m.idx.size(); a += kChunk) {
    const size_t b = std::min(m.idx.size(), a + kChunk);
    u.assign(m.idx.begin() + a, m.idx.begin() + b);
    fn(u.data(), u.size() * 8);
  }
  for (size_t a = 0; a < m.idx.size(); a += kChunk) {
    const size_t b = std::min(m.idx.size(), a + kChunk);
    if (m.val.empty())
      d.assign(b - a, 1.0);
    else
      d.assign(m.val.begin() + a, m.val.begin() + b);
    fn(d.data(), d.size() * 8);
  }
}

std::string hex(const std::array<uint8_t, 32>& d) {
  static const char* k = "0123456789abcdef";
  std::string s;
  for (uint8_t c : d) {
    s += k[c >> 4];
    s += k[c & 15];
  }
  return s;
}

[[noreturn]] void fail(const std::string& origin, const std::string& what) {
  throw RuntimeError(origin + ": " + what);
}

std::string lower(std::string s) {
  for (char& c : s) c = static_cast<char>(std::tolower(static_cast<unsigned char>(c)));
  return s;
}

}  // namespace

std::string csr_sha256(const HostCsr& m) {
  Sha256 h;
  for_each_export_chunk(m, [&](const void* p, size_t n) { h.update(p, n); });
  return hex(h.finish());
}

HostCsr csr_from_triplets(int64_t n, int64_t f, const std::vector<int64_t>& rows, const std::vector<int64_t>& cols,
                          const std::vector<double>& vals) {
  if (rows.size() != cols.size() || rows.size() != vals.size())
    throw InvalidArgument("csr_from_triplets: triplet arrays differ in length");
  const size_t z = rows.size();
  for (size_t k = 0; k < z; ++k) {
    if (rows[k] < 0 || rows[k] >= n || cols[k] < 0 || cols[k] >= f)
      throw InvalidArgument("csr_from_triplets: entry index out of range");
    if (!std::isfinite(vals[k])) throw InvalidArgument("csr_from_triplets: non-finite value");
  }
  std::vector<size_t> order(z);
  std::iota(order.begin(), order.end(), size_t{0});
  std::stable_sort(order.begin(), order.end(), [&](size_t a, size_t b) {
    return rows[a] != rows[b] ? rows[a] < rows[b] : cols[a] < cols[b];
  });
  HostCsr m;
  m.n = n;
  m.f = f;
  m.ptr.assign(n + 1, 0);
  for (size_t q = 0; q < z;) {  // duplicates summed in input order
    const size_t k = order[q];
    double v = vals[k];
    size_t e = q + 1;
    while (e < z && rows[order[e]] == rows[k] && cols[order[e]] == cols[k]) v += vals[order[e++]];
    m.idx.push_back(cols[k]);
    m.val.push_back(v);
    ++m.ptr[rows[k] + 1];
    q = e;
  }
  for (int64_t r = 0; r < n; ++r) m.ptr[r + 1] += m.ptr[r];
  return m;
}

HostCsr read_matrix_market(const std::string& path) {
  FILE* fp = std::fopen(path.c_str(), "r");
  if (fp == nullptr) throw RuntimeError("cannot open Matrix Market file: " + path);
  struct Closer {
    FILE* f;
    ~Closer() { std::fclose(f); }
  } closer{fp};
  std::vector<char> line(1 << 16);
  auto next = [&]() -> bool { return std::fgets(line.data(), static_cast<int>(line.size()), fp) != nullptr; };
  if (!next()) fail(path, "empty file");
  char b[64] = {}, o[64] = {}, fm[64] = {}, fl[64] = {}, sy[64] = {};
  std::sscanf(line.data(), "%63s %63s %63s %63s %63s", b, o, fm, fl, sy);
  const std::string object = lower(o), format = lower(fm), field = lower(fl), symmetry = lower(sy);
  if (std::string(b) != "%%MatrixMarket") fail(path, std::string("malformed header: '") + line.data() + "'");
  if (object != "matrix") fail(path, "unsupported object type '" + object + "'");
  if (format != "coordinate" && format != "array") fail(path, "unsupported format '" + format + "'");
  if (field != "real" && field != "integer" && field != "pattern")
    fail(path, "unsupported field type '" + field + "'");
  if (symmetry != "general" && symmetry != "symmetric") fail(path, "unsupported symmetry '" + symmetry + "'");
  if (format == "array" && field == "pattern") fail(path, "pattern field is not defined for array format");
  const bool sym = symmetry == "symmetric", pattern = field == "pattern";
  bool have = false;
  while (next()) {
    if (line[0] != '%' && line[0] != '\n' && line[0] != '\r' && line[0] != '\0') {
      have = true;
      break;
    }
  }
  if (!have) fail(path, "missing size line");
  long long rows = 0, cols = 0, declared = 0;
  if (format == "coordinate") {
    if (std::sscanf(line.data(), "%lld %lld %lld", &rows, &cols, &declared) != 3) fail(path, "malformed size line");
  } else if (std::sscanf(line.data(), "%lld %lld", &rows, &cols) != 2) {
    fail(path, "malformed size line");
  }
  if (rows <= 0 || cols <= 0) fail(path, "non-positive dimensions");
  if (sym && rows != cols) fail(path, "symmetric matrix must be square");
  std::vector<int64_t> ri, ci;
  std::vector<double> vv;
  auto add = [&](long long r, long long c, double v) {
    ri.push_back(r);
    ci.push_back(c);
    vv.push_back(v);
    if (sym && r != c) {
      ri.push_back(c);
      ci.push_back(r);
      vv.push_back(v);
    }
  };
  if (format == "coordinate") {
    if (declared < 0) fail(path, "negative entry count");
    long long seen = 0;
    while (next()) {
      if (line[0] == '%' || line[0] == '\n' || line[0] == '\r' || line[0] == '\0') continue;
      long long r = 0, c = 0;
      double v = 1.0;
      const int got = pattern ? std::sscanf(line.data(), "%lld %lld", &r, &c)
                              : std::sscanf(line.data(), "%lld %lld %lf", &r, &c, &v);
      if (got < 2) fail(path, std::string("malformed entry: '") + line.data() + "'");
      if (!pattern && got < 3) fail(path, std::string("entry missing value: '") + line.data() + "'");
      if (r < 1 || r > rows || c < 1 || c > cols) fail(path, std::string("entry index out of range: '") + line.data() + "'");
      if (!std::isfinite(v)) fail(path, std::string("non-finite value: '") + line.data() + "'");
      ++seen;
      add(r - 1, c - 1, v);
    }
    if (seen != declared)
      fail(path, "entry count mismatch: header declares " + std::to_string(declared) + ", file holds " +
                     std::to_string(seen));
  } else {  // dense column-major; zeros are not stored; symmetric: the lower triangle
    const long long expected = sym ? rows * (rows + 1) / 2 : rows * cols;
    long long idx = 0, r = 0, c = 0;
    double v = 0.0;
    while (std::fscanf(fp, "%lf", &v) == 1) {
      if (idx >= expected) fail(path, "array has more values than the size line declares");
      if (!std::isfinite(v)) fail(path, "non-finite value in array data");
      long long rr = idx % rows, cc = idx / rows;
      if (sym) {
        rr = r;
        cc = c;
        if (++r >= rows) {
          ++c;
          r = c;
        }
      }
      if (v != 0.0) add(rr, cc, v);
      ++idx;
    }
    if (idx != expected)
      fail(path, "array holds " + std::to_string(idx) + " values, expected " + std::to_string(expected));
  }
  return csr_from_triplets(rows, cols, ri, ci, vv);
}

void save_csr(const HostCsr& m, const std::string& path) {
  FILE* fp = std::fopen(path.c_str(), "wb");
  if (fp == nullptr) throw RuntimeError("cannot write CSR cache: " + path);
  struct Closer {
    FILE* f;
    ~Closer() { std::fclose(f); }
  } closer{fp};
  Sha256 h;
  for_each_export_chunk(m, [&](const void* p, size_t n) { h.update(p, n); });
  const std::array<uint8_t, 32> digest = h.finish();
  const uint64_t head[4] = {static_cast<uint64_t>(m.n), static_cast<uint64_t>(m.f), static_cast<uint64_t>(m.nnz()),
                            m.val.empty() ? uint64_t{0} : uint64_t{1}};
  bool ok = std::fwrite("RMGCSR01", 1, 8, fp) == 8 && std::fwrite(head, 8, 4, fp) == 4 &&
            std::fwrite(digest.data(), 1, 32, fp) == 32;
  for_each_export_chunk(m, [&](const void* p, size_t n) { ok = ok && std::fwrite(p, 1, n, fp) == n; });
  if (!ok) throw RuntimeError("short write to CSR cache: " + path);
}

HostCsr load_csr(const std::string& path, bool verify, std::string* sha_hex) {
  FILE* fp = std::fopen(path.c_str(), "rb");
  if (fp == nullptr) throw RuntimeError("cannot open CSR cache: " + path);
  struct Closer {
    FILE* f;
    ~Closer() { std::fclose(f); }
  } closer{fp};
  char magic[8];
  uint64_t head[4];
  std::array<uint8_t, 32> digest{};
  if (std::fread(magic, 1, 8, fp) != 8 || std::memcmp(magic, "RMGCSR01", 8) != 0 || std::fread(head, 8, 4, fp) != 4 ||
      std::fread(digest.data(), 1, 32, fp) != 32)
    fail(path, "not a ridgemg_b200 CSR cache");
  HostCsr m;
  m.n = static_cast<int64_t>(head[0]);
  m.f = static_cast<int64_t>(head[1]);
  const size_t nnz = head[2];
  std::vector<uint64_t> u(static_cast<size_t>(m.n) + 1);
  if (std::fread(u.data(), 8, u.size(), fp) != u.size()) fail(path, "truncated row offsets");
  m.ptr.assign(u.begin(), u.end());
  u.resize(nnz);
  if (nnz && std::fread(u.data(), 8, nnz, fp) != nnz) fail(path, "truncated column indices");
  m.idx.assign(u.begin(), u.end());
  std::vector<uint64_t>().swap(u);
  m.val.resize(nnz);  // a pattern's values are stored as 1.0 (the hashed bytes)
  if (nnz && std::fread(m.val.data(), 8, nnz, fp) != nnz) fail(path, "truncated values");
  if (head[3] == 0) m.val.clear();
  validate_csr(m);
  const std::string want = hex(digest);
  if (verify && csr_sha256(m) != want) fail(path, "SHA-256 mismatch: the cache is corrupt");
  if (sha_hex) *sha_hex = want;
  return m;
}

}  // namespace rmg
