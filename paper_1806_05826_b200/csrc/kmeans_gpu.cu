// k-means (clustering.cpp:189-355) on the GPU, labels bit-identical to the
// reference (and to host_setup.cpp's restatement):
//   * every floating-point operation the reference rounds separately is
//     rounded separately here (__dadd_rn / __dmul_rn / __dsub_rn: no FMA
//     contraction), in the reference's order;
//   * k-means++ seeding stays on the host (host_setup.cpp, threaded): it is a
//     sequence of fixed-order FP64 add chains, which B200 runs slower than a
//     host core (see the comment at the seeding call);
//   * Lloyd: one CTA per column, each thread owning prototypes s = tid + 256u
//     (u < 32): acc_s = ||p_s||^2 + sum over the column's rows in increasing
//     order of ((x - p)^2 - p^2); argmin of max(acc, 0) as the lexicographic
//     (value, index) minimum = the reference's strict-< scan;
//   * ||p_s||^2: one thread per prototype, rows in increasing order;
//   * means: one thread per sample row adds x into p[row][member[col]] over the
//     row's columns in increasing order (for a fixed (row, s) that is the
//     reference's column order), then p *= 1/size;
//   * empty-cluster repair and the convergence test: host, as the reference.
#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <cstring>
#include <limits>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include "kmeans_gpu.hpp"
#include "runtime.cuh"

namespace rmg {

namespace {

constexpr int kT = 256;
constexpr int kMaxPer = 32;  // prototypes per thread: K <= 8192

struct Cols {  // features as rows: column j of X (sample indices increasing)
  const int32_t* ptr;
  const int32_t* idx;
  const double* val;  // nullptr: 1.0
  int64_t f;
};
__device__ __forceinline__ double cval(const Cols& c, int64_t q) { return c.val ? c.val[q] : 1.0; }

// prototypes p[r * k + s] = column seeds[s]
__global__ void k_load_seeds(Cols c, const int32_t* seeds, int64_t k, double* proto) {
  for (int64_t s = blockIdx.x; s < k; s += gridDim.x) {
    const int64_t j = seeds[s];
    for (int64_t q = c.ptr[j] + threadIdx.x; q < c.ptr[j + 1]; q += blockDim.x) proto[(int64_t)c.idx[q] * k + s] = cval(c, q);
  }
}

// psq[s] = sum_r p[r][s]^2, rows in order
__global__ void k_psq(const double* proto, int64_t n, int64_t k, double* psq) {
  const int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= k) return;
  double acc = 0.0;
  int64_t r = 0;
  for (; r + 16 <= n; r += 16) {  // 16 independent loads ahead of the ordered adds
    double p[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) p[i] = proto[(r + i) * k + s];
#pragma unroll
    for (int i = 0; i < 16; ++i) acc = __dadd_rn(acc, __dmul_rn(p[i], p[i]));
  }
  for (; r < n; ++r) {
    const double p = proto[r * k + s];
    acc = __dadd_rn(acc, __dmul_rn(p, p));
  }
  psq[s] = acc;
}

// assignment: CTA per column j
__global__ void __launch_bounds__(kT) k_assign(Cols c, const double* proto, const double* psq, int64_t k,
                                               int32_t* member, double* own) {
  __shared__ int32_t srow[kT];
  __shared__ double sval[kT];
  __shared__ double bv[kT / 32];
  __shared__ int32_t bi[kT / 32];
  const int64_t j = blockIdx.x;
  const int tid = threadIdx.x;
  const int per = (int)((k + kT - 1) / kT);
  double acc[kMaxPer];
#pragma unroll
  for (int u = 0; u < kMaxPer; ++u) {
    const int64_t s = tid + (int64_t)u * kT;
    acc[u] = (u < per && s < k) ? psq[s] : 0.0;
  }
  const int64_t q0 = c.ptr[j], q1 = c.ptr[j + 1];
  for (int64_t base = q0; base < q1; base += kT) {
    const int cnt = (int)(q1 - base < kT ? q1 - base : kT);
    __syncthreads();
    if (tid < cnt) {
      srow[tid] = c.idx[base + tid];
      sval[tid] = cval(c, base + tid);
    }
    __syncthreads();
    for (int e = 0; e < cnt; ++e) {
      const double x = sval[e];
      const double* pr = proto + (int64_t)srow[e] * k;
#pragma unroll
      for (int u = 0; u < kMaxPer; ++u) {
        const int64_t s = tid + (int64_t)u * kT;
        if (u < per && s < k) {
          const double p = pr[s];
          const double diff = __dsub_rn(x, p);
          acc[u] = __dadd_rn(acc[u], __dsub_rn(__dmul_rn(diff, diff), __dmul_rn(p, p)));
        }
      }
    }
  }
  // argmin of max(acc, 0): strict < in increasing s == lexicographic (value, s) minimum
  double best = __longlong_as_double(0x7ff0000000000000LL);  // +inf
  int32_t bidx = 0x7fffffff;
#pragma unroll
  for (int u = 0; u < kMaxPer; ++u) {
    const int64_t s = tid + (int64_t)u * kT;
    if (u < per && s < k) {
      const double sq = fmax(acc[u], 0.0);
      if (sq < best) {
        best = sq;
        bidx = (int32_t)s;
      }
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const double ov = __shfl_xor_sync(0xffffffffu, best, o);
    const int32_t oi = __shfl_xor_sync(0xffffffffu, bidx, o);
    if (ov < best || (ov == best && oi < bidx)) {
      best = ov;
      bidx = oi;
    }
  }
  const int lane = tid & 31, wid = tid >> 5;
  if (lane == 0) {
    bv[wid] = best;
    bi[wid] = bidx;
  }
  __syncthreads();
  if (tid == 0) {
    double b = bv[0];
    int32_t i = bi[0];
    for (int w = 1; w < kT / 32; ++w)
      if (bv[w] < b || (bv[w] == b && bi[w] < i)) {
        b = bv[w];
        i = bi[w];
      }
    if (i == 0x7fffffff) {  // every distance NaN: the reference keeps best = 0 with +inf
      i = 0;
    }
    member[j] = i;
    own[j] = b;
  }
}

struct Rows {  // samples as rows (X itself): row r lists its columns in increasing order
  const int32_t* ptr;
  const int32_t* idx;
  const double* val;
  int64_t n;
};

// means: p[r][member[j]] += x over row r's columns in increasing order
__global__ void k_accumulate(Rows x, const int32_t* member, int64_t k, double* proto) {
  for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < x.n; r += (int64_t)gridDim.x * blockDim.x) {
    double* pr = proto + r * k;
    for (int64_t q = x.ptr[r]; q < x.ptr[r + 1]; ++q) {
      const int64_t s = member[x.idx[q]];
      pr[s] = __dadd_rn(pr[s], x.val ? x.val[q] : 1.0);
    }
  }
}

__global__ void k_scale(double* proto, int64_t total, int64_t k, const double* inv) {
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x)
    proto[e] = __dmul_rn(proto[e], inv[e % k]);
}

template <class T>
DBuf<T> upload_vec(const std::vector<T>& v, cudaStream_t s) {
  DBuf<T> d;
  d.upload(v.data(), v.size(), s);
  return d;
}

std::vector<int32_t> narrow32(const std::vector<int64_t>& v) {
  std::vector<int32_t> o(v.size());
  for (size_t i = 0; i < v.size(); ++i) o[i] = static_cast<int32_t>(v[i]);
  return o;
}

}  // namespace

bool kmeans_gpu_supported(int64_t n, int64_t f, int64_t k, int64_t nnz) {
  if (k <= 0 || k > static_cast<int64_t>(kMaxPer) * kT) return false;
  if (n > INT32_MAX || f > INT32_MAX || nnz > INT32_MAX) return false;
  size_t free_b = 0, total_b = 0;
  if (cudaMemGetInfo(&free_b, &total_b) != cudaSuccess) return false;
  const double need = static_cast<double>(n) * k * 8 + static_cast<double>(nnz) * 24 + (n + f) * 16.0;
  return need < 0.6 * static_cast<double>(free_b);
}

Clustering kmeans_gpu(cudaStream_t s, const HostCsr& cols, const HostCsr& rows, int64_t k, uint64_t max_iters,
                      uint64_t seed) {
  const int64_t f = cols.n, n = cols.f;
  if (k <= 0 || k > f) throw InvalidArgument("kmeans: k outside [1, F]");
  // columns (F x N) and rows (N x F) of the (possibly normalized) matrix
  DBuf<int32_t> cptr = upload_vec(narrow32(cols.ptr), s), cidx = upload_vec(narrow32(cols.idx), s);
  DBuf<int32_t> rptr = upload_vec(narrow32(rows.ptr), s), ridx = upload_vec(narrow32(rows.idx), s);
  DBuf<double> cval, rval;
  if (!cols.val.empty()) cval.upload(cols.val.data(), cols.val.size(), s);
  if (!rows.val.empty()) rval.upload(rows.val.data(), rows.val.size(), s);
  const Cols cd{cptr.get(), cidx.get(), cols.val.empty() ? nullptr : cval.get(), f};
  const Rows rd{rptr.get(), ridx.get(), rows.val.empty() ? nullptr : rval.get(), n};

  // ---- k-means++ seeding: host (kmeanspp_seed, threaded).  Its two ordered
  // passes per step (the running total and the draw scan) and every column's
  // merge distance are FP64 add chains in a fixed order; on B200 a dependent
  // FP64 add costs ~30 cycles, so the chains (up to ~90 k terms for a Zipf-hot
  // column on cfg 2) ran 2-8 ms per step on the device vs ~0.1 ms on a host
  // core (measured).
  const auto t_seed0 = std::chrono::steady_clock::now();
  const std::vector<int64_t> seeds = kmeanspp_seed(cols, k, seed, std::max(1u, std::thread::hardware_concurrency()));
  DBuf<int32_t> chosen = upload_vec(narrow32(seeds), s);
  if (std::getenv("RMG_KMEANS_LOG") != nullptr)
    std::fprintf(stderr, "[rmg kmeans] host seeding %.3f s\n",
                 std::chrono::duration<double>(std::chrono::steady_clock::now() - t_seed0).count());
  // ---- Lloyd
  DBuf<double> proto(static_cast<size_t>(std::max<int64_t>(1, n)) * k), psq(k), own(std::max<int64_t>(1, f)),
      inv(k);
  DBuf<int32_t> member(std::max<int64_t>(1, f));
  RMG_CK(cudaMemsetAsync(proto.get(), 0, proto.size() * sizeof(double), s));
  k_load_seeds<<<static_cast<int>(std::min<int64_t>(k, 65535)), 128, 0, s>>>(cd, chosen.get(), k, proto.get());
  const bool tlog = std::getenv("RMG_KMEANS_LOG") != nullptr;
  auto now = [&] {
    cudaStreamSynchronize(s);
    return std::chrono::steady_clock::now();
  };
  auto t_seed = now();
  double t_psq = 0, t_assign = 0, t_update = 0;
  Clustering out;
  std::vector<int32_t> mem(f), previous;
  std::vector<double> ownh(f);
  std::vector<int64_t> size(k);
  const int64_t total = n * k;
  for (uint64_t iter = 0; iter < std::max<uint64_t>(max_iters, 1); ++iter) {
    auto t0 = tlog ? now() : std::chrono::steady_clock::time_point{};
    k_psq<<<static_cast<int>((k + 127) / 128), 128, 0, s>>>(proto.get(), n, k, psq.get());
    auto t1 = tlog ? now() : t0;
    k_assign<<<static_cast<int>(f), kT, 0, s>>>(cd, proto.get(), psq.get(), k, member.get(), own.get());
    auto t2 = tlog ? now() : t0;
    if (tlog) {
      t_psq += std::chrono::duration<double>(t1 - t0).count();
      t_assign += std::chrono::duration<double>(t2 - t1).count();
    }
    RMG_CK(cudaGetLastError());
    RMG_CK(cudaMemcpyAsync(mem.data(), member.get(), f * sizeof(int32_t), cudaMemcpyDeviceToHost, s));
    RMG_CK(cudaMemcpyAsync(ownh.data(), own.get(), f * sizeof(double), cudaMemcpyDeviceToHost, s));
    RMG_CK(cudaStreamSynchronize(s));
    std::fill(size.begin(), size.end(), 0);
    for (int64_t j = 0; j < f; ++j) size[mem[j]]++;
    bool repaired = false;
    for (int64_t c = 0; c < k; ++c) {  // empty-cluster repair (clustering.cpp:303-321)
      if (size[c] != 0) continue;
      int64_t far = -1;
      double far_sq = -1.0;
      for (int64_t j = 0; j < f; ++j)
        if (size[mem[j]] > 1 && ownh[j] > far_sq) {
          far_sq = ownh[j];
          far = j;
        }
      if (far < 0) break;
      size[mem[far]]--;
      mem[far] = static_cast<int32_t>(c);
      size[c] = 1;
      ownh[far] = 0.0;
      repaired = true;
    }
    out.iterations = iter + 1;
    if (!previous.empty() && previous == mem) {
      out.converged = true;
      break;
    }
    previous = mem;
    if (repaired) member.upload(mem.data(), mem.size(), s);
    std::vector<double> invh(k);
    for (int64_t c = 0; c < k; ++c) invh[c] = 1.0 / static_cast<double>(size[c]);
    inv.upload(invh.data(), invh.size(), s);
    RMG_CK(cudaMemsetAsync(proto.get(), 0, proto.size() * sizeof(double), s));
    k_accumulate<<<static_cast<int>(std::min<int64_t>(148 * 16, (n + kT - 1) / kT)), kT, 0, s>>>(rd, member.get(), k,
                                                                                                 proto.get());
    k_scale<<<148 * 16, kT, 0, s>>>(proto.get(), total, k, inv.get());
    RMG_CK(cudaGetLastError());
    if (tlog) t_update += std::chrono::duration<double>(now() - t2).count();
  }
  if (tlog)
    std::fprintf(stderr, "[rmg kmeans] f=%lld n=%lld k=%lld iterations=%llu psq=%.3f assign=%.3f update=%.3f s\n",
                 (long long)f, (long long)n, (long long)k, (unsigned long long)out.iterations, t_psq, t_assign,
                 t_update);
  out.labels.assign(mem.begin(), mem.end());
  out.n_clusters = k;
  RMG_CK(cudaStreamSynchronize(s));
  return out;
}

}  // namespace rmg
