// Hierarchy setup for dense X on the device (dense_setup.hpp).
//
// The reference's setup arithmetic is a set of ordered FP64 chains: a column
// norm or a k-means++ distance sums over the rows in increasing order, a Lloyd
// distance (feature j, prototype s) starts at ||p_s||^2 and adds
// ((x - p)^2 - p^2) row by row, a Gram entry adds products row by row.  Such a
// chain cannot be split, so the parallelism is across chains and the kernels
// are built around keeping every chain fed:
//   * k_col_chain: one warp runs 32 column chains (lane = column) over row
//     chunks that the whole CTA stages into a shared-memory ring with
//     cp.async (the chain is latency bound; the other warps only copy);
//   * k_pair_chain: a CTA owns a 16 x 32 tile of (column, prototype) or
//     (column, column) pairs, two chains per thread, and streams both operand
//     strips through a 4-stage cp.async ring (FP64-throughput bound);
//   * means and coarsening: one thread per (row, cluster), members of the
//     cluster in increasing feature order.
// Every product / difference / sum the host rounds separately is a separate
// __dmul_rn / __dsub_rn / __dadd_rn here (no FMA contraction).
#include <algorithm>
#include <climits>
#include <cmath>
#include <limits>
#include <stdexcept>
#include <string>
#include <vector>

#include "dense_setup.hpp"
#include "runtime.cuh"

namespace rmg {

namespace {

constexpr int kT = 256;

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(s), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

// ---------------------------------------------------------------- column chains
// OP 0: out[j] = sum_r x[r][j]^2              (norms: sqrt; ||p_s||^2: plain)
// OP 1: out[j] = sqrt(sum_r (x[r][j] - c[r])^2) (k-means++ distances to column c)
// x: fp32 or fp64 row-major with leading dimension ld (16-byte aligned rows).
constexpr int kCcRows = 128, kCcStages = 3;

template <int OP, bool FP32>
__global__ void __launch_bounds__(kT) k_col_chain(const void* x, int64_t ld, int64_t n, int64_t cols,
                                                  const double* c, double* out, int take_sqrt) {
  constexpr int esz = FP32 ? 4 : 8;
  constexpr int row_bytes = 32 * esz;      // one 32-column strip of a row
  constexpr int pieces = row_bytes / 16;   // 16-byte copies per row
  extern __shared__ __align__(16) unsigned char cc_smem[];
  unsigned char* ring = cc_smem;                                             // [stages][rows][row_bytes]
  double* cring = reinterpret_cast<double*>(cc_smem + kCcStages * kCcRows * row_bytes);  // [stages][rows]
  const int tid = threadIdx.x, lane = tid & 31;
  const int64_t c0 = static_cast<int64_t>(blockIdx.x) * 32;
  const int64_t nchunks = (n + kCcRows - 1) / kCcRows;
  const unsigned char* base = static_cast<const unsigned char*>(x);
  auto stage = [&](int64_t ch) {
    if (ch < nchunks) {
      const int st = static_cast<int>(ch % kCcStages);
      const int64_t r0 = ch * kCcRows;
      const int rows = static_cast<int>(static_cast<int64_t>(kCcRows) < n - r0 ? static_cast<int64_t>(kCcRows) : n - r0);
      for (int q = tid; q < rows * pieces; q += kT) {
        const int rr = q / pieces, pc = q % pieces;
        const int64_t col = c0 + pc * (16 / esz);
        if (col < cols)
          cp_async16(ring + (static_cast<size_t>(st) * kCcRows + rr) * row_bytes + pc * 16,
                     base + ((r0 + rr) * ld + col) * esz);
      }
      if (OP == 1)
        for (int q = tid; q < (rows + 1) / 2; q += kT)
          if (2 * q + 1 < rows || (rows & 1) == 0)
            cp_async16(cring + st * kCcRows + 2 * q, c + r0 + 2 * q);
          else
            cring[st * kCcRows + 2 * q] = c[r0 + 2 * q];  // odd tail: one plain load
    }
    cp_async_commit();
  };
  stage(0);
  stage(1);
  double acc = 0.0;
  for (int64_t ch = 0; ch < nchunks; ++ch) {
    stage(ch + 2);
    cp_async_wait<2>();
    __syncthreads();
    if (tid < 32) {
      const int st = static_cast<int>(ch % kCcStages);
      const int rows = static_cast<int>(static_cast<int64_t>(kCcRows) < n - ch * kCcRows ? static_cast<int64_t>(kCcRows) : n - ch * kCcRows);
      const unsigned char* tile = ring + static_cast<size_t>(st) * kCcRows * row_bytes;
      const double* cv = cring + st * kCcRows;
      for (int r = 0; r < rows; ++r) {
        const double v = FP32 ? static_cast<double>(reinterpret_cast<const float*>(tile + r * row_bytes)[lane])
                              : reinterpret_cast<const double*>(tile + r * row_bytes)[lane];
        if (OP == 0) {
          acc = __dadd_rn(acc, __dmul_rn(v, v));
        } else {
          const double d = __dsub_rn(v, cv[r]);
          acc = __dadd_rn(acc, __dmul_rn(d, d));
        }
      }
    }
    __syncthreads();
  }
  if (tid < 32 && c0 + lane < cols) out[c0 + lane] = take_sqrt ? sqrt(acc) : acc;
}

// Few rows (a sketch: n <= 256): one thread per column walks the rows itself --
// the same ordered chain, without the staging ring (whose 100 KB of shared memory
// per CTA made every k-means++ step of a 500 k-column sketch 50+ waves).
template <int OP, bool FP32>
__global__ void __launch_bounds__(kT) k_small_chain(const void* x, int64_t ld, int64_t n, int64_t cols,
                                                    const double* c, double* out, int take_sqrt) {
  const int64_t j = static_cast<int64_t>(blockIdx.x) * kT + threadIdx.x;
  if (j >= cols) return;
  double acc = 0.0;
  for (int64_t r = 0; r < n; ++r) {
    const double v = FP32 ? static_cast<double>(static_cast<const float*>(x)[r * ld + j])
                          : static_cast<const double*>(x)[r * ld + j];
    if (OP == 0) {
      acc = __dadd_rn(acc, __dmul_rn(v, v));
    } else {
      const double d = __dsub_rn(v, c[r]);
      acc = __dadd_rn(acc, __dmul_rn(d, d));
    }
  }
  out[j] = take_sqrt ? sqrt(acc) : acc;
}

template <int OP>
void col_chain(cudaStream_t s, const void* x, bool fp32, int64_t ld, int64_t n, int64_t cols, const double* c,
               double* out, bool take_sqrt) {
  if (cols <= 0) return;
  if (n <= 256) {
    const dim3 g(static_cast<unsigned>((cols + kT - 1) / kT));
    if (fp32)
      k_small_chain<OP, true><<<g, kT, 0, s>>>(x, ld, n, cols, c, out, take_sqrt ? 1 : 0);
    else
      k_small_chain<OP, false><<<g, kT, 0, s>>>(x, ld, n, cols, c, out, take_sqrt ? 1 : 0);
    RMG_CK(cudaGetLastError());
    return;
  }
  const size_t smem = static_cast<size_t>(kCcStages) * kCcRows * 32 * (fp32 ? 4 : 8) +
                      static_cast<size_t>(kCcStages) * kCcRows * sizeof(double);
  const dim3 grid(static_cast<unsigned>((cols + 31) / 32));
  if (fp32) {
    RMG_CK(cudaFuncSetAttribute(k_col_chain<OP, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    k_col_chain<OP, true><<<grid, kT, smem, s>>>(x, ld, n, cols, c, out, take_sqrt ? 1 : 0);
  } else {
    RMG_CK(cudaFuncSetAttribute(k_col_chain<OP, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    k_col_chain<OP, false><<<grid, kT, smem, s>>>(x, ld, n, cols, c, out, take_sqrt ? 1 : 0);
  }
  RMG_CK(cudaGetLastError());
}

// ---------------------------------------------------------------- pair chains
// A CTA owns pairs (a, b) with a in [a0, a0 + 16), b in [b0, b0 + 32): warp w
// the rows a0 + w and a0 + w + 8, lane l the column b0 + l.  Both operand
// strips (16 and 32 fp64 columns of row-major A and B) stream through a
// cp.async ring.
// OP 0 (Lloyd, clustering.cpp:281-291 / host_setup.cpp:283-290):
//      acc = init[b];  acc += (x - p)^2 - p^2   (x = A[r][a], p = B[r][b])
// OP 1 (Gram, coarse_gram): acc = 0;  acc += A[r][a] * B[r][b]
// OP 2: OP 0 with the assignment's scan fused: per feature a, the tile's 32
//      prototypes reduce to the first minimum of max(acc, 0) (NaN never wins),
//      written as one (value, index) pair per (feature, prototype tile) --
//      F x K/32 pairs instead of the F x K distances (cfg 5: 12.5 GB, not 200 GB)
constexpr int kPcRows = 64, kPcStages = 4;

struct ArgMin {
  double v;
  long long s;
};

// first minimum in prototype order: strictly smaller value, or equal value and
// a smaller index (the reference's strict-< scan, clustering.cpp:292-302)
__device__ __forceinline__ ArgMin argmin_combine(ArgMin a, ArgMin b) {
  if (b.v < a.v || (b.v == a.v && b.s < a.s)) return b;
  return a;
}

__device__ __forceinline__ double lloyd_sq(double acc) {
  if (isnan(acc)) return INFINITY;  // std::max(NaN, 0) is NaN, never < best: like +inf here
  return acc < 0.0 ? 0.0 : acc;     // std::max(acc, 0.0)
}

template <int OP>
__global__ void __launch_bounds__(kT) k_pair_chain(const double* A, int64_t lda, int64_t na, const double* B,
                                                   int64_t ldb, int64_t nb, int64_t n, const double* init,
                                                   double* out, int64_t ldo) {
  extern __shared__ __align__(16) double pc_smem[];
  constexpr int stage_doubles = kPcRows * (16 + 32);
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int64_t a0 = static_cast<int64_t>(blockIdx.x) * 16, b0 = static_cast<int64_t>(blockIdx.y) * 32;
  const int64_t nchunks = (n + kPcRows - 1) / kPcRows;
  auto stage = [&](int64_t ch) {
    if (ch < nchunks) {
      double* sa = pc_smem + static_cast<size_t>(ch % kPcStages) * stage_doubles;
      double* sb = sa + kPcRows * 16;
      const int64_t r0 = ch * kPcRows;
      const int rows = static_cast<int>(static_cast<int64_t>(kPcRows) < n - r0 ? static_cast<int64_t>(kPcRows) : n - r0);
      // A strip: 8 pieces per row; B strip: 16 pieces per row
      for (int q = tid; q < rows * 24; q += kT) {
        const int rr = q / 24, pc = q % 24;
        if (pc < 8) {
          const int64_t col = a0 + 2 * pc;
          if (col < na) cp_async16(sa + rr * 16 + 2 * pc, A + (r0 + rr) * lda + col);
        } else {
          const int64_t col = b0 + 2 * (pc - 8);
          if (col < nb) cp_async16(sb + rr * 32 + 2 * (pc - 8), B + (r0 + rr) * ldb + col);
        }
      }
    }
    cp_async_commit();
  };
#pragma unroll
  for (int i = 0; i < kPcStages - 1; ++i) stage(i);
  const int64_t b = b0 + lane;
  double acc0 = 0.0, acc1 = 0.0;
  if ((OP == 0 || OP == 2) && b < nb) acc0 = acc1 = init[b];
  for (int64_t ch = 0; ch < nchunks; ++ch) {
    stage(ch + kPcStages - 1);
    cp_async_wait<kPcStages - 1>();
    __syncthreads();
    const double* sa = pc_smem + static_cast<size_t>(ch % kPcStages) * stage_doubles;
    const double* sb = sa + kPcRows * 16;
    const int rows = static_cast<int>(static_cast<int64_t>(kPcRows) < n - ch * kPcRows ? static_cast<int64_t>(kPcRows) : n - ch * kPcRows);
#pragma unroll 4
    for (int r = 0; r < rows; ++r) {
      const double x0 = sa[r * 16 + wid], x1 = sa[r * 16 + wid + 8], p = sb[r * 32 + lane];
      if (OP == 0 || OP == 2) {
        const double pp = __dmul_rn(p, p);
        const double d0 = __dsub_rn(x0, p), d1 = __dsub_rn(x1, p);
        acc0 = __dadd_rn(acc0, __dsub_rn(__dmul_rn(d0, d0), pp));
        acc1 = __dadd_rn(acc1, __dsub_rn(__dmul_rn(d1, d1), pp));
      } else {
        acc0 = __dadd_rn(acc0, __dmul_rn(x0, p));
        acc1 = __dadd_rn(acc1, __dmul_rn(x1, p));
      }
    }
    __syncthreads();
  }
  if constexpr (OP == 2) {
    ArgMin m0{b < nb ? lloyd_sq(acc0) : INFINITY, b < nb ? (long long)b : LLONG_MAX};
    ArgMin m1{b < nb ? lloyd_sq(acc1) : INFINITY, b < nb ? (long long)b : LLONG_MAX};
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      ArgMin t0{__shfl_xor_sync(0xffffffffu, m0.v, o), __shfl_xor_sync(0xffffffffu, m0.s, o)};
      ArgMin t1{__shfl_xor_sync(0xffffffffu, m1.v, o), __shfl_xor_sync(0xffffffffu, m1.s, o)};
      m0 = argmin_combine(m0, t0);
      m1 = argmin_combine(m1, t1);
    }
    ArgMin* tiles = reinterpret_cast<ArgMin*>(out);  // [na][gridDim.y]
    if (lane == 0) {
      if (a0 + wid < na) tiles[(a0 + wid) * gridDim.y + blockIdx.y] = m0;
      if (a0 + wid + 8 < na) tiles[(a0 + wid + 8) * gridDim.y + blockIdx.y] = m1;
    }
  } else if (b < nb) {
    if (a0 + wid < na) out[(a0 + wid) * ldo + b] = acc0;
    if (a0 + wid + 8 < na) out[(a0 + wid + 8) * ldo + b] = acc1;
  }
}

// per feature: the tiles' minima in prototype order, strict < from (inf, 0)
__global__ void k_argmin_tiles(const ArgMin* tiles, int ny, int64_t f, int32_t* member, double* own) {
  const int64_t j = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (j >= f) return;
  int64_t best = 0;
  double best_sq = INFINITY;
  for (int y = 0; y < ny; ++y) {
    const ArgMin t = tiles[j * ny + y];
    if (t.v < best_sq) {
      best_sq = t.v;
      best = t.s;
    }
  }
  member[j] = static_cast<int32_t>(best);
  own[j] = best_sq;
}

template <int OP>
void pair_chain(cudaStream_t s, const double* A, int64_t lda, int64_t na, const double* B, int64_t ldb, int64_t nb,
                int64_t n, const double* init, double* out, int64_t ldo) {
  if (na <= 0 || nb <= 0) return;
  const size_t smem = static_cast<size_t>(kPcStages) * kPcRows * (16 + 32) * sizeof(double);
  RMG_CK(cudaFuncSetAttribute(k_pair_chain<OP>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  const dim3 grid(static_cast<unsigned>((na + 15) / 16), static_cast<unsigned>((nb + 31) / 32));
  k_pair_chain<OP><<<grid, kT, smem, s>>>(A, lda, na, B, ldb, nb, n, init, out, ldo);
  RMG_CK(cudaGetLastError());
}

// ---------------------------------------------------------------- elementwise
// out[r][j] = widen(x[r][j]) (/ norm[j] when norm != nullptr; zeros stay zero),
// columns [cols, ldo) zero
__global__ void k_make_cols(const void* x, int fp32, int64_t ld, int64_t n, int64_t cols, const double* norm,
                            double* out, int64_t ldo) {
  const int64_t total = n * ldo;
  for (int64_t q = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; q < total;
       q += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t r = q / ldo, j = q % ldo;
    double v = 0.0;
    if (j < cols) {
      v = fp32 ? static_cast<double>(static_cast<const float*>(x)[r * ld + j]) : static_cast<const double*>(x)[r * ld + j];
      if (norm != nullptr && v != 0.0) v = __ddiv_rn(v, norm[j]);
    }
    out[q] = v;
  }
}

// dst[r * ldd + s] = src[r * lds + j]  (a column of X into prototype s; k-means load_column)
__global__ void k_copy_col(const double* src, int64_t lds, int64_t j, int64_t n, double* dst, int64_t ldd, int64_t s) {
  for (int64_t r = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; r < n;
       r += static_cast<int64_t>(gridDim.x) * blockDim.x)
    dst[r * ldd + s] = src[r * lds + j];
}

// out[r][c] = (sum over members m of c, increasing: x[r][m] (* w[m])) (* scale[c]);
// means (host_setup.cpp:329-335): w = nullptr, scale = 1/size;
// coarsen (host_setup.cpp:424-452): w = weights, scale = nullptr.
template <bool FP32>
__global__ void k_cluster_rows(const void* x, int64_t ld, int64_t n, const int32_t* mptr, const int32_t* members,
                               int64_t nc, const double* w, const double* scale, double* out, int64_t ldo) {
  const int64_t total = n * ldo;
  for (int64_t q = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; q < total;
       q += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t r = q / ldo, c = q % ldo;
    double acc = 0.0;
    if (c < nc) {
      for (int32_t e = mptr[c]; e < mptr[c + 1]; ++e) {
        const int32_t m = members[e];
        const double v = FP32 ? static_cast<double>(static_cast<const float*>(x)[r * ld + m])
                              : static_cast<const double*>(x)[r * ld + m];
        acc = __dadd_rn(acc, w != nullptr ? __dmul_rn(v, w[m]) : v);
      }
      if (scale != nullptr) acc = __dmul_rn(acc, scale[c]);
    }
    out[q] = acc;
  }
}

int grid_for(int64_t total) {
  return static_cast<int>(std::max<int64_t>(1, std::min<int64_t>((total + kT - 1) / kT, 148 * 16)));
}

void cluster_rows(cudaStream_t s, const void* x, bool fp32, int64_t ld, int64_t n, const int32_t* mptr,
                  const int32_t* members, int64_t nc, const double* w, const double* scale, double* out, int64_t ldo) {
  const int g = grid_for(n * ldo);
  if (fp32)
    k_cluster_rows<true><<<g, kT, 0, s>>>(x, ld, n, mptr, members, nc, w, scale, out, ldo);
  else
    k_cluster_rows<false><<<g, kT, 0, s>>>(x, ld, n, mptr, members, nc, w, scale, out, ldo);
  RMG_CK(cudaGetLastError());
}

int64_t even(int64_t v) { return (v + 1) / 2 * 2; }

// sign of the sketch entry G[r][c]: splitmix64 of a counter, top bit
__device__ __forceinline__ bool sketch_negative(uint64_t seed, int64_t r, int c, int d) {
  uint64_t z = (seed ^ 0xC0FFEE5CE7C4ull) + static_cast<uint64_t>(r * d + c + 1) * 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  z ^= z >> 31;
  return (z >> 63) != 0;
}

// warp per feature j (a row of X^T), lane c < d: S[c][j] = sum over the feature's
// nonzeros (increasing sample order) of +-x (x / norm_j when normalising)
__global__ void k_sketch_sparse(const int32_t* __restrict__ ptr, const int32_t* __restrict__ idx,
                                const double* __restrict__ val, int64_t f, const double* __restrict__ norm, int d,
                                uint64_t seed, double* __restrict__ S, int64_t ldS, int64_t row0) {
  const int64_t j = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int c = threadIdx.x & 31;
  if (j >= f || c >= d) return;
  const double nj = norm != nullptr ? norm[j] : 1.0;
  double acc = 0.0;
  for (int32_t q = ptr[j]; q < ptr[j + 1]; ++q) {
    double x = val != nullptr ? val[q] : 1.0;
    if (norm != nullptr) x = __ddiv_rn(x, nj);
    acc = __dadd_rn(acc, sketch_negative(seed, row0 + idx[q], c, d) ? -x : x);
  }
  S[c * ldS + j] = acc;
}

// G (n x d, row-major) of +-1 for the dense sketch
__global__ void k_sketch_signs(int64_t n, int d, uint64_t seed, double* g, int64_t row0) {
  const int64_t total = n * d;
  for (int64_t q = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; q < total;
       q += static_cast<int64_t>(gridDim.x) * blockDim.x)
    g[q] = sketch_negative(seed, row0 + q / d, static_cast<int>(q % d), d) ? -1.0 : 1.0;
}

// S[c][j] = st[j][c]
__global__ void k_transpose_st(const double* st, int64_t f, int d, double* S, int64_t ldS) {
  const int64_t total = f * d;
  for (int64_t q = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; q < total;
       q += static_cast<int64_t>(gridDim.x) * blockDim.x)
    S[(q % d) * ldS + q / d] = st[q];
}

}  // namespace

void sketch_sparse_gpu(cudaStream_t s, const SparseDev& xt, const double* norm, int d, uint64_t seed, double* S,
                       int64_t ldS, int64_t row0) {
  if (d < 1 || d > 32) throw InvalidArgument("kmeans_sketch: sketch dimension outside [1, 32]");
  const int64_t f = xt.rows;
  if (f > 0) {
    k_sketch_sparse<<<static_cast<unsigned>((f * 32 + kT - 1) / kT), kT, 0, s>>>(xt.ptr, xt.idx, xt.val, f, norm, d,
                                                                                   seed, S, ldS, row0);
    RMG_CK(cudaGetLastError());
  }
  RMG_CK(cudaStreamSynchronize(s));
}

void sketch_dense_gpu(cudaStream_t s, const double* xc, int64_t n, int64_t f, int64_t ld, int d, uint64_t seed,
                      double* S, int64_t ldS, int64_t row0) {
  if (d < 1 || d > 32) throw InvalidArgument("kmeans_sketch: sketch dimension outside [1, 32]");
  const int64_t ldg = even(d);
  DBuf<double> g(static_cast<size_t>(std::max<int64_t>(1, n)) * ldg), st(static_cast<size_t>(std::max<int64_t>(1, f)) * d);
  RMG_CK(cudaMemsetAsync(g.get(), 0, g.size() * sizeof(double), s));
  if (ldg == d) {
    k_sketch_signs<<<grid_for(n * d), kT, 0, s>>>(n, d, seed, g.get(), row0);
  } else {  // odd d: fill a d-wide scratch, then pad rows to even width
    DBuf<double> g0(static_cast<size_t>(std::max<int64_t>(1, n)) * d);
    k_sketch_signs<<<grid_for(n * d), kT, 0, s>>>(n, d, seed, g0.get(), row0);
    RMG_CK(cudaMemcpy2DAsync(g.get(), ldg * sizeof(double), g0.get(), d * sizeof(double), d * sizeof(double), n,
                             cudaMemcpyDeviceToDevice, s));
    RMG_CK(cudaStreamSynchronize(s));
  }
  RMG_CK(cudaGetLastError());
  // st[j][c] = sum_r xc[r][j] * G[r][c], rows in order (products by +-1 are exact)
  pair_chain<1>(s, xc, ld, f, g.get(), ldg, d, n, nullptr, st.get(), d);
  k_transpose_st<<<grid_for(f * d), kT, 0, s>>>(st.get(), f, d, S, ldS);
  RMG_CK(cudaGetLastError());
  RMG_CK(cudaStreamSynchronize(s));
}

void dense_columns_f64(cudaStream_t s, const DenseDev& x, bool normalize, double* out, int64_t ldo) {
  DBuf<double> norm;
  if (normalize) {  // normalized_columns (host_setup.cpp:79-90)
    norm.alloc(std::max<int64_t>(1, x.cols));
    col_chain<0>(s, x.data, x.fp32 != 0, x.ld, x.rows, x.cols, nullptr, norm.get(), true);
  }
  k_make_cols<<<grid_for(x.rows * ldo), kT, 0, s>>>(x.data, x.fp32, x.ld, x.rows, x.cols, norm.get(), out, ldo);
  RMG_CK(cudaGetLastError());
  RMG_CK(cudaStreamSynchronize(s));
}

Clustering kmeans_dense_gpu(cudaStream_t s, const double* xc, int64_t n, int64_t f, int64_t ld, int64_t k,
                            uint64_t max_iters, uint64_t seed) {
  if (k <= 0 || k > f) throw InvalidArgument("kmeans: k outside [1, F]");
  const int64_t ldk = even(k);
  const int64_t ny = (k + 31) / 32;  // prototype tiles of the fused assignment
  DBuf<ArgMin> tiles(static_cast<size_t>(f) * ny);
  DBuf<double> proto(static_cast<size_t>(std::max<int64_t>(1, n)) * ldk), psq(ldk), dist(static_cast<size_t>(f)),
      own_d(f), colv(std::max<int64_t>(1, n)), inv_d(k);
  DBuf<int32_t> member_d(f), mptr_d(k + 1), members_d(f);
  RMG_CK(cudaMemsetAsync(proto.get(), 0, proto.size() * sizeof(double), s));
  auto load_column = [&](int64_t j, int64_t slot) {
    k_copy_col<<<grid_for(n), kT, 0, s>>>(xc, ld, j, n, proto.get(), ldk, slot);
    RMG_CK(cudaGetLastError());
  };

  // k-means++ seeding (host_setup.cpp:205-255): distances on the device, draws here
  std::vector<int64_t> chosen;
  {
    CounterRng rng(seed);
    chosen.push_back(static_cast<int64_t>(rng.next_index(f)));
    std::vector<char> used(f, 0);
    used[chosen[0]] = 1;
    std::vector<double> d2(f, std::numeric_limits<double>::infinity()), cum(f, 0.0);
    double* dh = nullptr;  // pinned: one D2H of F distances per seeding step
    RMG_CK(cudaMallocHost(&dh, static_cast<size_t>(f) * sizeof(double)));
    struct PinnedFree {
      double* p;
      ~PinnedFree() { cudaFreeHost(p); }
    } dh_free{dh};
    while (static_cast<int64_t>(chosen.size()) < k) {
      const int64_t last = chosen.back();
      k_copy_col<<<grid_for(n), kT, 0, s>>>(xc, ld, last, n, colv.get(), 1, 0);
      RMG_CK(cudaGetLastError());
      col_chain<1>(s, xc, false, ld, n, f, colv.get(), dist.get(), true);
      RMG_CK(cudaMemcpyAsync(dh, dist.get(), f * sizeof(double), cudaMemcpyDeviceToHost, s));
      RMG_CK(cudaStreamSynchronize(s));
      // one pass: the running total after every column (the reference's second scan re-adds
      // the same terms in the same order -- skipped zeros add nothing -- so its `run` at j is
      // cum[j] bit for bit), then the draw is the first j with u < cum[j]
      double total = 0.0;
      for (int64_t j = 0; j < f; ++j) {
        if (used[j]) {
          d2[j] = 0.0;
        } else {
          d2[j] = std::min(d2[j], dh[j] * dh[j]);
          total += d2[j];
        }
        cum[j] = total;
      }
      int64_t pick = -1;
      if (total > 0.0) {
        const double u = rng.next_double() * total;
        // cum is non-decreasing; the first j with u < cum[j] has d2[j] > 0 (cum rose there)
        const int64_t j = std::upper_bound(cum.begin(), cum.end(), u) - cum.begin();
        if (j < f) pick = j;
        for (int64_t q = f - 1; pick < 0 && q >= 0; --q)
          if (!used[q] && d2[q] > 0.0) pick = q;
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
  }
  for (int64_t sI = 0; sI < k; ++sI) load_column(chosen[sI], sI);

  // Lloyd (host_setup.cpp:276-336)
  Clustering out;
  std::vector<int32_t> mh(f);
  std::vector<int64_t> member(f, 0), previous, size(k);
  std::vector<double> own(f), inv(k);
  std::vector<int32_t> mptr(k + 1), members(f);
  for (uint64_t iter = 0; iter < std::max<uint64_t>(max_iters, 1); ++iter) {
    col_chain<0>(s, proto.get(), false, ldk, n, k, nullptr, psq.get(), false);
    pair_chain<2>(s, xc, ld, f, proto.get(), ldk, k, n, psq.get(), reinterpret_cast<double*>(tiles.get()), 0);
    k_argmin_tiles<<<static_cast<unsigned>((f + kT - 1) / kT), kT, 0, s>>>(tiles.get(), static_cast<int>(ny), f,
                                                                           member_d.get(), own_d.get());
    RMG_CK(cudaGetLastError());
    RMG_CK(cudaMemcpyAsync(mh.data(), member_d.get(), f * sizeof(int32_t), cudaMemcpyDeviceToHost, s));
    RMG_CK(cudaMemcpyAsync(own.data(), own_d.get(), f * sizeof(double), cudaMemcpyDeviceToHost, s));
    RMG_CK(cudaStreamSynchronize(s));
    for (int64_t j = 0; j < f; ++j) member[j] = mh[j];
    std::fill(size.begin(), size.end(), 0);
    for (int64_t j = 0; j < f; ++j) size[member[j]]++;
    for (int64_t sI = 0; sI < k; ++sI) {  // empty-cluster repair (clustering.cpp:303-321)
      if (size[sI] != 0) continue;
      int64_t far = -1;
      double far_sq = -1.0;
      for (int64_t j = 0; j < f; ++j)
        if (size[member[j]] > 1 && own[j] > far_sq) {
          far_sq = own[j];
          far = j;
        }
      if (far < 0) break;
      size[member[far]]--;
      member[far] = sI;
      size[sI] = 1;
      load_column(far, sI);
      own[far] = 0.0;
    }
    out.iterations = iter + 1;
    if (!previous.empty() && previous == member) {
      out.converged = true;
      break;
    }
    previous = member;
    // means: proto[r][s] = (sum over members of s in increasing feature order) * (1 / size)
    std::fill(mptr.begin(), mptr.end(), 0);
    for (int64_t j = 0; j < f; ++j) mptr[member[j] + 1]++;
    for (int64_t sI = 0; sI < k; ++sI) mptr[sI + 1] += mptr[sI];
    {
      std::vector<int32_t> fill(mptr.begin(), mptr.end() - 1);
      for (int64_t j = 0; j < f; ++j) members[fill[member[j]]++] = static_cast<int32_t>(j);
    }
    for (int64_t sI = 0; sI < k; ++sI) inv[sI] = 1.0 / static_cast<double>(size[sI]);
    mptr_d.upload(mptr.data(), mptr.size(), s);
    members_d.upload(members.data(), members.size(), s);
    inv_d.upload(inv.data(), inv.size(), s);
    cluster_rows(s, xc, false, ld, n, mptr_d.get(), members_d.get(), k, nullptr, inv_d.get(), proto.get(), ldk);
  }
  RMG_CK(cudaStreamSynchronize(s));
  out.labels = std::move(member);
  out.n_clusters = k;
  return out;
}

void coarsen_dense_gpu(cudaStream_t s, const DenseDev& x, const Aggregation& agg, double* out, int64_t ldc) {
  if (agg.n_fine != x.cols) throw InvalidArgument("coarsen: prolongation does not match the matrix features");
  DBuf<int32_t> mptr, members;
  DBuf<double> w;
  mptr.upload(agg.mptr.data(), agg.mptr.size(), s);
  members.upload(agg.members.data(), agg.members.size(), s);
  w.upload(agg.weight.data(), agg.weight.size(), s);
  cluster_rows(s, x.data, x.fp32 != 0, x.ld, x.rows, mptr.get(), members.get(), agg.n_coarse, w.get(), nullptr, out,
               ldc);
  RMG_CK(cudaStreamSynchronize(s));
}

std::vector<double> gram_dense_gpu(cudaStream_t s, const DenseDev& x) {
  if (x.fp32) throw InvalidArgument("gram_dense_gpu: fp64 storage expected");
  const int64_t m = x.cols;
  DBuf<double> g(static_cast<size_t>(std::max<int64_t>(1, m * m)));
  const double* a = static_cast<const double*>(x.data);
  pair_chain<1>(s, a, x.ld, m, a, x.ld, m, x.rows, nullptr, g.get(), m);
  std::vector<double> h(static_cast<size_t>(m) * m);
  if (!h.empty()) RMG_CK(cudaMemcpyAsync(h.data(), g.get(), h.size() * sizeof(double), cudaMemcpyDeviceToHost, s));
  RMG_CK(cudaStreamSynchronize(s));
  return h;
}

}  // namespace rmg
