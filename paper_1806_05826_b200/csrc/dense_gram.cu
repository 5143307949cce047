// Dense Gram matrices of coarse levels: assembly and application (dense_gram.cuh).
#include <algorithm>
#include <cstdlib>
#include <stdexcept>
#include <string>

#include "dense_gram.cuh"

namespace rmg {
namespace {

constexpr unsigned kFull = 0xffffffffu;

inline void check(const char* what) {
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) throw std::runtime_error(std::string(what) + ": " + cudaGetErrorString(e));
}

// One warp per feature i (row of G) and column tile [c0, c0 + width): the
// warp walks the rows r of X^T row i in increasing order; for each, its lanes
// take the row's nonzeros (distinct columns, so no two lanes touch the same
// accumulator) and add x_ri * x_rj into the warp's shared-memory tile.  Every
// entry therefore sums its products in increasing row order, each product and
// sum rounded separately -- coarse_gram's (and krylov.cpp:350-365's) order.
__global__ void k_gram_rows(const int32_t* __restrict__ xptr, const int32_t* __restrict__ xidx,
                            const double* __restrict__ xval, const int32_t* __restrict__ tptr,
                            const int32_t* __restrict__ tidx, const double* __restrict__ tval, int64_t n, int64_t c0,
                            int width, double* __restrict__ G, int64_t ldg) {
  extern __shared__ double acc_all[];
  const int warps = blockDim.x >> 5, warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  double* acc = acc_all + static_cast<size_t>(warp) * width;
  const int64_t c1 = c0 + width;
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * warps + warp; i < n; i += static_cast<int64_t>(gridDim.x) * warps) {
    for (int q = lane; q < width; q += 32) acc[q] = 0.0;
    __syncwarp();
    const int32_t b = tptr[i], e = tptr[i + 1];
    for (int32_t base = b; base < e; base += 32) {
      const int m = min(32, e - base);
      int32_t rb = 0, re = 0;
      double vp = 0.0;
      if (lane < m) {
        const int32_t r = tidx[base + lane];
        vp = tval != nullptr ? tval[base + lane] : 1.0;
        rb = xptr[r];
        re = xptr[r + 1];
      }
      // rows in groups of 8: the first 64 entries of every row of the group are loaded before
      // any is used (one memory latency per group instead of two per row -- the rows of a
      // 16 M-row level are TLB-cold), then added row by row in the same order as before
      constexpr int kRG = 8;
      for (int t0 = 0; t0 < m; t0 += kRG) {
        int32_t jj[kRG][2];
        double xx[kRG][2];
#pragma unroll
        for (int g = 0; g < kRG; ++g) {
          const int t = min(t0 + g, m - 1);
          const bool live = t0 + g < m;
          const int32_t s0 = __shfl_sync(kFull, rb, t), s1 = __shfl_sync(kFull, re, t);
#pragma unroll
          for (int u = 0; u < 2; ++u) {
            const int32_t q = s0 + 32 * u + lane;
            const bool ok = live && q < s1;
            jj[g][u] = ok ? xidx[q] : -1;
            xx[g][u] = ok ? (xval != nullptr ? xval[q] : 1.0) : 0.0;
          }
        }
#pragma unroll
        for (int g = 0; g < kRG; ++g) {
          if (t0 + g < m) {  // warp-uniform
            const int t = t0 + g;
            const double v = __shfl_sync(kFull, vp, t);
            const int32_t s0 = __shfl_sync(kFull, rb, t), s1 = __shfl_sync(kFull, re, t);
#pragma unroll
            for (int u = 0; u < 2; ++u) {
              const int32_t j = jj[g][u];
              if (j >= c0 && j < c1) acc[j - c0] = __dadd_rn(acc[j - c0], __dmul_rn(v, xx[g][u]));
            }
            for (int32_t q = s0 + 64 + lane; q < s1; q += 32) {  // rows longer than 64 entries
              const int32_t j = xidx[q];
              if (j >= c0 && j < c1) {
                const double xv = xval != nullptr ? xval[q] : 1.0;
                acc[j - c0] = __dadd_rn(acc[j - c0], __dmul_rn(v, xv));
              }
            }
            __syncwarp();
          }
        }
      }
    }
    double* out = G + i * ldg + c0;
    for (int q = lane; q < width; q += 32) out[q] = acc[q];
    __syncwarp();
  }
}

// y = G x + beta x: one warp per row, G streamed once (evict-first loads), x
// from L1/L2.  Fixed per-lane order and butterfly: deterministic.
template <bool VEC>
__global__ void __launch_bounds__(256) k_gram_gemv(const double* __restrict__ G, int64_t ldg,
                                                   const double* __restrict__ x, double beta, double* __restrict__ y,
                                                   int64_t n, const int32_t* __restrict__ done) {
  if (done != nullptr && *done) return;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * 8 + warp; i < n; i += static_cast<int64_t>(gridDim.x) * 8) {
    const double* g = G + i * ldg;
    double a0 = 0.0, a1 = 0.0;
    if (VEC) {
      const int64_t n2 = n & ~int64_t{1};
#pragma unroll 4
      for (int64_t j = 2 * lane; j < n2; j += 64) {
        const double2 gv = __ldcs(reinterpret_cast<const double2*>(g + j));
        const double2 xv = __ldg(reinterpret_cast<const double2*>(x + j));
        a0 = fma(gv.x, xv.x, a0);
        a1 = fma(gv.y, xv.y, a1);
      }
      if ((n & 1) && lane == 0) a0 = fma(__ldcs(g + n - 1), x[n - 1], a0);
    } else {
#pragma unroll 4
      for (int64_t j = lane; j < n; j += 32) a0 = fma(__ldcs(g + j), __ldg(x + j), a0);
    }
    double a = a0 + a1;
#pragma unroll
    for (int off = 16; off >= 1; off >>= 1) a += __shfl_xor_sync(kFull, a, off);
    if (lane == 0) y[i] = a + beta * x[i];
  }
}

// Y = G V + beta V for one 16-column chunk [col0, col0 + kc) of row-major
// n x ldv blocks.  A CTA owns 16 rows of G (4 per warp); V's rows are staged
// in shared memory 256 at a time (column-major, padded: conflict-free), and
// lane l accumulates the j = l (mod 32) terms of its warp's 4 x 16 outputs;
// a warp reduce-scatter leaves lane l with outputs 2l, 2l + 1.
constexpr int kGemmRows = 4, kGemmWarps = 4, kGemmJ = 256, kGemmK = 16, kVsLd = kGemmJ + 1;

__global__ void __launch_bounds__(kGemmWarps * 32, 2)
    k_gram_gemm(const double* __restrict__ G, int64_t ldg, const double* __restrict__ V, int ldv, int col0, int kc,
                double beta, double* __restrict__ Y, int64_t n) {
  __shared__ double vs[kGemmK * kVsLd];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t row0 = (static_cast<int64_t>(blockIdx.x) * kGemmWarps + warp) * kGemmRows;
  const double* grow[kGemmRows];
#pragma unroll
  for (int r = 0; r < kGemmRows; ++r) grow[r] = G + min(row0 + r, n - 1) * ldg;
  double acc[kGemmRows * kGemmK];
#pragma unroll
  for (int e = 0; e < kGemmRows * kGemmK; ++e) acc[e] = 0.0;
  for (int64_t j0 = 0; j0 < n; j0 += kGemmJ) {
    const int jn = static_cast<int>(n - j0 < kGemmJ ? n - j0 : int64_t{kGemmJ});
    __syncthreads();
    for (int e = threadIdx.x; e < kGemmJ * kGemmK; e += blockDim.x) {
      const int jj = e / kGemmK, q = e % kGemmK;
      vs[q * kVsLd + jj] = (jj < jn && q < kc) ? V[(j0 + jj) * ldv + col0 + q] : 0.0;
    }
    __syncthreads();
#pragma unroll 4
    for (int t = 0; t < kGemmJ / 32; ++t) {
      const int jj = lane + 32 * t;
      double g[kGemmRows];
#pragma unroll
      for (int r = 0; r < kGemmRows; ++r) g[r] = jj < jn ? __ldcs(grow[r] + j0 + jj) : 0.0;
#pragma unroll
      for (int q = 0; q < kGemmK; ++q) {
        const double v = vs[q * kVsLd + jj];
#pragma unroll
        for (int r = 0; r < kGemmRows; ++r) acc[r * kGemmK + q] = fma(g[r], v, acc[r * kGemmK + q]);
      }
    }
  }
  // reduce-scatter over the warp: stage `off` halves the live values
#pragma unroll
  for (int off = 16, cnt = kGemmRows * kGemmK / 2; off >= 1; off >>= 1, cnt >>= 1) {
    const bool upper = (lane & off) != 0;
#pragma unroll
    for (int e = 0; e < cnt; ++e) {
      const double send = upper ? acc[e] : acc[e + cnt];
      const double keep = upper ? acc[e + cnt] : acc[e];
      acc[e] = keep + __shfl_xor_sync(kFull, send, off);
    }
  }
  // lane l now holds flattened outputs 2l and 2l + 1 (row l / 8, columns 2(l % 8) + {0, 1})
  const int r = lane >> 3, q = (2 * lane) & (kGemmK - 1);
  const int64_t row = row0 + r;
  if (row < n) {
#pragma unroll
    for (int u = 0; u < 2; ++u)
      if (q + u < kc) {
        const int64_t o = row * ldv + col0 + q + u;
        Y[o] = acc[u] + beta * V[o];
      }
  }
}

// The same product on the FP64 tensor cores (DMMA, mma.sync.m8n8k4.f64): the
// dense multi-right-hand-side contraction of north-star's "tensor cores for the
// dense multi-RHS variant".  A CTA owns 64 rows of G (16 per warp: two 8-row
// m-tiles) x the 16-column chunk (two 8-column n-tiles); G's fragments are read
// straight from global memory (each warp load is 8 rows x one 32-byte sector,
// every byte used once), V is staged 64 rows at a time in shared memory
// (double-buffered) and shared by the 4 warps.  Fragment layouts (PTX ISA,
// m8n8k4 f64): A[l/4][l%4], B[l%4][l/4], C[l/4][2(l%4) + {0,1}].
constexpr int kDmWarps = 4, kDmRows = 16 * kDmWarps, kDmK = 64, kDmLd = 17, kGramSplitsMax = 16;

__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};\n"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

// Split K: blockIdx.y takes columns [kb, ke) of G; each split writes its own
// partial block P[split] (n x 16), summed in split order by k_gram_finish.
__global__ void __launch_bounds__(kDmWarps * 32)
    k_gram_gemm_dmma(const double* __restrict__ G, int64_t ldg, const double* __restrict__ V, int ldv, int col0,
                     int kc, int64_t n, int64_t kspan, double* __restrict__ P) {
  __shared__ double vs[2][kDmK * kDmLd];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t rbase = static_cast<int64_t>(blockIdx.x) * kDmRows + warp * 16;
  const int64_t kb = static_cast<int64_t>(blockIdx.y) * kspan, ke = min(n, kb + kspan);
  // this lane's A rows (one per m-tile), clamped in range; column lane % 4
  const int64_t ra0 = min(rbase + (lane >> 2), n - 1), ra1 = min(rbase + 8 + (lane >> 2), n - 1);
  const double* g0 = G + ra0 * ldg + (lane & 3);
  const double* g1 = G + ra1 * ldg + (lane & 3);
  double c[2][2][2] = {};  // [m-tile][n-tile][2]
  auto stage = [&](int buf, int64_t k0) {
    for (int e = threadIdx.x; e < kDmK * 16; e += kDmWarps * 32) {
      const int kk = e >> 4, q = e & 15;
      const int64_t kr = k0 + kk;
      vs[buf][kk * kDmLd + q] = (kr < ke && q < kc) ? V[kr * ldv + col0 + q] : 0.0;
    }
  };
  stage(0, kb);
  __syncthreads();
  int buf = 0;
  for (int64_t k0 = kb; k0 < ke; k0 += kDmK) {
    if (k0 + kDmK < ke) stage(buf ^ 1, k0 + kDmK);  // next chunk's V while this one is multiplied
    const double* vb = vs[buf];
#pragma unroll 4
    for (int kk = 0; kk < kDmK; kk += 4) {
      const int64_t kcol = k0 + kk + (lane & 3);
      const double a0 = kcol < ke ? __ldcs(g0 + k0 + kk) : 0.0;
      const double a1 = kcol < ke ? __ldcs(g1 + k0 + kk) : 0.0;
      const double b0 = vb[(kk + (lane & 3)) * kDmLd + (lane >> 2)];
      const double b1 = vb[(kk + (lane & 3)) * kDmLd + 8 + (lane >> 2)];
      dmma(c[0][0][0], c[0][0][1], a0, b0);
      dmma(c[0][1][0], c[0][1][1], a0, b1);
      dmma(c[1][0][0], c[1][0][1], a1, b0);
      dmma(c[1][1][0], c[1][1][1], a1, b1);
    }
    __syncthreads();
    buf ^= 1;
  }
  double* part = P + static_cast<int64_t>(blockIdx.y) * n * 16;
#pragma unroll
  for (int mt = 0; mt < 2; ++mt) {
    const int64_t row = rbase + 8 * mt + (lane >> 2);
    if (row >= n) continue;
#pragma unroll
    for (int nt = 0; nt < 2; ++nt)
      *reinterpret_cast<double2*>(part + row * 16 + 8 * nt + 2 * (lane & 3)) =
          make_double2(c[mt][nt][0], c[mt][nt][1]);
  }
}

// Y = sum over the splits, in split order, + beta V
__global__ void k_gram_finish(const double* __restrict__ P, int splits, const double* __restrict__ V, int ldv,
                              int col0, int kc, double beta, double* __restrict__ Y, int64_t n) {
  const int64_t total = n * kc;
  for (int64_t e = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; e < total;
       e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t row = e / kc;
    const int q = static_cast<int>(e - row * kc);
    double sum = 0.0;
    for (int sp = 0; sp < splits; ++sp) sum += P[(static_cast<int64_t>(sp) * n + row) * 16 + q];
    const int64_t o = row * ldv + col0 + q;
    Y[o] = sum + beta * V[o];
  }
}

// Warp per row; the row's (label, product) pairs staged in shared memory (rows
// longer than kCoarsenStage are read from global memory instead).  Lane e is the
// first occurrence of its label -> it sums that label's products in element
// (= fine column) order and writes at the label's rank among the row's labels.
constexpr int kCoarsenWarps = 8, kCoarsenStage = 256;

__global__ void __launch_bounds__(kCoarsenWarps * 32)
    k_coarsen_rows(const int32_t* __restrict__ xptr, const int32_t* __restrict__ xidx, const double* __restrict__ xval,
                   int64_t n, const int32_t* __restrict__ label, const double* __restrict__ weight,
                   int32_t* __restrict__ count, int32_t* __restrict__ cidx, double* __restrict__ cval) {
  __shared__ int32_t sl_all[kCoarsenWarps][kCoarsenStage];
  __shared__ double sp_all[kCoarsenWarps][kCoarsenStage];
  __shared__ unsigned char sf_all[kCoarsenWarps][kCoarsenStage];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  int32_t* sl = sl_all[warp];
  double* sp = sp_all[warp];
  unsigned char* sf = sf_all[warp];
  for (int64_t r = static_cast<int64_t>(blockIdx.x) * kCoarsenWarps + warp; r < n;
       r += static_cast<int64_t>(gridDim.x) * kCoarsenWarps) {
    const int32_t b = xptr[r], len = xptr[r + 1] - b;
    const bool staged = len <= kCoarsenStage;
    auto lab = [&](int e) { return staged ? sl[e] : label[xidx[b + e]]; };
    auto prod = [&](int e) {
      if (staged) return sp[e];
      const int32_t i = xidx[b + e];
      return __dmul_rn(xval != nullptr ? xval[b + e] : 1.0, weight[i]);
    };
    auto is_first = [&](int e) {  // no earlier entry of the row has e's label
      const int32_t t = lab(e);
      for (int u = 0; u < e; ++u)
        if (lab(u) == t) return false;
      return true;
    };
    if (staged) {
      for (int e = lane; e < len; e += 32) {
        const int32_t i = xidx[b + e];
        sl[e] = label[i];
        sp[e] = __dmul_rn(xval != nullptr ? xval[b + e] : 1.0, weight[i]);
      }
      __syncwarp();
      for (int e = lane; e < len; e += 32) sf[e] = is_first(e) ? 1 : 0;
    }
    __syncwarp();
    int distinct = 0;
    for (int e = lane; e < len; e += 32) {
      const int32_t s = lab(e);
      if (!(staged ? sf[e] != 0 : is_first(e))) continue;
      ++distinct;
      double acc = __dadd_rn(0.0, prod(e));  // the dense accumulator starts at 0.0
      int rank = 0;  // distinct labels of the row below s
      for (int q = 0; q < len; ++q) {
        const int32_t t = lab(q);
        if (q > e && t == s) acc = __dadd_rn(acc, prod(q));
        if (t < s && (staged ? sf[q] != 0 : is_first(q))) ++rank;
      }
      cidx[b + rank] = s;
      cval[b + rank] = acc;
    }
#pragma unroll
    for (int off = 16; off >= 1; off >>= 1) distinct += __shfl_xor_sync(kFull, distinct, off);
    if (lane == 0) count[r] = distinct;
    __syncwarp();
  }
}

}  // namespace

void coarsen_rows_gpu(cudaStream_t s, const int32_t* xptr, const int32_t* xidx, const double* xval, int64_t n,
                      const int32_t* label, const double* weight, int32_t* count, int32_t* cidx, double* cval) {
  if (n <= 0) return;
  const int grid = static_cast<int>(std::min<int64_t>((n + kCoarsenWarps - 1) / kCoarsenWarps, 148 * 16));
  k_coarsen_rows<<<grid, kCoarsenWarps * 32, 0, s>>>(xptr, xidx, xval, n, label, weight, count, cidx, cval);
  check("coarsen_rows");
}

void sparse_gram_gpu(cudaStream_t s, const int32_t* xptr, const int32_t* xidx, const double* xval,
                     const int32_t* tptr, const int32_t* tidx, const double* tval, int64_t n, double* G,
                     int64_t ldg) {
  if (n <= 0) return;
  const int tile = static_cast<int>(std::min<int64_t>(n, 6144));
  const int warps = std::max(1, std::min(16, (200 * 1024) / (tile * 8)));
  const size_t smem = static_cast<size_t>(warps) * tile * sizeof(double);
  cudaFuncSetAttribute(k_gram_rows, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
  const int64_t blocks_needed = (n + warps - 1) / warps;
  const int grid = static_cast<int>(std::min<int64_t>(blocks_needed, 148 * std::max(1, 16 / warps)));
  for (int64_t c0 = 0; c0 < n; c0 += tile) {
    const int width = static_cast<int>(std::min<int64_t>(tile, n - c0));
    k_gram_rows<<<grid, warps * 32, smem, s>>>(xptr, xidx, xval, tptr, tidx, tval, n, c0, width, G, ldg);
    check("gram_rows");
  }
}

void launch_gram_gemv(const double* G, int64_t ldg, const double* x, double beta, double* y, int64_t n,
                      const int32_t* done, cudaStream_t s) {
  if (n <= 0) return;
  const int grid = static_cast<int>(std::min<int64_t>((n + 7) / 8, 148 * 8));
  const bool vec = (ldg % 2 == 0) && (reinterpret_cast<uintptr_t>(G) % 16 == 0) &&
                   (reinterpret_cast<uintptr_t>(x) % 16 == 0);
  if (vec)
    k_gram_gemv<true><<<grid, 256, 0, s>>>(G, ldg, x, beta, y, n, done);
  else
    k_gram_gemv<false><<<grid, 256, 0, s>>>(G, ldg, x, beta, y, n, done);
  check("gram_gemv");
}

// ---------------------------------------------------------------------------
// G = X^T X of a dense row-major X (fp64 or fp32 storage, fp64 arithmetic) on the
// FP64 tensor cores: the "dense multi-right-hand-side / beta-sweep variant, where the
// operator becomes a dense contraction" of the north star.  A CTA owns one 64 x 64
// tile (ti <= tj) of G and one split of the rows; it stages 16 rows of the tile's two
// column strips at a time in shared memory (leading dimension 68: the A / B fragment
// reads of a half-warp hit 16 different bank pairs) while the previous 16 rows are
// multiplied; warp w computes the 32 x 32 quadrant (w / 2, w % 2): 4 x 4 DMMA tiles
// per 4-row step.  Split partials are summed in split order by k_syrk_finish, which
// also mirrors the tile into the lower triangle.
constexpr int kSyTile = 64, kSyKC = 16, kSyLd = 68, kSyThreads = 128, kSySplitsMax = 64;

template <bool F32>
__global__ void __launch_bounds__(kSyThreads)
    k_syrk_dmma(const void* __restrict__ X, int64_t ldx, int64_t rows, int cols, int64_t rows_per_split, int nt,
                double* __restrict__ P) {
  __shared__ double sa[2][kSyKC * kSyLd], sb[2][kSyKC * kSyLd];
  // tile (ti, tj), ti <= tj, from the linear index (row-major over the upper triangle)
  int ti = 0, rem = blockIdx.x;
  while (rem >= nt - ti) {
    rem -= nt - ti;
    ++ti;
  }
  const int tj = ti + rem;
  const int i0 = ti * kSyTile, j0 = tj * kSyTile;
  const int64_t r0 = static_cast<int64_t>(blockIdx.y) * rows_per_split, r1 = min(rows, r0 + rows_per_split);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, wm = (warp >> 1) * 32, wn = (warp & 1) * 32;
  auto ld = [&](int64_t r, int c) -> double {
    if (r >= r1 || c >= cols) return 0.0;
    return F32 ? static_cast<double>(__ldg(static_cast<const float*>(X) + r * ldx + c))
               : __ldg(static_cast<const double*>(X) + r * ldx + c);
  };
  double stage[16];
  auto fetch = [&](int64_t rr) {  // 16 rows x (64 + 64) columns: 16 elements per thread, coalesced
#pragma unroll
    for (int u = 0; u < 16; ++u) {
      const int e = threadIdx.x + u * kSyThreads, kk = e >> 7, c = e & 127;
      stage[u] = ld(rr + kk, c < 64 ? i0 + c : j0 + c - 64);
    }
  };
  auto put = [&](int buf) {
#pragma unroll
    for (int u = 0; u < 16; ++u) {
      const int e = threadIdx.x + u * kSyThreads, kk = e >> 7, c = e & 127;
      if (c < 64) sa[buf][kk * kSyLd + c]= stage[u]; else sb[buf][kk * kSyLd + c - 64] = stage[u];
    }
  };
  double acc[4][4][2] = {};
  int buf = 0;
  if (r0 < r1) {
    fetch(r0);
    put(0);
  }
  __syncthreads();
  for (int64_t rr = r0; rr < r1; rr += kSyKC) {
    const bool more = rr + kSyKC < r1;
    if (more) fetch(rr + kSyKC);  // in flight while this chunk is multiplied
    const double* a = sa[buf];
    const double* b = sb[buf];
#pragma unroll
    for (int k4 = 0; k4 < kSyKC; k4 += 4) {
      double af[4], bf[4];
#pragma unroll
      for (int t = 0; t < 4; ++t) {
        af[t] = a[(k4 + (lane & 3)) * kSyLd + wm + 8 * t + (lane >> 2)];
        bf[t] = b[(k4 + (lane & 3)) * kSyLd + wn + 8 * t + (lane >> 2)];
      }
#pragma unroll
      for (int mt = 0; mt < 4; ++mt)
#pragma unroll
        for (int nt2 = 0; nt2 < 4; ++nt2) dmma(acc[mt][nt2][0], acc[mt][nt2][1], af[mt], bf[nt2]);
    }
    if (more) put(buf ^ 1);
    __syncthreads();
    buf ^= 1;
  }
  double* part = P + (static_cast<int64_t>(blockIdx.y) * gridDim.x + blockIdx.x) * (kSyTile * kSyTile);
#pragma unroll
  for (int mt = 0; mt < 4; ++mt)
#pragma unroll
    for (int nt2 = 0; nt2 < 4; ++nt2)
      *reinterpret_cast<double2*>(part + (wm + 8 * mt + (lane >> 2)) * kSyTile + wn + 8 * nt2 + 2 * (lane & 3)) =
          make_double2(acc[mt][nt2][0], acc[mt][nt2][1]);
}

__global__ void k_syrk_finish(const double* __restrict__ P, int splits, int ntiles, int nt, int cols,
                              double* __restrict__ G, int64_t ldg) {
  int ti = 0, rem = blockIdx.x;
  while (rem >= nt - ti) {
    rem -= nt - ti;
    ++ti;
  }
  const int tj = ti + rem;
  for (int e = threadIdx.x; e < kSyTile * kSyTile; e += blockDim.x) {
    double sum = 0.0;
    for (int sp = 0; sp < splits; ++sp) sum += P[(static_cast<int64_t>(sp) * ntiles + blockIdx.x) * (kSyTile * kSyTile) + e];
    const int i = ti * kSyTile + e / kSyTile, j = tj * kSyTile + e % kSyTile;
    if (i < cols && j < cols) {
      G[static_cast<int64_t>(i) * ldg + j] = sum;
      G[static_cast<int64_t>(j) * ldg + i] = sum;
    }
  }
}

void syrk_dense_dmma(cudaStream_t s, const void* X, int fp32, int64_t ldx, int64_t rows, int64_t cols, double* G,
                     int64_t ldg) {
  if (cols <= 0) return;
  const int nt = static_cast<int>((cols + kSyTile - 1) / kSyTile), ntiles = nt * (nt + 1) / 2;
  // splits: enough CTAs for ~8 per SM, at least 512 rows each
  int splits = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>({int64_t{kSySplitsMax}, (148 * 8 + ntiles - 1) / ntiles,
                                                                         (rows + 511) / 512})));
  const int64_t rps = ((rows + splits - 1) / splits + kSyKC - 1) / kSyKC * kSyKC;
  splits = static_cast<int>(std::max<int64_t>(1, (rows + rps - 1) / std::max<int64_t>(1, rps)));
  double* P = nullptr;
  if (cudaMalloc(&P, static_cast<size_t>(splits) * ntiles * kSyTile * kSyTile * sizeof(double)) != cudaSuccess)
    throw std::runtime_error("syrk_dense_dmma: out of device memory");
  const dim3 grid(static_cast<unsigned>(ntiles), static_cast<unsigned>(splits));
  if (fp32)
    k_syrk_dmma<true><<<grid, kSyThreads, 0, s>>>(X, ldx, rows, static_cast<int>(cols), rps, nt, P);
  else
    k_syrk_dmma<false><<<grid, kSyThreads, 0, s>>>(X, ldx, rows, static_cast<int>(cols), rps, nt, P);
  k_syrk_finish<<<ntiles, 256, 0, s>>>(P, splits, ntiles, nt, static_cast<int>(cols), G, ldg);
  const cudaError_t e = cudaStreamSynchronize(s);
  cudaFree(P);
  if (e != cudaSuccess) throw std::runtime_error(std::string("syrk_dense_dmma: ") + cudaGetErrorString(e));
  check("syrk_dense");
}

// ---------------------------------------------------------------------------
// out (F x k) = X^T B for a dense X and k right-hand sides in ONE sweep of X (the rhs
// of a batched solve; 16 single-vector sweeps before): M = F, N = 16, K = rows on the
// FP64 tensor cores.  One persistent CTA per SM owns a contiguous row range and streams
// it through a 3-stage cp.async ring (X rows in their storage type, fp32 converted at
// the fragment load; the matching rows of B); warp w accumulates the columns
// [128 w, 128 w + 128) x 16 in registers (16 x 2 DMMA tiles); per-CTA partials are summed
// in CTA order by k_xtb_finish.  HBM-bound when the DMMA pipe keeps up (fp32 storage).
constexpr int kXbThreads = 256, kXbStages = 3, kXbLdB = 20;

__device__ __forceinline__ void xb_cp_async16(void* smem_dst, const void* gsrc) {
  const unsigned d = static_cast<unsigned>(__cvta_generic_to_shared(smem_dst));
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(d), "l"(gsrc) : "memory");
}

template <bool F32>
__global__ void __launch_bounds__(kXbThreads, 1)
    k_xtb_dmma(const void* __restrict__ X, int64_t ldx, int64_t rows, int cols, const double* __restrict__ Bt,
               int64_t rows_per_cta, double* __restrict__ P) {
  constexpr int KC = F32 ? 16 : 8;
  constexpr int ESZ = F32 ? 4 : 8;
  extern __shared__ __align__(16) unsigned char xb_sm[];
  const int cpad = (cols + 15) / 16 * 16;
  const int ldS = cpad + (F32 ? 8 : 4);  // elements: the 16 lanes of a fragment read hit 16 bank pairs
  const size_t xbytes = static_cast<size_t>(KC) * ldS * ESZ, sbytes = xbytes + KC * kXbLdB * 8;
  const int64_t r0 = static_cast<int64_t>(blockIdx.x) * rows_per_cta, r1 = min(rows, r0 + rows_per_cta);
  const int nchunks = r0 < r1 ? static_cast<int>((r1 - r0 + KC - 1) / KC) : 0;
  const int ppr = (cols * ESZ + 15) / 16;  // 16-byte pieces per row of X
  const unsigned char* xg = static_cast<const unsigned char*>(X);
  auto issue = [&](int c) {
    if (c < nchunks) {
      unsigned char* st = xb_sm + static_cast<size_t>(c % kXbStages) * sbytes;
      const int64_t rb = r0 + static_cast<int64_t>(c) * KC;
      for (int e = threadIdx.x; e < KC * ppr; e += kXbThreads) {
        const int kk = e / ppr, pc = e - kk * ppr;
        unsigned char* dst = st + (static_cast<size_t>(kk) * ldS * ESZ) + pc * 16;
        if (rb + kk < r1)
          xb_cp_async16(dst, xg + (rb + kk) * ldx * ESZ + static_cast<size_t>(pc) * 16);
        else
          *reinterpret_cast<uint4*>(dst) = make_uint4(0u, 0u, 0u, 0u);
      }
      for (int e = threadIdx.x; e < KC * 8; e += kXbThreads) {
        const int kk = e >> 3, pc = e & 7;
        unsigned char* dst = st + xbytes + (static_cast<size_t>(kk) * kXbLdB * 8) + pc * 16;
        if (rb + kk < r1)
          xb_cp_async16(dst, reinterpret_cast<const unsigned char*>(Bt + (rb + kk) * 16) + pc * 16);
        else
          *reinterpret_cast<uint4*>(dst) = make_uint4(0u, 0u, 0u, 0u);
      }
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  };
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  double acc[16][2][2] = {};
#pragma unroll
  for (int d = 0; d < kXbStages - 1; ++d) issue(d);
  for (int c = 0; c < nchunks; ++c) {
    asm volatile("cp.async.wait_group %0;" ::"n"(kXbStages - 2) : "memory");
    __syncthreads();  // chunk c landed for every thread; chunk c - 1's stage is free
    issue(c + kXbStages - 1);
    const unsigned char* st = xb_sm + static_cast<size_t>(c % kXbStages) * sbytes;
    const double* bs = reinterpret_cast<const double*>(st + xbytes);
#pragma unroll
    for (int k4 = 0; k4 < KC; k4 += 4) {
      const int kr = k4 + (lane & 3);
      const double b0 = bs[kr * kXbLdB + (lane >> 2)], b1 = bs[kr * kXbLdB + 8 + (lane >> 2)];
#pragma unroll
      for (int j = 0; j < 16; ++j) {
        const int f0 = (warp * 16 + j) * 8;
        if (f0 < cols) {  // warp-uniform
          const int f = f0 + (lane >> 2);
          double a;
          if (F32)
            a = static_cast<double>(reinterpret_cast<const float*>(st)[kr * ldS + f]);
          else
            a = reinterpret_cast<const double*>(st)[kr * ldS + f];
          if (f >= cols) a = 0.0;
          dmma(acc[j][0][0], acc[j][0][1], a, b0);
          dmma(acc[j][1][0], acc[j][1][1], a, b1);
        }
      }
    }
  }
  asm volatile("cp.async.wait_group 0;" ::: "memory");
  double* part = P + static_cast<int64_t>(blockIdx.x) * cpad * 16;
#pragma unroll
  for (int j = 0; j < 16; ++j) {
    const int f = (warp * 16 + j) * 8 + (lane >> 2);
    if (f < cpad) {
      *reinterpret_cast<double2*>(part + f * 16 + 2 * (lane & 3)) = make_double2(acc[j][0][0], acc[j][0][1]);
      *reinterpret_cast<double2*>(part + f * 16 + 8 + 2 * (lane & 3)) = make_double2(acc[j][1][0], acc[j][1][1]);
    }
  }
}

// out[f][c0 + q] = the CTA partials summed in CTA order
__global__ void k_xtb_finish(const double* __restrict__ P, int ncta, int cols, int cpad, int k, int c0, int kc,
                             double* __restrict__ out) {
  const int total = cols * kc;
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < total; e += gridDim.x * blockDim.x) {
    const int f = e / kc, q = e - f * kc;
    double sum = 0.0;
    for (int b = 0; b < ncta; ++b) sum += P[(static_cast<int64_t>(b) * cpad + f) * 16 + q];
    out[static_cast<int64_t>(f) * k + c0 + q] = sum;
  }
}

// Bt[r][q] = column c0 + q of the column-major block (k vectors of n), zero for q >= kc
__global__ void k_bcol2row16(const double* __restrict__ cm, int64_t n, int c0, int kc, double* __restrict__ bt) {
  const int64_t total = n * 16;
  for (int64_t e = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; e < total;
       e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t r = e >> 4;
    const int q = static_cast<int>(e & 15);
    bt[e] = q < kc ? cm[static_cast<int64_t>(c0 + q) * n + r] : 0.0;
  }
}

int64_t xtb_scratch(int64_t rows, int64_t cols) {
  const int64_t cpad = (cols + 15) / 16 * 16;
  return rows * 16 + 148 * 2 * cpad * 16;  // the row-major 16-column block of B + per-CTA partials
}

void launch_xtb_dmma(cudaStream_t s, const void* X, int fp32, int64_t ldx, int64_t rows, int64_t cols,
                     const double* b_cm, int k, double* out, double* scratch) {
  if (cols <= 0 || k <= 0) return;
  if (cols > 1024) throw std::runtime_error("xtb_dmma: at most 1024 columns");
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  sms = std::min(sms, 296);
  const int cpad = static_cast<int>((cols + 15) / 16 * 16);
  const int KC = fp32 ? 16 : 8, esz = fp32 ? 4 : 8;
  const size_t smem = static_cast<size_t>(kXbStages) * (static_cast<size_t>(KC) * (cpad + (fp32 ? 8 : 4)) * esz + KC * kXbLdB * 8);
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(k_xtb_dmma<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    cudaFuncSetAttribute(k_xtb_dmma<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    attr = true;
  }
  const int64_t rpc = ((rows + sms - 1) / sms + KC - 1) / KC * KC;
  const int ncta = static_cast<int>(std::max<int64_t>(1, (rows + rpc - 1) / std::max<int64_t>(1, rpc)));
  double* bt = scratch;
  double* P = scratch + rows * 16;
  for (int c0 = 0; c0 < k; c0 += 16) {
    const int kc = std::min(16, k - c0);
    k_bcol2row16<<<148 * 8, 256, 0, s>>>(b_cm, rows, c0, kc, bt);
    if (fp32)
      k_xtb_dmma<true><<<ncta, kXbThreads, smem, s>>>(X, ldx, rows, static_cast<int>(cols), bt, rpc, P);
    else
      k_xtb_dmma<false><<<ncta, kXbThreads, smem, s>>>(X, ldx, rows, static_cast<int>(cols), bt, rpc, P);
    k_xtb_finish<<<std::max(1, std::min(148 * 4, static_cast<int>((cols * kc + 255) / 256))), 256, 0, s>>>(
        P, ncta, static_cast<int>(cols), cpad, k, c0, kc, out);
  }
  check("xtb_dmma");
}

int64_t gram_gemm_scratch(int64_t n) { return static_cast<int64_t>(kGramSplitsMax) * n * 16; }

void launch_gram_gemm(const double* G, int64_t ldg, const double* V, double beta, double* Y, int64_t n, int k,
                      double* scratch, cudaStream_t s) {
  if (n <= 0 || k <= 0) return;
  static const bool cuda_cores = [] {
    const char* e = std::getenv("RMG_GRAM_GEMM");
    return e != nullptr && std::string(e) == "cuda";
  }();
  for (int c0 = 0; c0 < k; c0 += kGemmK) {
    const int kc = std::min(kGemmK, k - c0);
    if (cuda_cores) {  // CUDA-core FP64 variant (A/B comparisons)
      const int rows = kGemmRows * kGemmWarps;
      k_gram_gemm<<<static_cast<int>((n + rows - 1) / rows), kGemmWarps * 32, 0, s>>>(G, ldg, V, k, c0, kc, beta, Y,
                                                                                      n);
    } else {
      // split K so that the grid fills the GPU: ~8 CTAs (32 warps) per SM
      const int64_t tiles = (n + kDmRows - 1) / kDmRows;
      int splits = static_cast<int>(std::min<int64_t>(kGramSplitsMax, std::max<int64_t>(1, (148 * 8) / tiles)));
      int64_t kspan = ((n + splits - 1) / splits + kDmK - 1) / kDmK * kDmK;
      splits = static_cast<int>((n + kspan - 1) / kspan);
      k_gram_gemm_dmma<<<dim3(static_cast<unsigned>(tiles), static_cast<unsigned>(splits)), kDmWarps * 32, 0, s>>>(
          G, ldg, V, k, c0, kc, n, kspan, scratch);
      k_gram_finish<<<static_cast<int>(std::min<int64_t>(148 * 4, (n * kc + 255) / 256)), 256, 0, s>>>(
          scratch, splits, V, k, c0, kc, beta, Y, n);
    }
    check("gram_gemm");
  }
}

}  // namespace rmg
