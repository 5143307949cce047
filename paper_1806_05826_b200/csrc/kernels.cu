// sm_100a kernels for the ridgemg_b200 solve path.  See kernels.cuh for the
// data layout and DESIGN.md §4 for the per-kernel roofline.
//
// All of this path is HBM/L2-bandwidth or latency bound integer-indexed fp64
// work (2 flops per nonzero), so it deliberately uses CUDA cores, coalesced
// index streams, read-only gathers and fixed-order reductions rather than
// tensor cores.
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <mutex>
#include <stdexcept>
#include <string>
#include <unordered_set>

#include "kernels.cuh"
#include "spmm_tma.cuh"

namespace rmg {

namespace {

constexpr int kThreads = 256;
constexpr int kWarps = kThreads / 32;

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

template <int W>
__device__ __forceinline__ double group_sum(double v) {
#pragma unroll
  for (int o = W / 2; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Fixed-tree block sum; the result is valid in thread 0.
__device__ __forceinline__ double block_sum(double v, double* sh) {
  v = warp_sum(v);
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  __syncthreads();
  if (lane == 0) sh[wid] = v;
  __syncthreads();
  double r = 0.0;
  if (wid == 0) {
    r = lane < (int)(blockDim.x >> 5) ? sh[lane] : 0.0;
    r = warp_sum(r);
  }
  return r;
}

// "Last block" detection for single-kernel grid reductions: every block's
// thread 0 publishes its slot before the ticket; the final arriver then owns
// all slots (threadFenceReduction pattern).  Deterministic: slots are summed
// in index order by the last block, whoever it is.
__device__ __forceinline__ bool grid_last(unsigned* ticket) {
  __shared__ unsigned s_last;
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    const unsigned t = atomicAdd(ticket, 1u);
    s_last = (t == gridDim.x - 1) ? 1u : 0u;
    if (s_last) {
      __threadfence();
      *ticket = 0u;  // ready for the next launch
    }
  }
  __syncthreads();
  return s_last != 0u;
}

// Sum `n` slots (stride `stride`, component `c`) in a fixed order with the
// whole block; result valid in thread 0.
__device__ __forceinline__ double sum_slots(const double* slots, int n, int stride, int c, double* sh) {
  double acc = 0.0;
  for (int i = threadIdx.x; i < n; i += blockDim.x) acc += __ldcg(slots + (size_t)i * stride + c);
  return block_sum(acc, sh);
}

__device__ __forceinline__ int ring_slot(const KrylovScalars* sc) { return sc->it % (sc->keep + 1); }

// Streamed (read-once) index / value loads bypass L1 allocation so the L1
// keeps the reused gather operand (v in K1, u in K2) instead of the stream.
__device__ __forceinline__ int ld_stream(const int32_t* p) {
  int v;
  asm("ld.global.nc.L1::no_allocate.b32 %0, [%1];" : "=r"(v) : "l"(p));
  return v;
}
__device__ __forceinline__ int ld_stream(const uint16_t* p) {
  unsigned short v;
  asm("ld.global.nc.L1::no_allocate.b16 %0, [%1];" : "=h"(v) : "l"(p));
  return (int)v;
}
__device__ __forceinline__ double ld_stream(const double* p) {
  double v;
  asm("ld.global.nc.L1::no_allocate.f64 %0, [%1];" : "=d"(v) : "l"(p));
  return v;
}
__device__ __forceinline__ uint4 ld_stream_u32x4(const void* p) {  // 16-byte aligned
  uint4 v;
  asm("ld.global.nc.L1::no_allocate.v4.u32 {%0, %1, %2, %3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p));
  return v;
}

// ------------------------------------------------------------------ K1: t = X v
// Row-parallel CSR gather; W lanes per row, two rows per lane group in flight
// and 4 elements per lane per round, so each thread keeps up to 8 index loads
// and 8 gathers outstanding (the first version was long-scoreboard bound at
// 1 TB/s, profiles/r1_ncu_summary.md).  Column indices are uint16 when F <=
// 65536 (half the index stream).  Warp-uniform trip counts keep the group
// reductions convergent.  Per-row order: lane-strided partials, xor tree.
// Column relabeling for K1: when the matrix's columns are
// renumbered by descending popularity, v is first gathered into that order
// (vperm[j] = v[inv[j]]) so the hot columns' gathers share L1 lines.
__global__ void __launch_bounds__(kThreads) k_vperm(const double* __restrict__ v_in, const int32_t* __restrict__ inv,
                                                    double* __restrict__ vperm, int64_t cols, const int32_t* done,
                                                    const KrylovScalars* sc, int ring_stride) {
  if (done != nullptr && *done) return;
  const double* v = v_in;
  if (sc != nullptr) {
    if (sc->done) return;
    v += (size_t)ring_slot(sc) * ring_stride;
  }
  for (int64_t j = (int64_t)blockIdx.x * kThreads + threadIdx.x; j < cols; j += (int64_t)gridDim.x * kThreads)
    vperm[j] = __ldg(v + inv[j]);
}

// K1 over SELL-32: one warp per 32-row slice, one lane per
// row, elements column-major inside the slice (every index load is one
// coalesced 128 B line).  Rows hold their elements in descending column
// popularity, so instruction j gathers the j-th most popular column of 32
// rows: the first instructions land on a handful of L1 lines instead of 32.
// Per-row sum: sequential in that order (deterministic).
// HOTV (relabeled columns): labels < n_hot -- the most popular columns -- are
// staged in SMEM once per persistent 1024-thread CTA (108 KB, one CTA per SM
// at 42 registers); the cold rest is gathered with L1::no_allocate.  Measured
// on the cfg 5 shard: 523 -> 484 us; two CTAs per SM (32 registers, U = 4 or
// spilling at U = 8) ran 864-870 us.
template <bool PAT, bool NARROW, bool HOTV = false, int NT = kThreads>
__global__ void __launch_bounds__(NT) k_spmv_sell(const int32_t* __restrict__ off,
                                                        const int32_t* __restrict__ srow,
                                                        const int32_t* __restrict__ slen,
                                                        const int32_t* __restrict__ idx,
                                                        const uint16_t* __restrict__ idx16,
                                                        const double* __restrict__ val,
                                                        const double* __restrict__ v_in, double* __restrict__ t,
                                                        int64_t n_slices, const int32_t* done,
                                                        const KrylovScalars* sc, int ring_stride, int n_hot = 0) {
  if (done != nullptr && *done) return;
  const double* __restrict__ v = v_in;
  if (sc != nullptr) {
    if (sc->done) return;
    v += (size_t)ring_slot(sc) * ring_stride;
  }
  extern __shared__ double vh[];
  if constexpr (HOTV) {
    for (int i = threadIdx.x; i < n_hot; i += NT) vh[i] = __ldcg(v + i);
    __syncthreads();
  }
  constexpr int U = HOTV ? 16 : 8;  // HOTV (1 CTA of 1024 per SM): deeper lookahead measured 478 -> 417 us
  const int lane = threadIdx.x & 31;
  const int64_t nwarps = ((int64_t)gridDim.x * NT) >> 5;
  for (int64_t sl = ((int64_t)blockIdx.x * NT + threadIdx.x) >> 5; sl < n_slices; sl += nwarps) {
    const int64_t base = off[sl];
    const int L = (off[sl + 1] - off[sl]) >> 5;
    const int row = srow[sl * 32 + lane];
    const int len = slen[sl * 32 + lane];
    double s = 0.0;
    for (int j = 0; j < L; j += U) {
      int c[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int64_t q = base + (int64_t)(j + u) * 32 + lane;
        c[u] = j + u < len ? (NARROW ? ld_stream(idx16 + q) : ld_stream(idx + q)) : -1;
      }
      double x[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        if constexpr (HOTV)
          x[u] = c[u] < 0 ? 0.0 : (c[u] < n_hot ? vh[c[u]] : ld_stream(v + c[u]));
        else
          x[u] = c[u] >= 0 ? __ldg(v + c[u]) : 0.0;
      }
#pragma unroll
      for (int u = 0; u < U; ++u)
        if (c[u] >= 0) s += PAT ? x[u] : ld_stream(val + base + (int64_t)(j + u) * 32 + lane) * x[u];
    }
    if (row >= 0) t[row] = s;
  }
}

// Software-pipelined SELL K1: the index batch of round j + 1 (or the first
// batch of the warp's next slice, whose header is also fetched a slice ahead)
// is in flight while round j's gathers are, so a round costs one memory
// latency instead of two (index load, then the dependent gather).  Same
// elements, same per-row order, same sums as k_spmv_sell.
template <bool PAT, bool NARROW, bool HOTV, int NT, int U>
__global__ void __launch_bounds__(NT) k_spmv_sell_pipe(const int32_t* __restrict__ off,
                                                       const int32_t* __restrict__ srow,
                                                       const int32_t* __restrict__ slen,
                                                       const int32_t* __restrict__ idx,
                                                       const uint16_t* __restrict__ idx16,
                                                       const double* __restrict__ val,
                                                       const double* __restrict__ v_in, double* __restrict__ t,
                                                       int64_t n_slices, const int32_t* done,
                                                       const KrylovScalars* sc, int ring_stride, int n_hot = 0) {
  if (done != nullptr && *done) return;
  const double* __restrict__ v = v_in;
  if (sc != nullptr) {
    if (sc->done) return;
    v += (size_t)ring_slot(sc) * ring_stride;
  }
  extern __shared__ double vh[];
  if constexpr (HOTV) {
    for (int i = threadIdx.x; i < n_hot; i += NT) vh[i] = __ldcg(v + i);
    __syncthreads();
  }
  const int lane = threadIdx.x & 31;
  const int64_t nwarps = ((int64_t)gridDim.x * NT) >> 5;
  int64_t sl = ((int64_t)blockIdx.x * NT + threadIdx.x) >> 5;
  if (sl >= n_slices) return;
  auto load_idx = [&](int (&c)[U], int64_t base, int j, int len) {
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t q = base + (int64_t)(j + u) * 32 + lane;
      c[u] = j + u < len ? (NARROW ? ld_stream(idx16 + q) : ld_stream(idx + q)) : -1;
    }
  };
  int64_t base = off[sl];
  int L = (off[sl + 1] - base) >> 5;
  int row = srow[sl * 32 + lane];
  int len = slen[sl * 32 + lane];
  int cn[U];
  load_idx(cn, base, 0, len);
  for (;;) {
    const int64_t nsl = sl + nwarps;
    const bool more = nsl < n_slices;
    int64_t nbase = 0;
    int nL = 0, nrow = -1, nlen = 0;
    if (more) {  // next slice's header, a slice ahead
      nbase = off[nsl];
      nL = (off[nsl + 1] - nbase) >> 5;
      nrow = srow[nsl * 32 + lane];
      nlen = slen[nsl * 32 + lane];
    }
    double s = 0.0;
    for (int j = 0; j < L; j += U) {
      int c[U];
#pragma unroll
      for (int u = 0; u < U; ++u) c[u] = cn[u];
      if (j + U < L)
        load_idx(cn, base, j + U, len);
      else if (more)
        load_idx(cn, nbase, 0, nlen);
      double x[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        if constexpr (HOTV)
          x[u] = c[u] < 0 ? 0.0 : (c[u] < n_hot ? vh[c[u]] : ld_stream(v + c[u]));
        else
          x[u] = c[u] >= 0 ? __ldg(v + c[u]) : 0.0;
      }
#pragma unroll
      for (int u = 0; u < U; ++u)
        if (c[u] >= 0) s += PAT ? x[u] : ld_stream(val + base + (int64_t)(j + u) * 32 + lane) * x[u];
    }
    if (L == 0 && more) load_idx(cn, nbase, 0, nlen);
    if (row >= 0) t[row] = s;
    if (!more) break;
    sl = nsl;
    base = nbase;
    L = nL;
    row = nrow;
    len = nlen;
  }
}

// K1 over row CSR (RMG_K1=csr diagnostics; the default is SELL-32 above).
// Tried in r1 and measured slower than SELL on cfg 2 and the cfg 5 shard
// (profiles/r1_operator.md): v staged in SMEM; a CSR-Adaptive variant (block
// products in SMEM, lane-per-row sums); the hottest columns in SMEM (halved
// occupancy); L1::evict_last for hot / no_allocate for cold columns.
template <int W, bool PAT, bool NARROW, int NT = kThreads>
__global__ void __launch_bounds__(NT) k_spmv_rows(const int32_t* __restrict__ ptr,
                                                  const int32_t* __restrict__ idx,
                                                  const uint16_t* __restrict__ idx16,
                                                  const double* __restrict__ val,
                                                  const double* __restrict__ v_in,
                                                  double* __restrict__ t, int64_t rows,
                                                  const int32_t* done,
                                                  const KrylovScalars* sc, int ring_stride) {
  if (done != nullptr && *done) return;
  const double* v = v_in;
  if (sc != nullptr) {
    if (sc->done) return;
    v += (size_t)ring_slot(sc) * ring_stride;
  }
  constexpr int G = 32 / W;  // rows per warp per pass
  constexpr int U = 4;       // elements per lane per round
  const int lane = threadIdx.x & (W - 1);
  const int grp = (threadIdx.x & 31) / W;
  const int64_t warp = ((int64_t)blockIdx.x * NT + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * NT) >> 5;
  const int64_t span = nwarps * G;
  for (int64_t rb = warp * G; rb < rows; rb += 2 * span) {
    const int64_t ra = rb + grp, rbb = rb + span + grp;
    const int a0 = ra < rows ? ld_stream(ptr + ra) : 0, a1 = ra < rows ? ld_stream(ptr + ra + 1) : 0;
    const int b0 = rbb < rows ? ld_stream(ptr + rbb) : 0, b1 = rbb < rows ? ld_stream(ptr + rbb + 1) : 0;
    double sa = 0.0, sb = 0.0;
    for (int ka = a0 + lane, kb = b0 + lane; ka < a1 || kb < b1; ka += U * W, kb += U * W) {
      int ca[U], cb[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int pa = ka + u * W, pb = kb + u * W;
        ca[u] = pa < a1 ? (NARROW ? ld_stream(idx16 + pa) : ld_stream(idx + pa)) : -1;
        cb[u] = pb < b1 ? (NARROW ? ld_stream(idx16 + pb) : ld_stream(idx + pb)) : -1;
      }
      double xa[U], xb[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        xa[u] = ca[u] >= 0 ? __ldg(v + ca[u]) : 0.0;
        xb[u] = cb[u] >= 0 ? __ldg(v + cb[u]) : 0.0;
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        if (ca[u] >= 0) sa += PAT ? xa[u] : ld_stream(val + ka + u * W) * xa[u];
        if (cb[u] >= 0) sb += PAT ? xb[u] : ld_stream(val + kb + u * W) * xb[u];
      }
    }
    sa = group_sum<W>(sa);
    sb = group_sum<W>(sb);
    if (lane == 0) {
      if (ra < rows) t[ra] = sa;
      if (rbb < rows) t[rbb] = sb;
    }
  }
}

// ------------------------------------------------------------------ block operator (cfg 3)
// Columns are processed in chunks of up to 16 (c0 .. c0 + kc) of row-major
// blocks with leading dimension k.
constexpr int kBlockCols = 16;

__global__ void __launch_bounds__(kThreads) k_vperm_block(const double* __restrict__ v, const int32_t* __restrict__ inv,
                                                          double* __restrict__ vp, int64_t cols, int k) {
  const int64_t total = cols * k;
  for (int64_t e = (int64_t)blockIdx.x * kThreads + threadIdx.x; e < total; e += (int64_t)gridDim.x * kThreads) {
    const int64_t j = e / k, q = e - j * k;
    vp[e] = __ldg(v + (int64_t)inv[j] * k + q);
  }
}

// Volatile loads keep their program order among themselves: a batch of them
// issues back to back (nvcc otherwise interleaves each gather with its use).
__device__ __forceinline__ int ldv_s32(const int32_t* p) {
  int v;
  asm volatile("ld.global.nc.L1::no_allocate.s32 %0, [%1];" : "=r"(v) : "l"(p));
  return v;
}
__device__ __forceinline__ int ldv_u16(const uint16_t* p) {
  unsigned short v;
  asm volatile("ld.global.nc.L1::no_allocate.u16 %0, [%1];" : "=h"(v) : "l"(p));
  return (int)v;
}
__device__ __forceinline__ double ldv_f64_stream(const double* p) {
  double v;
  asm volatile("ld.global.nc.L1::no_allocate.f64 %0, [%1];" : "=d"(v) : "l"(p));
  return v;
}
__device__ __forceinline__ double ldv_f64(const double* p) {
  double v;
  asm volatile("ld.global.nc.f64 %0, [%1];" : "=d"(v) : "l"(p));
  return v;
}

// T[row][c0 + q] = sum over the row's elements of x * V[col][c0 + q].  A
// half-warp per row, lane q owning column q: every gathered row of V is one
// coalesced access (2 lines per warp instruction), and each lane sums its
// column in the row's element order (the single-vector K1's order).  A warp
// walks its SELL slice two rows at a time; element loads run 4 ahead.
// HOT: the n_hot most popular labels' V rows (relabeled columns: labels in
// descending popularity, ~2/3 of the gathers on cfg 3) are staged once per
// persistent CTA in shared memory; only the rest is gathered from L1 / L2.
template <bool PAT, bool NARROW, bool HOT>
__global__ void __launch_bounds__(HOT ? 512 : kThreads, HOT ? 1 : 3) k_spmm_sell(const int32_t* __restrict__ off,
                                                        const int32_t* __restrict__ srow,
                                                        const int32_t* __restrict__ slen,
                                                        const int32_t* __restrict__ idx,
                                                        const uint16_t* __restrict__ idx16,
                                                        const double* __restrict__ val,
                                                        const double* __restrict__ V, double* __restrict__ T,
                                                        int64_t slice0, int64_t n_slices, int k, int c0, int kc,
                                                        int n_hot, int acc_in) {
  extern __shared__ double vs[];
  const int lane = threadIdx.x & 31, h = lane >> 4, q = lane & 15;
  const bool colq = q < kc;
  if (HOT) {
    for (int e = threadIdx.x; e < n_hot * 16; e += blockDim.x) {
      const int r = e >> 4, cq = e & 15;
      vs[e] = cq < kc ? __ldg(V + (int64_t)r * k + c0 + cq) : 0.0;
    }
    __syncthreads();
  }
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t sl = slice0 + (((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5); sl < slice0 + n_slices;
       sl += nwarps) {
    const int64_t base = off[sl];
    for (int p = 0; p < 16; ++p) {
      const int slot = 2 * p + h;
      const int row = srow[sl * 32 + slot];
      const int len = slen[sl * 32 + slot];
      const int lmax = max(len, __shfl_xor_sync(0xffffffffu, len, 16));
      double acc = 0.0;
      // lane q of the half-warp loads element j + q's index (and value) once;
      // shuffles hand the 16 indices to every lane, whose 16 row gathers are
      // then independent (the per-element broadcast loads compiled to one
      // dependent index -> gather pair at a time)
      const int qq = colq ? q : 0;
      const int src0 = lane & 16;
      // the next batch's index / value loads are issued before this batch's
      // gathers, so a batch costs one memory latency instead of two
      auto load = [&](int j, int& ci, double& xv) {
        const bool okq = j + q < len;
        const int64_t eq = okq ? base + (int64_t)(j + q) * 32 + slot : base + slot;
        ci = okq ? (NARROW ? (int)ld_stream(idx16 + eq) : ld_stream(idx + eq)) : -1;
        xv = PAT ? 1.0 : ld_stream(val + eq);
      };
      int ci_next;
      double x_next;
      load(0, ci_next, x_next);
      for (int j = 0; j < lmax; j += 16) {
        const int ciq = ci_next;
        const double xq = x_next;
        if (j + 16 < lmax) load(j + 16, ci_next, x_next);
        int c[16];
        double x[16], vv[16];
#pragma unroll
        for (int u = 0; u < 16; ++u) {
          c[u] = __shfl_sync(0xffffffffu, ciq, src0 | u);
          x[u] = PAT ? 1.0 : __shfl_sync(0xffffffffu, xq, src0 | u);
        }
#pragma unroll
        for (int u = 0; u < 16; ++u)
          vv[u] = (HOT && c[u] < n_hot) ? vs[(c[u] < 0 ? 0 : c[u]) * 16 + qq]
                                        : __ldg(V + (int64_t)(c[u] < 0 ? 0 : c[u]) * k + c0 + qq);
#pragma unroll
        for (int u = 0; u < 16; ++u) {
          const double add = acc + (PAT ? vv[u] : x[u] * vv[u]);
          acc = c[u] >= 0 ? add : acc;
        }
      }
      if (row >= 0 && colq) {  // acc_in: the hot entries' sum is already in T (k_spmm_hot)
        const int64_t o = (int64_t)row * k + c0 + q;
        T[o] = acc_in ? T[o] + acc : acc;
      }
    }
  }
}

// X^T pass over a block: a half-warp per unit of work, lane q owning column q,
// elements in order.  Units: the rows with <= 512 nonzeros in the sample chunk
// (whole rows, sorted by length so the two half-warps of a warp share a trip
// count), then the items of longer rows (segment partials for k_block_finish).
// Lane q loads element e + q of each 16-element batch once and shuffles hand
// the indices to every lane (16 independent T-row gathers); the next batch's
// loads are issued before this batch's gathers.
template <bool PAT>
__global__ void __launch_bounds__(kThreads, 3) k_xt_block(const int32_t* __restrict__ ptr, const int32_t* __restrict__ idx,
                                                       const double* __restrict__ val, BlockXtSchedule bs,
                                                       const double* __restrict__ T, const double* __restrict__ V,
                                                       double* __restrict__ out, double beta, int k, int c0, int kc,
                                                       int first, int last) {
  const int lane = threadIdx.x & 31, q = lane & 15, src0 = lane & 16;
  const bool colq = q < kc;
  const int64_t unit = ((int64_t)blockIdx.x * kThreads + threadIdx.x) >> 4;
  const int64_t n_units = (int64_t)bs.n_short + bs.n_items;
  if (((unit >> 1) << 1) >= n_units) return;  // both half-warps out of range: the whole warp
  const bool valid = unit < n_units;
  int row = 0, e0 = 0, e1 = 0, seg = -1;
  if (valid && unit >= bs.n_items) {  // the items of split rows (the longest units) go first
    row = bs.short_rows[unit - bs.n_items];
    e0 = bs.e_begin[row];
    e1 = bs.e_end[row];
  } else if (valid) {
    const int4 it = bs.items[unit];
    row = it.x;
    e0 = it.y;
    e1 = it.z;
    seg = it.w;
  }
  const int len = e1 - e0;
  const int lmax = max(len, __shfl_xor_sync(0xffffffffu, len, 16));
  auto load = [&](int j, int& ci, double& xv) {
    const bool ok = j + q < len;
    ci = ok ? ld_stream(idx + e0 + j + q) : -1;
    xv = (PAT || !ok) ? 1.0 : ld_stream(val + e0 + j + q);
  };
  int ci_next;
  double x_next;
  load(0, ci_next, x_next);
  double acc = 0.0;
  for (int j = 0; j < lmax; j += 16) {
    const int ci = ci_next;
    const double xv = x_next;
    if (j + 16 < lmax) load(j + 16, ci_next, x_next);
    int c[16];
    double x[16], tv[16];
#pragma unroll
    for (int u = 0; u < 16; ++u) {
      c[u] = __shfl_sync(0xffffffffu, ci, src0 | u);
      x[u] = PAT ? 1.0 : __shfl_sync(0xffffffffu, xv, src0 | u);
    }
#pragma unroll
    for (int u = 0; u < 16; ++u) tv[u] = (c[u] >= 0 && colq) ? __ldg(T + (int64_t)c[u] * k + c0 + q) : 0.0;
#pragma unroll
    for (int u = 0; u < 16; ++u)
      if (c[u] >= 0) acc += PAT ? tv[u] : x[u] * tv[u];
  }
  if (!colq || !valid) return;
  if (seg < 0) {  // chunks accumulate in chunk order; the last one adds beta V
    const int64_t o = (int64_t)row * k + c0 + q;
    double r = first ? acc : out[o] + acc;
    if (last && beta != 0.0) r = r + beta * V[o];  // beta = 0: V is never read (the X^T-only pass has none)
    out[o] = r;
  } else {
    bs.seg[(int64_t)seg * kBlockCols + q] = acc;
  }
}

// Hot part of K1: the H1 most popular labels' V rows (label order = vperm's) staged
// once per persistent CTA (16-byte chunks XOR-swizzled by label); a group of 4 lanes
// per row sums the row's hot entries (popularity order), lane g owning columns
// 4g .. 4g + 3, and writes T; the cold SELL pass then adds the rest.
template <bool PAT>
__global__ void __launch_bounds__(1024, 1) k_spmm_hot(BlockHotK1 h1, const double* __restrict__ Vp, int k, int c0,
                                                     int kc, int64_t r0, int64_t r1, double* __restrict__ T) {
  extern __shared__ double vs[];
  for (int e = threadIdx.x; e < h1.H1 * 16; e += blockDim.x) {
    const int r = e >> 4, q = e & 15;
    vs[r * 16 + ((((q >> 1) ^ r) & 7) << 1) + (q & 1)] = q < kc ? __ldg(Vp + (int64_t)r * k + c0 + q) : 0.0;
  }
  __syncthreads();
  const double2* __restrict__ vs2 = reinterpret_cast<const double2*>(vs);
  const int g = threadIdx.x & 3;
  const int64_t ngroups = (int64_t)gridDim.x * (blockDim.x >> 2);
  for (int64_t r = r0 + (((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 2); r < r1; r += ngroups) {
    const int e0 = h1.ptr[r], e1 = h1.ptr[r + 1];
    double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
    int e = e0;
    for (; e + 8 <= e1; e += 8) {
      int l[8];
      double x[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        l[u] = h1.lab[e + u];
        x[u] = PAT ? 1.0 : h1.val[e + u];
      }
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const double2 lo = vs2[l[u] * 8 + ((2 * g) ^ (l[u] & 7))], hi = vs2[l[u] * 8 + ((2 * g + 1) ^ (l[u] & 7))];
        a0 = PAT ? a0 + lo.x : fma(x[u], lo.x, a0);
        a1 = PAT ? a1 + lo.y : fma(x[u], lo.y, a1);
        a2 = PAT ? a2 + hi.x : fma(x[u], hi.x, a2);
        a3 = PAT ? a3 + hi.y : fma(x[u], hi.y, a3);
      }
    }
    for (; e < e1; ++e) {
      const int l = h1.lab[e];
      const double x = PAT ? 1.0 : h1.val[e];
      const double2 lo = vs2[l * 8 + ((2 * g) ^ (l & 7))], hi = vs2[l * 8 + ((2 * g + 1) ^ (l & 7))];
      a0 = PAT ? a0 + lo.x : fma(x, lo.x, a0);
      a1 = PAT ? a1 + lo.y : fma(x, lo.y, a1);
      a2 = PAT ? a2 + hi.x : fma(x, hi.x, a2);
      a3 = PAT ? a3 + hi.y : fma(x, hi.y, a3);
    }
    double* out = T + r * k + c0 + 4 * g;
    const double a[4] = {a0, a1, a2, a3};
#pragma unroll
    for (int u = 0; u < 4; ++u)
      if (4 * g + u < kc) out[u] = a[u];
  }
}

// ---- block passes over chunk-interleaved records (BlockK1v2 / BlockHot) ----
__device__ __forceinline__ double2 ldv_f64x2(const double* p) {
  double2 v;
  asm volatile("ld.global.nc.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "l"(p));
  return v;
}
__device__ __forceinline__ void cp_async16(void* smem_dst, const void* gsrc) {
  const unsigned d = static_cast<unsigned>(__cvta_generic_to_shared(smem_dst));
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(d), "l"(gsrc) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

// A record = 4 entries of each of a slice's 8 rows: int32 label[8][4], then (valued
// matrices) double value[8][4] -- 384 bytes (pattern: 128).  Every warp owns a
// contiguous run of records and streams it through a private shared-memory ring with
// cp.async (16 bytes per lane, kRingDepth records in flight), so the entry stream's
// DRAM latency is paid once per warp, not once per chunk; a group of 4 lanes reads its
// row's 4 labels / values of the current record as one 16-byte and two 16-byte
// shared loads (broadcast inside the group).
constexpr int kRecLab = 128;

// first slice in [a, b] whose first record is >= target (off ascending)
__device__ __forceinline__ int64_t first_slice_at(const int32_t* __restrict__ off, int64_t a, int64_t b, int64_t target) {
  while (a < b) {
    const int64_t m = (a + b) >> 1;
    if (off[m] < target) a = m + 1; else b = m;
  }
  return a;
}

// K1.  One persistent CTA per SM stages the H1 hottest labels' V rows
// (plus a zero row for padding) in shared memory, rows at their natural 128-byte
// stride.  A group of 4 lanes owns a row of X; lane g owns the 16-byte column pairs g
// and 4 + g.  Even groups read pair g first and 4 + g second, odd groups the other
// way round: the 8 lanes one shared-memory wavefront serves (two groups) cover all
// 32 banks whatever the two labels are -- no swizzle, no conflicts.  A slice's first
// nhot records hold hot labels only (shared memory), the rest cold labels (16-byte
// gathers from the label-ordered V in L2, 8 in flight per lane): the cold gathers of
// some warps overlap the shared-memory phase of others, and T is written once.
template <bool PAT, bool VEC, int THREADS, int D>
__global__ void __launch_bounds__(THREADS, 1) k_spmm_k1v3(BlockK1v2 h, const double* __restrict__ Vp, int k, int c0,
                                                         int kc, int64_t s0, int64_t s1, double* __restrict__ T) {
  constexpr int REC = PAT ? kRecLab : kRecLab + 256;
  constexpr int NS = D + 1;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  double* vs = reinterpret_cast<double*>(smem_raw);
  const int H1 = h.H1;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, g = lane & 3, i = lane >> 2;
  unsigned char* ring = smem_raw + (size_t)(H1 + 1) * 128 + (size_t)warp * NS * REC;
  // this warp's run of records: an equal share of the launch's records, whole slices
  const int W = gridDim.x * (THREADS / 32), w = blockIdx.x * (THREADS / 32) + warp;
  const int64_t r0 = h.off[s0], r1 = h.off[s1], R = r1 - r0;
  const int64_t sA = first_slice_at(h.off, s0, s1, r0 + R * w / W);
  const int64_t sB = w == W - 1 ? s1 : first_slice_at(h.off, s0, s1, r0 + R * (w + 1) / W);
  const int recA = sA < s1 ? h.off[sA] : (int)r1, recB = h.off[sB];
  const unsigned char* __restrict__ gsrc = reinterpret_cast<const unsigned char*>(h.rec);
  auto issue = [&](int rec) {
    if (rec < recB && lane < REC / 16) cp_async16(ring + (rec % NS) * REC + lane * 16, gsrc + (size_t)rec * REC + lane * 16);
    cp_async_commit();
  };
#pragma unroll
  for (int d = 0; d < D; ++d) issue(recA + d);
  for (int e = threadIdx.x; e < (H1 + 1) * 16; e += THREADS) {
    const int r = e >> 4, q = e & 15;
    vs[e] = (r < H1 && q < kc) ? __ldg(Vp + (int64_t)r * k + c0 + q) : 0.0;
  }
  __syncthreads();
  const double2* __restrict__ vs2 = reinterpret_cast<const double2*>(vs);
  const int cA = (i & 1) ? 4 + g : g, cB = (i & 1) ? g : 4 + g;
  const double* vA = Vp + c0 + 2 * cA;
  const double* vB = Vp + c0 + 2 * cB;
  int cur = recA;
  int n_end = 0, n_hot = 0, n_row = -1;  // the next slice's header, loaded one slice ahead
  if (sA < sB) {
    n_end = h.off[sA + 1];
    n_hot = h.nhot[sA];
    n_row = h.srow[sA * 8 + i];
  }
  for (int64_t sl = sA; sl < sB; ++sl) {
    const int e_end = n_end, e_hot = cur + n_hot, row = n_row;
    if (sl + 1 < sB) {
      n_end = h.off[sl + 2];
      n_hot = h.nhot[sl + 1];
      n_row = h.srow[(sl + 1) * 8 + i];
    }
    double a0 = 0.0, a1 = 0.0, b0 = 0.0, b1 = 0.0;
    for (; cur < e_end; ++cur) {
      cp_async_wait<D - 1>();
      __syncwarp();
      issue(cur + D);
      const unsigned char* slot = ring + (cur % NS) * REC;
      const int4 lc = *reinterpret_cast<const int4*>(slot + i * 16);
      double2 x0 = make_double2(1.0, 1.0), x1 = make_double2(1.0, 1.0);
      if (!PAT) {
        x0 = *reinterpret_cast<const double2*>(slot + kRecLab + i * 32);
        x1 = *reinterpret_cast<const double2*>(slot + kRecLab + i * 32 + 16);
      }
      double2 A0, B0, A1, B1, A2, B2, A3, B3;
      if (cur < e_hot) {  // labels < H1, padding = H1 (the zero row, value 0)
        A0 = vs2[lc.x * 8 + cA]; B0 = vs2[lc.x * 8 + cB]; A1 = vs2[lc.y * 8 + cA]; B1 = vs2[lc.y * 8 + cB];
        A2 = vs2[lc.z * 8 + cA]; B2 = vs2[lc.z * 8 + cB]; A3 = vs2[lc.w * 8 + cA]; B3 = vs2[lc.w * 8 + cB];
      } else {  // labels >= H1, padding = -1 (value 0; the gathered row is then discarded)
        const int64_t m0 = (int64_t)max(lc.x, 0) * k, m1 = (int64_t)max(lc.y, 0) * k;
        const int64_t m2 = (int64_t)max(lc.z, 0) * k, m3 = (int64_t)max(lc.w, 0) * k;
        if (VEC) {
          A0 = ldv_f64x2(vA + m0); B0 = ldv_f64x2(vB + m0); A1 = ldv_f64x2(vA + m1); B1 = ldv_f64x2(vB + m1);
          A2 = ldv_f64x2(vA + m2); B2 = ldv_f64x2(vB + m2); A3 = ldv_f64x2(vA + m3); B3 = ldv_f64x2(vB + m3);
        } else {
          const bool pa0 = 2 * cA < kc, pa1 = 2 * cA + 1 < kc, pb0 = 2 * cB < kc, pb1 = 2 * cB + 1 < kc;
          auto ldp = [&](const double* p, bool p0, bool p1) {
            return make_double2(p0 ? __ldg(p) : 0.0, p1 ? __ldg(p + 1) : 0.0);
          };
          A0 = ldp(vA + m0, pa0, pa1); B0 = ldp(vB + m0, pb0, pb1); A1 = ldp(vA + m1, pa0, pa1);
          B1 = ldp(vB + m1, pb0, pb1); A2 = ldp(vA + m2, pa0, pa1); B2 = ldp(vB + m2, pb0, pb1);
          A3 = ldp(vA + m3, pa0, pa1); B3 = ldp(vB + m3, pb0, pb1);
        }
        if (lc.x < 0) { A0 = make_double2(0.0, 0.0); B0 = A0; }
        if (lc.y < 0) { A1 = make_double2(0.0, 0.0); B1 = A1; }
        if (lc.z < 0) { A2 = make_double2(0.0, 0.0); B2 = A2; }
        if (lc.w < 0) { A3 = make_double2(0.0, 0.0); B3 = A3; }
      }
      if (PAT) {
        a0 += A0.x; a1 += A0.y; b0 += B0.x; b1 += B0.y;
        a0 += A1.x; a1 += A1.y; b0 += B1.x; b1 += B1.y;
        a0 += A2.x; a1 += A2.y; b0 += B2.x; b1 += B2.y;
        a0 += A3.x; a1 += A3.y; b0 += B3.x; b1 += B3.y;
      } else {
        a0 = fma(x0.x, A0.x, a0); a1 = fma(x0.x, A0.y, a1); b0 = fma(x0.x, B0.x, b0); b1 = fma(x0.x, B0.y, b1);
        a0 = fma(x0.y, A1.x, a0); a1 = fma(x0.y, A1.y, a1); b0 = fma(x0.y, B1.x, b0); b1 = fma(x0.y, B1.y, b1);
        a0 = fma(x1.x, A2.x, a0); a1 = fma(x1.x, A2.y, a1); b0 = fma(x1.x, B2.x, b0); b1 = fma(x1.x, B2.y, b1);
        a0 = fma(x1.y, A3.x, a0); a1 = fma(x1.y, A3.y, a1); b0 = fma(x1.y, B3.x, b0); b1 = fma(x1.y, B3.y, b1);
      }
    }
    if (row >= 0) {
      double* o = T + (int64_t)row * k + c0;
      if (VEC) {
        *reinterpret_cast<double2*>(o + 2 * cA) = make_double2(a0, a1);
        *reinterpret_cast<double2*>(o + 2 * cB) = make_double2(b0, b1);
      } else {
        if (2 * cA < kc) o[2 * cA] = a0;
        if (2 * cA + 1 < kc) o[2 * cA + 1] = a1;
        if (2 * cB < kc) o[2 * cB] = b0;
        if (2 * cB + 1 < kc) o[2 * cB + 1] = b1;
      }
    }
  }
  cp_async_wait<0>();
}

// Hot features: one CTA per sample block b stages T[bR .. bR + R) (16 columns) in
// shared memory once (rows at their 128-byte stride, row R zero), then sums the
// block's segments from it exactly as K1's hot phase does: a group of 4 lanes per
// segment, records streamed through per-warp cp.async rings, conflict-free reads.
constexpr int kHotBlkThreads = 512, kHotBlkDepth = 4;

template <bool PAT>
__global__ void __launch_bounds__(kHotBlkThreads, 1) k_xt_hotblk(BlockHot hb, const double* __restrict__ T, int k,
                                                                int c0, int kc, int64_t N) {
  constexpr int REC = PAT ? kRecLab : kRecLab + 256;
  constexpr int D = kHotBlkDepth, NS = D + 1;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  double* ts = reinterpret_cast<double*>(smem_raw);
  const int b = blockIdx.x;
  const int64_t s0 = (int64_t)b * hb.R;
  const int nb = (int)(N - s0 < (int64_t)hb.R ? N - s0 : (int64_t)hb.R);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, g = lane & 3, i = lane >> 2;
  unsigned char* ring = smem_raw + (size_t)(hb.R + 1) * 128 + (size_t)warp * NS * REC;
  const bool vec = kc == 16 && k == 16 && c0 == 0;  // the block's T rows are one contiguous run
  if (vec) {
    const unsigned char* src = reinterpret_cast<const unsigned char*>(T + s0 * 16);
    for (int e = threadIdx.x; e < nb * 8; e += kHotBlkThreads) cp_async16(smem_raw + (size_t)e * 16, src + (size_t)e * 16);
  }
  cp_async_commit();
  // this warp's run of the block's records
  const int64_t slA = hb.boff[b], slB = hb.boff[b + 1];
  constexpr int W = kHotBlkThreads / 32;
  const int64_t r0 = hb.off[slA], r1 = hb.off[slB], Rn = r1 - r0;
  const int64_t sA = first_slice_at(hb.off, slA, slB, r0 + Rn * warp / W);
  const int64_t sB = warp == W - 1 ? slB : first_slice_at(hb.off, slA, slB, r0 + Rn * (warp + 1) / W);
  const int recA = sA < slB ? hb.off[sA] : (int)r1, recB = hb.off[sB];
  const unsigned char* __restrict__ gsrc = reinterpret_cast<const unsigned char*>(hb.rec);
  auto issue = [&](int rec) {
    if (rec < recB && lane < REC / 16) cp_async16(ring + (rec % NS) * REC + lane * 16, gsrc + (size_t)rec * REC + lane * 16);
    cp_async_commit();
  };
#pragma unroll
  for (int d = 0; d < D; ++d) issue(recA + d);
  if (!vec)
    for (int e = threadIdx.x; e < nb * 16; e += kHotBlkThreads) {
      const int r = e >> 4, q = e & 15;
      ts[e] = q < kc ? __ldcg(T + (s0 + r) * k + c0 + q) : 0.0;
    }
  if (threadIdx.x < 16) ts[hb.R * 16 + threadIdx.x] = 0.0;
  cp_async_wait<D>();  // the T rows (the first group); the records stay in flight
  __syncthreads();
  const double2* __restrict__ ts2 = reinterpret_cast<const double2*>(ts);
  const int cA = (i & 1) ? 4 + g : g, cB = (i & 1) ? g : 4 + g;
  int cur = recA;
  int n_end = sA < sB ? hb.off[sA + 1] : 0;
  for (int64_t sl = sA; sl < sB; ++sl) {
    const int e_end = n_end;
    if (sl + 1 < sB) n_end = hb.off[sl + 2];
    double a0 = 0.0, a1 = 0.0, b0 = 0.0, b1 = 0.0;
    for (; cur < e_end; ++cur) {
      cp_async_wait<D - 1>();
      __syncwarp();
      issue(cur + D);
      const unsigned char* slot = ring + (cur % NS) * REC;
      const int4 lc = *reinterpret_cast<const int4*>(slot + i * 16);
      const double2 A0 = ts2[lc.x * 8 + cA], B0 = ts2[lc.x * 8 + cB], A1 = ts2[lc.y * 8 + cA], B1 = ts2[lc.y * 8 + cB];
      const double2 A2 = ts2[lc.z * 8 + cA], B2 = ts2[lc.z * 8 + cB], A3 = ts2[lc.w * 8 + cA], B3 = ts2[lc.w * 8 + cB];
      if (PAT) {
        a0 += A0.x; a1 += A0.y; b0 += B0.x; b1 += B0.y;
        a0 += A1.x; a1 += A1.y; b0 += B1.x; b1 += B1.y;
        a0 += A2.x; a1 += A2.y; b0 += B2.x; b1 += B2.y;
        a0 += A3.x; a1 += A3.y; b0 += B3.x; b1 += B3.y;
      } else {
        const double2 x0 = *reinterpret_cast<const double2*>(slot + kRecLab + i * 32);
        const double2 x1 = *reinterpret_cast<const double2*>(slot + kRecLab + i * 32 + 16);
        a0 = fma(x0.x, A0.x, a0); a1 = fma(x0.x, A0.y, a1); b0 = fma(x0.x, B0.x, b0); b1 = fma(x0.x, B0.y, b1);
        a0 = fma(x0.y, A1.x, a0); a1 = fma(x0.y, A1.y, a1); b0 = fma(x0.y, B1.x, b0); b1 = fma(x0.y, B1.y, b1);
        a0 = fma(x1.x, A2.x, a0); a1 = fma(x1.x, A2.y, a1); b0 = fma(x1.x, B2.x, b0); b1 = fma(x1.x, B2.y, b1);
        a0 = fma(x1.y, A3.x, a0); a1 = fma(x1.y, A3.y, a1); b0 = fma(x1.y, B3.x, b0); b1 = fma(x1.y, B3.y, b1);
      }
    }
    double* out = hb.part + ((size_t)sl * 8 + i) * 16;
    *reinterpret_cast<double2*>(out + 2 * cA) = make_double2(a0, a1);
    *reinterpret_cast<double2*>(out + 2 * cB) = make_double2(b0, b1);
  }
  cp_async_wait<0>();
}

// out[feat[h]] = the feature's partials summed + beta V: a CTA per hot feature, thread
// (s, q) sums every 64th partial of the (block, segment)-ordered list (8 loads in
// flight), the 64 sub-sums added in s order.
constexpr int kFoldSubs = 64;
__global__ void __launch_bounds__(kFoldSubs * 16) k_hot_fold(BlockHot hb, const double* __restrict__ V,
                                                            double* __restrict__ out, double beta, int k, int c0,
                                                            int kc) {
  __shared__ double sh[kFoldSubs][16];
  const int h = blockIdx.x, q = threadIdx.x & 15, sub = threadIdx.x >> 4;
  double sum = 0.0;
  const int j1 = hb.fptr[h + 1];
  for (int j = hb.fptr[h] + sub; j < j1; j += 8 * kFoldSubs) {
    int id[8];
    double pv[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) id[u] = j + u * kFoldSubs < j1 ? hb.fidx[j + u * kFoldSubs] : -1;
#pragma unroll
    for (int u = 0; u < 8; ++u) pv[u] = id[u] >= 0 ? __ldcg(hb.part + (size_t)id[u] * 16 + q) : 0.0;
#pragma unroll
    for (int u = 0; u < 8; ++u) sum += pv[u];
  }
  sh[sub][q] = sum;
  __syncthreads();
  if (sub == 0 && q < kc) {
    double tot = sh[0][q];
#pragma unroll 8
    for (int u = 1; u < kFoldSubs; ++u) tot += sh[u][q];
    const int64_t o = (int64_t)hb.feat[h] * k + c0 + q;
    out[o] = beta != 0.0 ? tot + beta * V[o] : tot;
  }
}

// rows split into several items: warp per row, lanes over the items
// (lane-strided, fixed order) + warp tree, for each column
__global__ void k_block_finish(BlockXtSchedule bs, const double* __restrict__ V, double* __restrict__ out,
                               double beta, int k, int c0, int kc, int first, int last) {
  const int lane = threadIdx.x & 31;
  const int64_t w = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (w >= bs.n_multi) return;
  const int4 m = bs.multi[w];
  for (int q = 0; q < kc; ++q) {
    double sum = 0.0;
    for (int g = lane; g < m.z; g += 32) sum += bs.seg[(int64_t)(m.y + g) * kBlockCols + q];
    sum = warp_sum(sum);
    if (lane == 0) {
      const int64_t o = (int64_t)m.x * k + c0 + q;
      double r = first ? sum : out[o] + sum;
      if (last && beta != 0.0) r = r + beta * V[o];
      out[o] = r;
    }
  }
}

// ------------------------------------------------------------------ K2 hot part (hybrid X^T pass)
constexpr int kHotThreads = 1024;  // 2 CTAs x 32 warps per SM: latency hiding for SMEM gathers
// One CTA per sample block b: t[b*B, b*B + B) is staged in SMEM (coalesced,
// once), then every hot row (b, h) gathers from SMEM instead of moving a 32 B
// L2 sector per nonzero.  Long rows (h < hA): a warp each; short rows: 8 lanes.
template <bool PAT>
__global__ void __launch_bounds__(kHotThreads) k_xt_hot(HotXtDev h, const double* __restrict__ t, const int32_t* done,
                                                     const KrylovScalars* sc) {
  if (done != nullptr && *done) return;
  if (sc != nullptr && sc->done) return;
  extern __shared__ double ts[];
  const int b = blockIdx.x;
  const int64_t s0 = (int64_t)b * h.B;
  const int nb = (int)(h.N - s0 < (int64_t)h.B ? h.N - s0 : (int64_t)h.B);
  for (int j = threadIdx.x; j < nb; j += kHotThreads) ts[j] = __ldcg(t + s0 + j);
  if (threadIdx.x == 0) ts[h.B] = 0.0;  // the padding entries' slot
  __syncthreads();
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int32_t* __restrict__ p = h.ptr + (size_t)b * h.H;
  double* __restrict__ out = h.partial + (size_t)b * h.H;
  for (int r = wid; r < h.hA; r += kHotThreads / 32) {  // long rows: warp per row
    const int k0 = p[r], k1 = p[r + 1];
    double acc = 0.0;
    if (PAT) {
      // 8 indices per 16-byte load (segments are padded to 8 and 16-byte aligned, padding ->
      // the zero slot), two loads in flight per lane: 4x the bytes in flight of 2-byte loads
      for (int k = k0 + 8 * lane; k < k1; k += 512) {
        const uint4 w0 = ld_stream_u32x4(h.idx16 + k);
        const bool two = k + 256 < k1;
        uint4 w1 = make_uint4(0u, 0u, 0u, 0u);
        if (two) w1 = ld_stream_u32x4(h.idx16 + k + 256);
        acc += ts[w0.x & 0xffffu]; acc += ts[w0.x >> 16]; acc += ts[w0.y & 0xffffu]; acc += ts[w0.y >> 16];
        acc += ts[w0.z & 0xffffu]; acc += ts[w0.z >> 16]; acc += ts[w0.w & 0xffffu]; acc += ts[w0.w >> 16];
        if (two) {
          acc += ts[w1.x & 0xffffu]; acc += ts[w1.x >> 16]; acc += ts[w1.y & 0xffffu]; acc += ts[w1.y >> 16];
          acc += ts[w1.z & 0xffffu]; acc += ts[w1.z >> 16]; acc += ts[w1.w & 0xffffu]; acc += ts[w1.w >> 16];
        }
      }
    } else
    for (int k = k0 + lane; k < k1; k += 128) {
      int c[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) c[u] = k + 32 * u < k1 ? ld_stream(h.idx16 + k + 32 * u) : -1;
#pragma unroll
      for (int u = 0; u < 4; ++u)
        if (c[u] >= 0) acc += PAT ? ts[c[u]] : ld_stream(h.val + k + 32 * u) * ts[c[u]];
    }
    acc = warp_sum(acc);
    if (lane == 0) out[r] = acc;
  }
  // short rows: 8 rows per warp, 4 lanes each, 4 index loads in flight per lane;
  // the next round's row bounds are loaded while the current round runs
  constexpr int G = 4, RPW = 32 / G, NW = kHotThreads / 32;
  const int gl = lane & (G - 1), gw = lane / G;
  const int step = NW * RPW;
  int r = h.hA + wid * RPW + gw;
  int nk0 = r < h.H ? p[r] : 0, nk1 = r < h.H ? p[r + 1] : 0;
  for (int r0 = h.hA + wid * RPW; r0 < h.H; r0 += step) {  // warp-uniform trip count
    const int k0 = nk0, k1 = nk1, rr = r;
    r += step;
    nk0 = r < h.H ? p[r] : 0;
    nk1 = r < h.H ? p[r + 1] : 0;
    double acc = 0.0;
    for (int k = k0 + gl; k < k1; k += 4 * G) {
      int c[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) c[u] = k + u * G < k1 ? ld_stream(h.idx16 + k + u * G) : -1;
#pragma unroll
      for (int u = 0; u < 4; ++u)
        if (c[u] >= 0) acc += PAT ? ts[c[u]] : ld_stream(h.val + k + u * G) * ts[c[u]];
    }
    acc = group_sum<G>(acc);
    if (gl == 0 && rr < h.H) out[rr] = acc;
  }
}

// Cross-block sums of the hot rows, fixed order: stage 1 sums chunk s of the
// blocks for each h (coalesced over h), stage 2 adds the S chunk sums in order.
__global__ void __launch_bounds__(kThreads) k_xt_hot_chunks(HotXtDev h, const int32_t* done, const KrylovScalars* sc) {
  if (done != nullptr && *done) return;
  if (sc != nullptr && sc->done) return;
  const int r = blockIdx.x * kThreads + threadIdx.x;
  if (r >= h.H) return;
  const int per = (h.nblk + h.S - 1) / h.S;
  const int b0 = blockIdx.y * per, b1 = min(h.nblk, b0 + per);
  double acc = 0.0;
#pragma unroll 8
  for (int b = b0; b < b1; ++b) acc += __ldcg(h.partial + (size_t)b * h.H + r);
  h.red2[(size_t)blockIdx.y * h.H + r] = acc;
}

__global__ void __launch_bounds__(kThreads) k_xt_hot_final(HotXtDev h, double* sums, const int32_t* done,
                                                           const KrylovScalars* sc) {
  if (done != nullptr && *done) return;
  if (sc != nullptr && sc->done) return;
  const int r = blockIdx.x * kThreads + threadIdx.x;
  if (r >= h.H) return;
  double acc = 0.0;
  for (int q = 0; q < h.S; ++q) acc += h.red2[(size_t)q * h.H + r];
  sums[h.feat[r]] = acc;
}

// ------------------------------------------------------------------ K2: X^T pass + epilogue
template <Epi E>
__device__ __forceinline__ void xt_epilogue(int col, double s, const XtArgs& a, const double* v,
                                            double* out, double& d0, double& d1) {
  if constexpr (E == Epi::Plain) {
    out[col] = s;
  } else if constexpr (E == Epi::Axpby) {
    out[col] = s + a.beta * v[col];
  } else if constexpr (E == Epi::Fcg) {
    const double pj = v[col];
    const double apj = s + a.beta * pj;
    out[col] = apj;
    d0 += pj * apj;
    d1 += pj * a.r[col];
  } else if constexpr (E == Epi::Cg) {
    const double pj = v[col];
    const double apj = s + a.beta * pj;
    out[col] = apj;
    d0 += pj * apj;
  } else if constexpr (E == Epi::Rich) {
    const double z1 = v[col];
    const double az1 = s + a.beta * z1;
    out[col] = z1 + a.omega * (a.r[col] - az1);
  } else {  // Gram
    out[col] = s;
    d0 += s * s;
  }
}

template <Epi E>
constexpr bool has_dots() {
  return E == Epi::Fcg || E == Epi::Cg || E == Epi::Gram;
}

// Scalar finalization of the dot-carrying epilogues (one thread).
template <Epi E>
__device__ __forceinline__ void xt_finalize(KrylovScalars* sc, double s0, double s1) {
  if constexpr (E == Epi::Fcg) {  // krylov.cpp:199-208
    sc->pap = s0;
    sc->pr = s1;
    if (s0 == 0.0) {
      sc->status = 1;
      sc->done = 1;
    } else if (s0 < 0.0) {
      sc->status = 2;
      sc->done = 1;
    } else {
      sc->alpha = s1 / s0;
      sc->pap_ring[ring_slot(sc)] = s0;
    }
  } else if constexpr (E == Epi::Cg) {  // krylov.cpp:126-134
    sc->pap = s0;
    if (!(s0 > 0.0)) {
      sc->status = 2;
      sc->done = 1;
    } else {
      sc->alpha = sc->rz / s0;
    }
  } else if constexpr (E == Epi::Gram) {  // lambda = ||A v|| (krylov.cpp:80-81)
    sc->lambda = sqrt(s0);
  }
}

// Sum of one X^T row (elements [k0, k1)) with `lanes` lanes, 8 elements per
// lane per round (independent loads in flight); lane-strided order.
template <bool PAT, bool NA = false>
__device__ __forceinline__ double xt_row_sum(const int32_t* __restrict__ idx, const double* __restrict__ val,
                                             const double* __restrict__ t, int k0, int k1, int lane, int lanes) {
  constexpr int U = 8;  // elements per lane per round (independent loads in flight)
  double s = 0.0;
  for (int k = k0 + lane; k < k1; k += U * lanes) {
    int c[U];
#pragma unroll
    for (int u = 0; u < U; ++u) c[u] = k + u * lanes < k1 ? ld_stream(idx + k + u * lanes) : -1;
    double x[U];
#pragma unroll
    for (int u = 0; u < U; ++u) x[u] = c[u] >= 0 ? (NA ? ld_stream(t + c[u]) : __ldg(t + c[u])) : 0.0;
#pragma unroll
    for (int u = 0; u < U; ++u)
      if (c[u] >= 0) s += PAT ? x[u] : ld_stream(val + k + u * lanes) * x[u];
  }
  return s;
}

// K2: one work item per CTA (see XtSchedule).  Short rows take W lanes, medium
// rows a full warp, long rows fixed CTA-wide segments combined in segment
// order by the last-arriving CTA.  The epilogue runs here.
template <int W, bool PAT, Epi E, bool NA = false>
__global__ void __launch_bounds__(kThreads) k_xt(const int32_t* __restrict__ ptr,
                                                 const int32_t* __restrict__ idx,
                                                 const double* __restrict__ val, XtSchedule sch,
                                                 XtArgs a) {
  if (a.done != nullptr && *a.done) return;
  const double* v = a.v;
  double* out = a.out;
  if constexpr (E == Epi::Fcg) {
    if (a.sc->done) return;
    const size_t off = (size_t)ring_slot(a.sc) * a.ring_stride;
    v += off;
    out += off;
  } else if constexpr (E == Epi::Cg) {
    if (a.sc->done) return;
  }
  __shared__ double sh[kWarps];
  __shared__ int s_fin;
  const double* __restrict__ t = a.t;
  const int4 item = sch.items[blockIdx.x];
  double d0 = 0.0, d1 = 0.0;
  if (item.z == -1 || item.z == -2) {
    const bool medium = item.z == -2;
    const int lanes = medium ? 32 : W;
    const int per_warp = 32 / lanes;
    const int lane = threadIdx.x & (lanes - 1);
    const int grp = (threadIdx.x & 31) / lanes;
    const int wid = threadIdx.x >> 5;
    for (int qb = item.x + wid * per_warp; qb < item.y; qb += kWarps * per_warp) {
      const int q = qb + grp;
      int vrow = -1;
      double s = 0.0;
      if (q < item.y) {
        vrow = sch.perm[q];
        s = xt_row_sum<PAT, NA>(idx, val, t, ptr[vrow], ptr[vrow + 1], lane, lanes);
      }
      if (medium) {
        s = warp_sum(s);
      } else {
        s = group_sum<W>(s);
      }
      if (vrow >= 0 && lane == 0) xt_epilogue<E>(vrow, s, a, v, out, d0, d1);
    }
    if constexpr (has_dots<E>()) {
      const double b0 = block_sum(d0, sh);
      const double b1 = (E == Epi::Fcg) ? block_sum(d1, sh) : 0.0;
      if (threadIdx.x == 0) {
        sch.slots[(size_t)item.w * 2] = b0;
        sch.slots[(size_t)item.w * 2 + 1] = b1;
      }
    }
  } else {
    // one fixed segment [item.y, item.z) of long row long_col[item.x]
    const int vrow = sch.long_col[item.x];
    double s = xt_row_sum<PAT, NA>(idx, val, t, item.y, item.z, threadIdx.x, kThreads);
    s = block_sum(s, sh);
    if (threadIdx.x == 0) {
      sch.seg_partial[item.w] = s;
      __threadfence();
      const unsigned tk = atomicAdd(sch.col_ticket + item.x, 1u);
      s_fin = (tk == (unsigned)sch.long_nseg[item.x] - 1u) ? 1 : 0;
      if (s_fin) {
        __threadfence();
        sch.col_ticket[item.x] = 0u;
        const int first = sch.long_first_seg[item.x], nseg = sch.long_nseg[item.x];
        double tot = 0.0;
        for (int q = 0; q < nseg; ++q) tot += __ldcg(sch.seg_partial + first + q);
        xt_epilogue<E>(vrow, tot, a, v, out, d0, d1);
        if constexpr (has_dots<E>()) {
          const int slot = sch.long_slot[item.x];
          sch.slots[(size_t)slot * 2] = d0;
          sch.slots[(size_t)slot * 2 + 1] = d1;
        }
      }
    }
  }
  if constexpr (has_dots<E>()) {
    if (grid_last(sch.grid_ticket)) {
      const double s0 = sum_slots(sch.slots, sch.n_slots, 2, 0, sh);
      const double s1 = (E == Epi::Fcg) ? sum_slots(sch.slots, sch.n_slots, 2, 1, sh) : 0.0;
      if (threadIdx.x == 0) xt_finalize<E>(a.sc, s0, s1);
    }
  }
}

// Epilogue pass over precomputed sums s_j (sharded: after the all-reduce;
// hybrid: hot + cold parts), with the deterministic dot reduction.
template <Epi E>
__global__ void __launch_bounds__(kThreads) k_xt_finish(XtSchedule sch, XtArgs a) {
  if (a.done != nullptr && *a.done) return;
  const double* v = a.v;
  double* out = a.out;
  if constexpr (E == Epi::Fcg) {
    if (a.sc->done) return;
    const size_t off = (size_t)ring_slot(a.sc) * a.ring_stride;
    v += off;
    out += off;
  } else if constexpr (E == Epi::Cg) {
    if (a.sc->done) return;
  }
  __shared__ double sh[kWarps];
  const int64_t F = sch.features;
  double d0 = 0.0, d1 = 0.0;
  for (int64_t j = (int64_t)blockIdx.x * kThreads + threadIdx.x; j < F; j += (int64_t)gridDim.x * kThreads) {
    xt_epilogue<E>((int)j, sch.partial[j], a, v, out, d0, d1);
  }
  if constexpr (has_dots<E>()) {
    const double b0 = block_sum(d0, sh);
    const double b1 = (E == Epi::Fcg) ? block_sum(d1, sh) : 0.0;
    if (threadIdx.x == 0) {
      sch.fin_slots[blockIdx.x * 2] = b0;
      sch.fin_slots[blockIdx.x * 2 + 1] = b1;
    }
    if (grid_last(sch.fin_ticket)) {
      const double s0 = sum_slots(sch.fin_slots, gridDim.x, 2, 0, sh);
      const double s1 = (E == Epi::Fcg) ? sum_slots(sch.fin_slots, gridDim.x, 2, 1, sh) : 0.0;
      if (threadIdx.x == 0) xt_finalize<E>(a.sc, s0, s1);
    }
  }
}

// ------------------------------------------------------------------ dense X
// One fused sweep: warp per row, lane l owns columns l + 32k.  MODE 0:
// t = x.v (warp tree), acc += t x; MODE 1: t = u_i given (X^T u); MODE 2:
// y_i = x.v only; MODE 3: acc += x^2 (Gram diagonal).  Warp partials are
// combined in warp order per CTA and stored column-major [col][cta] for the
// finishing kernel.  Row order per warp and every combine order are fixed.
// TMA 1D bulk copies (no tensor map: a row tile is one contiguous range) into
// a 3-stage SMEM ring, completion tracked by mbarriers.
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void tma_load_1d(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  uint32_t done = 0;
  while (!done) {
    asm volatile(
        "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
        : "=r"(done)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
  }
}

constexpr int kDenseStages = 3;
constexpr int kDenseTileBytes = 64 * 1024;

// Warp reduce-scatter of 16 per-lane row partials: afterwards lanes 2r and 2r + 1
// hold the warp sum of row r.  15 shuffles instead of 5 per row (80) for 16 warp
// trees; fixed order, deterministic.
__device__ __forceinline__ double warp_rows_sum16(double (&acc)[16]) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int w = 8, off = 16; w >= 1; w >>= 1, off >>= 1) {
    const bool hi = (lane & off) != 0;
#pragma unroll
    for (int k = 0; k < w; ++k) {
      const double send = hi ? acc[k] : acc[k + w];
      const double keep = hi ? acc[k + w] : acc[k];
      acc[k] = keep + __shfl_xor_sync(0xffffffffu, send, off);
    }
  }
  acc[0] += __shfl_xor_sync(0xffffffffu, acc[0], 1);
  return acc[0];
}

// One fused sweep: the CTA streams tiles of consecutive rows (<= 64 KB) through
// the SMEM ring; thread tid owns columns 4 tid .. 4 tid + 3 (v and the column
// partials live in its registers).  MODE 0: t_r = x_r . v (thread products,
// warp tree, then the kW warp sums in order), acc += t_r x_r; MODE 1: t_r =
// u_r; MODE 2: y_r = t_r only; MODE 3: acc += x_r^2.  Rows are consumed in
// increasing order per CTA; every combine order is fixed.
template <typename T, int MODE>
__global__ void __launch_bounds__(kThreads, 1) k_dense_ata(DenseDev d, const double* v_in, const double* u, double* y,
                                                           const int32_t* done, const KrylovScalars* sc,
                                                           int ring_stride) {
  if (done != nullptr && *done) return;
  const double* v = v_in;
  if (sc != nullptr) {
    if (sc->done) return;
    v += (size_t)ring_slot(sc) * ring_stride;
  }
  extern __shared__ __align__(128) unsigned char dsm_raw[];
  __shared__ __align__(8) uint64_t bar[kDenseStages];
  __shared__ double wdot[kWarps][16];
  __shared__ double trow[16];
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int64_t row_bytes = d.ld * (int64_t)sizeof(T);
  const int64_t tr_fit = kDenseTileBytes / row_bytes;
  const int TR = (int)(tr_fit < 16 ? tr_fit : 16);  // rows per tile
  const int64_t n_tiles = (d.rows + TR - 1) / TR;
  const int c0 = 4 * tid;
  const bool own = c0 < d.cols;
  constexpr bool DOT = MODE == 0 || MODE == 2;
  double vr[4] = {0.0, 0.0, 0.0, 0.0}, acc[4] = {0.0, 0.0, 0.0, 0.0};
  if (DOT && own)
#pragma unroll
    for (int q = 0; q < 4; ++q) vr[q] = c0 + q < d.cols ? __ldg(v + c0 + q) : 0.0;
  const unsigned char* X = static_cast<const unsigned char*>(d.data);
  auto tile_rows = [&](int64_t k) {
    const int64_t left = d.rows - k * TR;
    return (int)(left < TR ? left : TR);
  };
  auto issue = [&](int64_t k, int stage) {
    tma_load_1d(dsm_raw + (size_t)stage * kDenseTileBytes, X + k * TR * row_bytes,
                (uint32_t)(tile_rows(k) * row_bytes), &bar[stage]);
  };
  if (tid == 0) {
    for (int st = 0; st < kDenseStages; ++st) mbar_init(&bar[st], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  int64_t j = 0;  // local tile sequence
  if (tid == 0)
    for (int st = 0; st < kDenseStages; ++st) {
      const int64_t k = blockIdx.x + (int64_t)st * gridDim.x;
      if (k < n_tiles) issue(k, st);
    }
  for (int64_t k = blockIdx.x; k < n_tiles; k += gridDim.x, ++j) {
    const int st = (int)(j % kDenseStages);
    mbar_wait(&bar[st], (uint32_t)((j / kDenseStages) & 1));
    const T* tile = reinterpret_cast<const T*>(dsm_raw + (size_t)st * kDenseTileBytes);
    const int nr = tile_rows(k);
    const int64_t r0 = k * TR;
    // this thread's 4 columns of every tile row, vector loads (ld % 4 == 0, c0 % 4 == 0);
    // columns past F are zero padding in the stored rows
    double xs[16][4];
#pragma unroll
    for (int r = 0; r < 16; ++r) {
      if (r < nr && own) {
        if constexpr (sizeof(T) == 4) {
          const float4 q4 = *reinterpret_cast<const float4*>(tile + (size_t)r * d.ld + c0);
          xs[r][0] = q4.x;
          xs[r][1] = q4.y;
          xs[r][2] = q4.z;
          xs[r][3] = q4.w;
        } else {
          const double2 a2 = *reinterpret_cast<const double2*>(tile + (size_t)r * d.ld + c0);
          const double2 b2 = *reinterpret_cast<const double2*>(tile + (size_t)r * d.ld + c0 + 2);
          xs[r][0] = a2.x;
          xs[r][1] = a2.y;
          xs[r][2] = b2.x;
          xs[r][3] = b2.y;
        }
      } else {
        xs[r][0] = xs[r][1] = xs[r][2] = xs[r][3] = 0.0;
      }
    }
    __syncthreads();  // every thread holds its slice of the tile: the stage is free
    if (tid == 0 && k + (int64_t)kDenseStages * gridDim.x < n_tiles) issue(k + (int64_t)kDenseStages * gridDim.x, st);
    if constexpr (DOT) {
      double p[16];  // all 16 rows' warp trees interleave (rows past nr are zeros)
#pragma unroll
      for (int r = 0; r < 16; ++r) p[r] = ((xs[r][0] * vr[0] + xs[r][1] * vr[1]) + xs[r][2] * vr[2]) + xs[r][3] * vr[3];
      const double rs = warp_rows_sum16(p);  // lanes 2r, 2r + 1: row r
      if ((lane & 1) == 0) wdot[wid][lane >> 1] = rs;
      __syncthreads();
      if (tid < nr) {
        double t = 0.0;
#pragma unroll
        for (int w = 0; w < kWarps; ++w) t += wdot[w][tid];
        trow[tid] = t;
        if (MODE == 2) y[r0 + tid] = t;
      }
      __syncthreads();
    } else if constexpr (MODE == 1) {
      if (tid < nr) trow[tid] = __ldg(u + r0 + tid);
      __syncthreads();
    }
    if constexpr (MODE != 2) {
#pragma unroll
      for (int r = 0; r < 16; ++r) {  // rows past nr hold zeros: adding them is exact
        const double t = MODE == 3 ? 0.0 : (r < nr ? trow[r] : 0.0);
#pragma unroll
        for (int q = 0; q < 4; ++q) acc[q] += MODE == 3 ? xs[r][q] * xs[r][q] : t * xs[r][q];
      }
    }
    if constexpr (DOT || MODE == 1) __syncthreads();  // trow / wdot reused by the next tile
  }
  if constexpr (MODE != 2) {
    if (own)
#pragma unroll
      for (int q = 0; q < 4; ++q)
        if (c0 + q < d.cols) d.partial[(int64_t)(c0 + q) * d.n_cta + blockIdx.x] = acc[q];
  }
}

// Per column: sum of the CTA partials (contiguous, warp per column, fixed
// lane-strided order + warp tree), then the X^T epilogue and its dots.
template <Epi E>
__global__ void __launch_bounds__(kThreads) k_dense_finish(DenseDev d, XtArgs a) {
  if (a.done != nullptr && *a.done) return;
  const double* v = a.v;
  double* out = a.out;
  if constexpr (E == Epi::Fcg) {
    if (a.sc->done) return;
    const size_t off = (size_t)ring_slot(a.sc) * a.ring_stride;
    v += off;
    out += off;
  } else if constexpr (E == Epi::Cg) {
    if (a.sc->done) return;
  }
  __shared__ double sh[kWarps];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  double d0 = 0.0, d1 = 0.0;
  for (int64_t j = (int64_t)blockIdx.x * kWarps + wid; j < d.cols; j += (int64_t)gridDim.x * kWarps) {
    const double* pj = d.partial + j * d.n_cta;
    double sum = 0.0;
    for (int b = lane; b < d.n_cta; b += 32) sum += __ldcg(pj + b);
    sum = warp_sum(sum);
    if (lane == 0) xt_epilogue<E>((int)j, sum, a, v, out, d0, d1);
  }
  if constexpr (has_dots<E>()) {
    const double b0 = block_sum(d0, sh);
    const double b1 = (E == Epi::Fcg) ? block_sum(d1, sh) : 0.0;
    if (threadIdx.x == 0) {
      d.fin_slots[blockIdx.x * 2] = b0;
      d.fin_slots[blockIdx.x * 2 + 1] = b1;
    }
    if (grid_last(d.fin_ticket)) {
      const double s0 = sum_slots(d.fin_slots, gridDim.x, 2, 0, sh);
      const double s1 = (E == Epi::Fcg) ? sum_slots(d.fin_slots, gridDim.x, 2, 1, sh) : 0.0;
      if (threadIdx.x == 0) xt_finalize<E>(a.sc, s0, s1);
    }
  }
}

__global__ void k_add_const(double* x, double c, int64_t n) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    x[i] += c;
}


// ------------------------------------------------------------------ Krylov vector kernels
template <class F>
__device__ __forceinline__ void grid_stride(int64_t n, F&& f) {
  for (int64_t i = (int64_t)blockIdx.x * kThreads + threadIdx.x; i < n; i += (int64_t)gridDim.x * kThreads) f(i);
}

// x = 0, r = b, nb = ||b|| (krylov.cpp:164-176), rhs finiteness (krylov.cpp:23-31)
__global__ void __launch_bounds__(kThreads) k_krylov_begin(const double* __restrict__ b, double* __restrict__ x,
                                                           double* __restrict__ r, int64_t n, KrylovScalars* sc,
                                                           double* hist, double* slots, unsigned* ticket) {
  __shared__ double sh[kWarps];
  double acc = 0.0, bad = 0.0;
  grid_stride(n, [&](int64_t i) {
    const double bi = b[i];
    x[i] = 0.0;
    r[i] = bi;
    acc += bi * bi;
    if (!isfinite(bi)) bad += 1.0;
  });
  const double s0 = block_sum(acc, sh);
  const double s1 = block_sum(bad, sh);
  if (threadIdx.x == 0) {
    slots[blockIdx.x * 2] = s0;
    slots[blockIdx.x * 2 + 1] = s1;
  }
  if (grid_last(ticket)) {
    const double t0 = sum_slots(slots, gridDim.x, 2, 0, sh);
    const double t1 = sum_slots(slots, gridDim.x, 2, 1, sh);
    if (threadIdx.x == 0) {
      sc->it = 0;
      sc->use = 0;
      sc->status = t1 > 0.0 ? 3 : 0;
      sc->nb = sqrt(t0);
      sc->converged = 0;
      sc->done = sc->status != 0 ? 1 : 0;
      sc->rel = 1.0;
      if (sc->status == 0 && sc->nb == 0.0) {  // krylov.cpp:170-175
        sc->converged = 1;
        sc->done = 1;
        sc->rel = 0.0;
        hist[0] = 0.0;
      }
    }
  }
}

// Gram-Schmidt coefficients c_q = <z, Ap_q> / <p_q, Ap_q> over the newest
// use = min(m_i, |history|) directions (krylov.cpp:189-197).
__global__ void __launch_bounds__(kThreads) k_fcg_gs_dots(const double* __restrict__ z,
                                                          const double* __restrict__ ap_ring, int64_t n,
                                                          KrylovScalars* sc, double* slots, unsigned* ticket) {
  if (sc->done) return;
  const int it = sc->it, keep = sc->keep;
  const int mi = it == 0 ? 0 : max(1, it % (keep + 1));
  const int use = min(mi, min(it, keep));
  if (use == 0) {
    if (blockIdx.x == 0 && threadIdx.x == 0) sc->use = 0;
    return;
  }
  __shared__ double sh[kWarps][32];
  const int R = keep + 1;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  // one pass: z[i] read once, all `use` dots accumulated in registers
  double acc[32];
#pragma unroll
  for (int q = 0; q < 32; ++q) acc[q] = 0.0;
  grid_stride(n, [&](int64_t i) {
    const double zi = z[i];
#pragma unroll
    for (int q = 0; q < 32; ++q)
      if (q < use) acc[q] += zi * ap_ring[(size_t)((it - use + q) % R) * n + i];
  });
#pragma unroll
  for (int q = 0; q < 32; ++q) {
    if (q < use) {
      const double v = warp_sum(acc[q]);
      if (lane == 0) sh[wid][q] = v;
    }
  }
  __syncthreads();
  if (threadIdx.x < use) {  // fixed warp order
    double v = 0.0;
#pragma unroll
    for (int w = 0; w < kWarps; ++w) v += sh[w][threadIdx.x];
    slots[(size_t)blockIdx.x * 32 + threadIdx.x] = v;
  }
  if (grid_last(ticket)) {  // warp per coefficient, lanes over the CTAs (fixed order)
    for (int q = wid; q < use; q += kWarps) {
      double v = 0.0;
      for (int b = lane; b < (int)gridDim.x; b += 32) v += __ldcg(slots + (size_t)b * 32 + q);
      v = warp_sum(v);
      if (lane == 0) sc->coeff[q] = v / sc->pap_ring[(it - use + q) % R];
    }
    if (threadIdx.x == 0) sc->use = use;
  }
}

// p = z - sum_q c_q p_q, oldest -> newest, written into ring slot it % (m+1)
__global__ void __launch_bounds__(kThreads) k_fcg_update_p(const double* __restrict__ z, double* p_ring, int64_t n,
                                                           const KrylovScalars* sc) {
  if (sc->done) return;
  __shared__ double cf[32];
  const int it = sc->it, R = sc->keep + 1, use = sc->use;
  if (threadIdx.x < use) cf[threadIdx.x] = sc->coeff[threadIdx.x];
  __syncthreads();
  double* p = p_ring + (size_t)(it % R) * n;
  grid_stride(n, [&](int64_t i) {
    double pi = z[i];
    for (int q = 0; q < use; ++q) pi -= cf[q] * p_ring[(size_t)((it - use + q) % R) * n + i];
    p[i] = pi;
  });
}

// x += alpha p; r -= alpha Ap; rel = ||r|| / ||rhs|| (krylov.cpp:208-223)
__global__ void __launch_bounds__(kThreads) k_fcg_axpy(double* __restrict__ x, double* __restrict__ r,
                                                       const double* __restrict__ p_ring,
                                                       const double* __restrict__ ap_ring, int64_t n,
                                                       KrylovScalars* sc, double* hist, double* slots,
                                                       unsigned* ticket) {
  if (sc->done) return;
  __shared__ double sh[kWarps];
  const size_t off = (size_t)ring_slot(sc) * n;
  const double* p = p_ring + off;
  const double* ap = ap_ring + off;
  const double alpha = sc->alpha;
  double acc = 0.0;
  grid_stride(n, [&](int64_t i) {
    x[i] += alpha * p[i];
    const double ri = r[i] - alpha * ap[i];
    r[i] = ri;
    acc += ri * ri;
  });
  const double s = block_sum(acc, sh);
  if (threadIdx.x == 0) slots[blockIdx.x * 2] = s;
  if (grid_last(ticket)) {
    const double rr = sum_slots(slots, gridDim.x, 2, 0, sh);
    if (threadIdx.x == 0) {
      const double rel = sqrt(rr) / sc->nb;
      hist[sc->it] = rel;
      sc->rel = rel;
      sc->it += 1;
      if (rel <= sc->tol) {
        sc->converged = 1;
        sc->done = 1;
      } else if (sc->it >= sc->max_iters) {
        sc->done = 1;
      }
    }
  }
}

// CG start (krylov.cpp:100-123): x = 0, r = b, z = D^-1 r (or r), p = z, rz = <r,z>
__global__ void __launch_bounds__(kThreads) k_cg_begin(const double* __restrict__ b, const double* __restrict__ inv,
                                                       double* x, double* r, double* z, double* p, int64_t n,
                                                       KrylovScalars* sc, double* hist, double* slots,
                                                       unsigned* ticket) {
  __shared__ double sh[kWarps];
  double bb = 0.0, rz = 0.0, bad = 0.0;
  grid_stride(n, [&](int64_t i) {
    const double bi = b[i];
    x[i] = 0.0;
    r[i] = bi;
    const double zi = inv != nullptr ? inv[i] * bi : bi;
    if (inv != nullptr) z[i] = zi;
    p[i] = zi;
    bb += bi * bi;
    rz += bi * zi;
    if (!isfinite(bi)) bad += 1.0;
  });
  const double s0 = block_sum(bb, sh), s1 = block_sum(rz, sh), s2 = block_sum(bad, sh);
  if (threadIdx.x == 0) {
    slots[blockIdx.x * 4] = s0;
    slots[blockIdx.x * 4 + 1] = s1;
    slots[blockIdx.x * 4 + 2] = s2;
  }
  if (grid_last(ticket)) {
    const double t0 = sum_slots(slots, gridDim.x, 4, 0, sh);
    const double t1 = sum_slots(slots, gridDim.x, 4, 1, sh);
    const double t2 = sum_slots(slots, gridDim.x, 4, 2, sh);
    if (threadIdx.x == 0) {
      sc->it = 0;
      sc->status = t2 > 0.0 ? 3 : 0;
      sc->nb = sqrt(t0);
      sc->rz = t1;
      sc->converged = 0;
      sc->done = sc->status != 0 ? 1 : 0;
      sc->rel = 1.0;
      if (sc->status == 0 && sc->nb == 0.0) {
        sc->converged = 1;
        sc->done = 1;
        sc->rel = 0.0;
        hist[0] = 0.0;
      }
    }
  }
}

// x += alpha p; r -= alpha Ap; rel; z = D^-1 r; rz' = <r,z>; beta = rz'/rz (krylov.cpp:134-153)
__global__ void __launch_bounds__(kThreads) k_cg_axpy(double* __restrict__ x, double* __restrict__ r, double* z,
                                                      const double* __restrict__ inv, const double* __restrict__ p,
                                                      const double* __restrict__ ap, int64_t n, KrylovScalars* sc,
                                                      double* hist, double* slots, unsigned* ticket,
                                                      int general_m) {
  if (sc->done) return;
  __shared__ double sh[kWarps];
  const double alpha = sc->alpha;
  double rr = 0.0, rz = 0.0;
  grid_stride(n, [&](int64_t i) {
    x[i] += alpha * p[i];
    const double ri = r[i] - alpha * ap[i];
    r[i] = ri;
    rr += ri * ri;
    const double zi = inv != nullptr ? inv[i] * ri : ri;
    if (inv != nullptr) z[i] = zi;
    rz += ri * zi;
  });
  const double s0 = block_sum(rr, sh), s1 = block_sum(rz, sh);
  if (threadIdx.x == 0) {
    slots[blockIdx.x * 2] = s0;
    slots[blockIdx.x * 2 + 1] = s1;
  }
  if (grid_last(ticket)) {
    const double t0 = sum_slots(slots, gridDim.x, 2, 0, sh);
    const double t1 = sum_slots(slots, gridDim.x, 2, 1, sh);
    if (threadIdx.x == 0) {
      const double rel = sqrt(t0) / sc->nb;
      hist[sc->it] = rel;
      sc->rel = rel;
      sc->it += 1;
      if (rel <= sc->tol) {
        sc->converged = 1;
        sc->done = 1;
      } else {
        if (!general_m) {  // general preconditioner: <r, z> after z = M r (k_pcg_rz)
          sc->beta_cg = t1 / sc->rz;
          sc->rz = t1;
        }
        if (sc->it >= sc->max_iters) sc->done = 1;
      }
    }
  }
}

__global__ void __launch_bounds__(kThreads) k_cg_update_p(double* __restrict__ p, const double* __restrict__ z,
                                                          int64_t n, const KrylovScalars* sc) {
  if (sc->done) return;
  const double b = sc->beta_cg;
  grid_stride(n, [&](int64_t i) { p[i] = z[i] + b * p[i]; });
}

// ------------------------------------------------------------------ aggregation
// r_c(s) = sum over members i of s, increasing i, of w_i r_i; zero r_i skipped
// (coarsening.cpp:43-55 scatter order == this gather order, bit for bit).
__global__ void __launch_bounds__(kThreads) k_restrict(const int32_t* __restrict__ mptr,
                                                       const int32_t* __restrict__ members,
                                                       const double* __restrict__ weight,
                                                       const double* __restrict__ fine, double* __restrict__ coarse,
                                                       int64_t nc, const int32_t* done) {
  if (done != nullptr && *done) return;
  grid_stride(nc, [&](int64_t s) {
    double acc = 0.0;
    for (int q = mptr[s]; q < mptr[s + 1]; ++q) {
      const int i = members[q];
      const double fi = fine[i];
      if (fi == 0.0) continue;
      acc = __dadd_rn(acc, __dmul_rn(weight[i], fi));  // no contraction: bit-equal to the reference
    }
    coarse[s] = acc;
  });
}

// z1_i = 0.0 + w_i e_c(label_i)   (coarsening.cpp:30-41)
__global__ void __launch_bounds__(kThreads) k_prolong(const int32_t* __restrict__ label,
                                                      const double* __restrict__ weight,
                                                      const double* __restrict__ coarse, double* __restrict__ fine,
                                                      int64_t nf, const int32_t* done) {
  if (done != nullptr && *done) return;
  grid_stride(nf, [&](int64_t i) {
    fine[i] = __dadd_rn(0.0, __dmul_rn(weight[i], coarse[label[i]]));
  });
}

// y = A x, warp per row
__global__ void __launch_bounds__(kThreads) k_dense_gemv(const double* __restrict__ a, const double* __restrict__ x,
                                                         double* __restrict__ y, int64_t n, const int32_t* done) {
  if (done != nullptr && *done) return;
  const int lane = threadIdx.x & 31;
  const int64_t warp = ((int64_t)blockIdx.x * kThreads + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * kThreads) >> 5;
  for (int64_t row = warp; row < n; row += nw) {
    const double* ar = a + row * n;
    double s = 0.0;
    for (int64_t j = lane; j < n; j += 32) s += ar[j] * __ldg(x + j);
    s = warp_sum(s);
    if (lane == 0) y[row] = s;
  }
}

__global__ void k_scale_by_lambda(const double* __restrict__ w, double* __restrict__ v, int64_t n,
                                  const KrylovScalars* sc) {
  const double lam = sc->lambda;
  if (lam == 0.0) return;
  grid_stride(n, [&](int64_t i) { v[i] = w[i] / lam; });
}

// d_j = beta + sum_r X(r,j)^2 in increasing r (ridge.cpp:30-37 storage order)
template <bool PAT>
__global__ void k_diag_gram(const int32_t* __restrict__ ptr, const double* __restrict__ val, int64_t f,
                            double beta, double* __restrict__ out) {
  grid_stride(f, [&](int64_t j) {
    double d = beta;
    for (int k = ptr[j]; k < ptr[j + 1]; ++k) {
      const double x = PAT ? 1.0 : val[k];
      d = __dadd_rn(d, __dmul_rn(x, x));  // uncontracted: bit-equal to ridge.cpp:34
    }
    out[j] = d;
  });
}

__global__ void k_fill(double* p, double v, int64_t n) {
  grid_stride(n, [&](int64_t i) { p[i] = v; });
}

__global__ void k_copy_inner_count(const KrylovScalars* inner, KrylovScalars* outer, uint64_t* hist) {
  if (outer->done) return;
  hist[outer->it] = (uint64_t)inner->it;
  if (inner->status >= 1 && inner->status <= 3) {  // inner breakdown / bad rhs ends the outer solve too
    outer->status = 100 + inner->status;            // (the host turns it into the inner solve's error)
    outer->done = 1;
  }
}

inline void check_launch(const char* what) {
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) throw std::runtime_error(std::string("CUDA launch failed (") + what + "): " + cudaGetErrorString(e));
}

// K1 / K2 keep almost no SMEM: ask for the largest L1 carveout (once per kernel).
template <typename K>
void prefer_l1(K kern) {
  static std::mutex mu;
  static std::unordered_set<const void*> set;
  std::lock_guard<std::mutex> lock(mu);
  if (set.insert(reinterpret_cast<const void*>(kern)).second)
    cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout, 0);
}

template <typename K>
void allow_smem(K kern, int bytes) {  // once per kernel
  static std::mutex mu;
  static std::unordered_set<const void*> set;
  std::lock_guard<std::mutex> lock(mu);
  if (set.insert(reinterpret_cast<const void*>(kern)).second)
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
}

int num_sms() {
  static const int n = [] {
    int dev = 0, v = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
    return v;
  }();
  return n;
}

int grid_for(int64_t work_threads, int cap) {
  const int64_t g = (work_threads + kThreads - 1) / kThreads;
  return (int)std::max<int64_t>(1, std::min<int64_t>(g, cap));
}

template <int W, bool PAT>
void spmv_rows_impl(const SparseDev& x, const double* v, double* t, const int32_t* done,
                    const KrylovScalars* sc, int ring_stride, cudaStream_t s) {
  const int grid = grid_for((x.rows + 1) / 2 * W, 148 * 8);
  prefer_l1(k_spmv_rows<W, PAT, true>);
  prefer_l1(k_spmv_rows<W, PAT, false>);
  if (x.idx16 != nullptr)
    k_spmv_rows<W, PAT, true><<<grid, kThreads, 0, s>>>(x.ptr, x.idx, x.idx16, x.val, v, t, x.rows, done, sc,
                                                        ring_stride);
  else
    k_spmv_rows<W, PAT, false><<<grid, kThreads, 0, s>>>(x.ptr, x.idx, x.idx16, x.val, v, t, x.rows, done, sc,
                                                         ring_stride);
}

template <bool PAT>
void spmv_rows_w(const SparseDev& x, const double* v, double* t, const int32_t* done, const KrylovScalars* sc,
                 int ring_stride, cudaStream_t s) {
  if (x.col_inv != nullptr) {  // relabeled columns: v -> popularity order first
    k_vperm<<<grid_for(x.cols, 148 * 4), kThreads, 0, s>>>(v, x.col_inv, x.vperm, x.cols, done, sc, ring_stride);
    if (sc != nullptr) done = &sc->done;
    v = x.vperm;
    sc = nullptr;
    ring_stride = 0;
  }
  static const bool no_hotv = std::getenv("RMG_K1_NO_HOTV") != nullptr;
  if (x.sell_off != nullptr && x.col_inv != nullptr && !no_hotv) {
    constexpr int NT = 1024;
    const int n_hot = static_cast<int>(std::min<int64_t>(x.cols, kHotBlockMax));
    const int grid = static_cast<int>(std::min<int64_t>(num_sms(), (x.n_slices * 32 + NT - 1) / NT));
    auto go = [&](auto kern) {
      allow_smem(kern, kHotBlockMax * 8);
      kern<<<grid, NT, static_cast<size_t>(n_hot) * 8, s>>>(x.sell_off, x.sell_row, x.sell_len, x.idx, x.idx16, x.val,
                                                            v, t, x.n_slices, done, sc, ring_stride, n_hot);
    };
    // default: the pipelined kernel, 12 elements per round (cfg 5 shard K1 416 -> 378 us;
    // RMG_K1_PIPE=0 selects k_spmv_sell, 8 the 8-element variant: 391 us)
    static const int pipe = std::getenv("RMG_K1_PIPE") ? std::atoi(std::getenv("RMG_K1_PIPE")) : 12;
    if (pipe == 8) {
      if (x.idx16 != nullptr)
        go(k_spmv_sell_pipe<PAT, true, true, NT, 8>);
      else
        go(k_spmv_sell_pipe<PAT, false, true, NT, 8>);
    } else if (pipe == 12) {
      if (x.idx16 != nullptr)
        go(k_spmv_sell_pipe<PAT, true, true, NT, 12>);
      else
        go(k_spmv_sell_pipe<PAT, false, true, NT, 12>);
    } else {
      if (x.idx16 != nullptr)
        go(k_spmv_sell<PAT, true, true, NT>);
      else
        go(k_spmv_sell<PAT, false, true, NT>);
    }
    return;
  }
  if (x.sell_off != nullptr) {
    const int grid = grid_for(x.n_slices * 32, 148 * 8);
    auto go = [&](auto kern) {
      prefer_l1(kern);
      kern<<<grid, kThreads, 0, s>>>(x.sell_off, x.sell_row, x.sell_len, x.idx, x.idx16, x.val, v, t, x.n_slices,
                                     done, sc, ring_stride, 0);
    };
    // RMG_K1_PIPE=8: the pipelined kernel (60 registers: half the occupancy; cfg 2 cold
    // 19.0 -> 18.3 us, warm 15.9 -> 18.2 us), so the plain kernel stays the default here
    static const int pipe = std::getenv("RMG_K1_PIPE") ? std::atoi(std::getenv("RMG_K1_PIPE")) : 0;
    if (pipe == 8) {
      if (x.idx16 != nullptr)
        go(k_spmv_sell_pipe<PAT, true, false, kThreads, 8>);
      else
        go(k_spmv_sell_pipe<PAT, false, false, kThreads, 8>);
    } else {
      if (x.idx16 != nullptr)
        go(k_spmv_sell<PAT, true>);
      else
        go(k_spmv_sell<PAT, false>);
    }
    return;
  }
  switch (x.width) {
    case 4: spmv_rows_impl<4, PAT>(x, v, t, done, sc, ring_stride, s); break;
    case 8: spmv_rows_impl<8, PAT>(x, v, t, done, sc, ring_stride, s); break;
    case 16: spmv_rows_impl<16, PAT>(x, v, t, done, sc, ring_stride, s); break;
    default: spmv_rows_impl<32, PAT>(x, v, t, done, sc, ring_stride, s); break;
  }
}

template <int W, bool PAT>
void xt_impl_w(const SparseDev& xt, const XtSchedule& sch, Epi epi, const XtArgs& a, cudaStream_t s) {
  const dim3 grid(sch.n_items), block(kThreads);
  auto go = [&](auto kern) {
    prefer_l1(kern);
    kern<<<grid, block, 0, s>>>(xt.ptr, xt.idx, xt.val, sch, a);
  };
  switch (epi) {
    case Epi::Plain:
      if (sch.stream_t)
        go(k_xt<W, PAT, Epi::Plain, true>);
      else
        go(k_xt<W, PAT, Epi::Plain>);
      break;
    case Epi::Axpby: go(k_xt<W, PAT, Epi::Axpby>); break;
    case Epi::Fcg: go(k_xt<W, PAT, Epi::Fcg>); break;
    case Epi::Cg: go(k_xt<W, PAT, Epi::Cg>); break;
    case Epi::Rich: go(k_xt<W, PAT, Epi::Rich>); break;
    case Epi::Gram: go(k_xt<W, PAT, Epi::Gram>); break;
  }
}

template <bool PAT>
void xt_impl(const SparseDev& xt, const XtSchedule& sch, Epi epi, const XtArgs& a, cudaStream_t s) {
  switch (sch.width) {
    case 4: xt_impl_w<4, PAT>(xt, sch, epi, a, s); break;
    case 8: xt_impl_w<8, PAT>(xt, sch, epi, a, s); break;
    case 16: xt_impl_w<16, PAT>(xt, sch, epi, a, s); break;
    default: xt_impl_w<32, PAT>(xt, sch, epi, a, s); break;
  }
}

}  // namespace

int vec_grid(int64_t n) { return grid_for((n + 3) / 4, 296); }

void launch_spmv_rows(const SparseDev& x, const double* v, double* t, const int32_t* done, cudaStream_t s) {
  if (x.rows == 0) return;
  if (x.val == nullptr)
    spmv_rows_w<true>(x, v, t, done, nullptr, 0, s);
  else
    spmv_rows_w<false>(x, v, t, done, nullptr, 0, s);
  check_launch("spmv_rows");
}

void launch_spmv_rows_ring(const SparseDev& x, const double* v_ring, int ring_stride, const KrylovScalars* sc,
                           double* t, cudaStream_t s) {
  if (x.rows == 0) return;
  if (x.val == nullptr)
    spmv_rows_w<true>(x, v_ring, t, nullptr, sc, ring_stride, s);
  else
    spmv_rows_w<false>(x, v_ring, t, nullptr, sc, ring_stride, s);
  check_launch("spmv_rows_ring");
}

void launch_xt_epilogue(const double* sums, int64_t features, Epi epi, const XtArgs& a, double* fin_slots,
                        unsigned* fin_ticket, int fin_grid, cudaStream_t s) {
  XtSchedule sch;
  sch.features = features;
  sch.partial = const_cast<double*>(sums);
  sch.fin_slots = fin_slots;
  sch.fin_ticket = fin_ticket;
  const dim3 fg(fin_grid), block(kThreads);
  switch (epi) {
    case Epi::Plain: k_xt_finish<Epi::Plain><<<fg, block, 0, s>>>(sch, a); break;
    case Epi::Axpby: k_xt_finish<Epi::Axpby><<<fg, block, 0, s>>>(sch, a); break;
    case Epi::Fcg: k_xt_finish<Epi::Fcg><<<fg, block, 0, s>>>(sch, a); break;
    case Epi::Cg: k_xt_finish<Epi::Cg><<<fg, block, 0, s>>>(sch, a); break;
    case Epi::Rich: k_xt_finish<Epi::Rich><<<fg, block, 0, s>>>(sch, a); break;
    case Epi::Gram: k_xt_finish<Epi::Gram><<<fg, block, 0, s>>>(sch, a); break;
  }
  check_launch("xt_epilogue");
}

void launch_xt_hot(const HotXtDev& h, const double* t, const int32_t* done, const KrylovScalars* sc, double* sums,
                   cudaStream_t s) {
  if (h.H == 0) return;
  const size_t smem = static_cast<size_t>(h.B + 1) * sizeof(double);  // + the padding entries' zero slot
  if (h.val == nullptr) {
    allow_smem(k_xt_hot<true>, kHotBlockMax * 8 + 8);
    k_xt_hot<true><<<h.nblk, kHotThreads, smem, s>>>(h, t, done, sc);
  } else {
    allow_smem(k_xt_hot<false>, kHotBlockMax * 8 + 8);
    k_xt_hot<false><<<h.nblk, kHotThreads, smem, s>>>(h, t, done, sc);
  }
  k_xt_hot_chunks<<<dim3((h.H + kThreads - 1) / kThreads, h.S), kThreads, 0, s>>>(h, done, sc);
  k_xt_hot_final<<<(h.H + kThreads - 1) / kThreads, kThreads, 0, s>>>(h, sums, done, sc);
  check_launch("xt_hot");
}

// out[f] = sum over chunks c (in order) of part[c][f], for the listed (cold) features
__global__ void __launch_bounds__(kThreads) k_chunk_combine(const double* __restrict__ part, int nchunks, int64_t F,
                                                            const int32_t* __restrict__ list, int64_t nlist,
                                                            double* __restrict__ out, const int32_t* done,
                                                            const KrylovScalars* sc) {
  if (done != nullptr && *done) return;
  if (sc != nullptr && sc->done) return;
  grid_stride(nlist, [&](int64_t q) {
    const int64_t f = list[q];
    double acc = 0.0;
    for (int c = 0; c < nchunks; ++c) acc += part[(int64_t)c * F + f];
    out[f] = acc;
  });
}

void launch_chunk_combine(const double* part, int nchunks, int64_t F, const int32_t* list, int64_t nlist, double* out,
                          const int32_t* done, const KrylovScalars* sc, cudaStream_t s) {
  k_chunk_combine<<<grid_for(nlist, 148 * 4), kThreads, 0, s>>>(part, nchunks, F, list, nlist, out, done, sc);
  check_launch("chunk_combine");
}

void launch_xt(const SparseDev& xt, const XtSchedule& sch, Epi epi, const XtArgs& a, cudaStream_t s) {
  if (sch.n_items == 0) return;
  if (xt.val == nullptr)
    xt_impl<true>(xt, sch, epi, a, s);
  else
    xt_impl<false>(xt, sch, epi, a, s);
  check_launch("xt");
}

void launch_krylov_begin(const double* b, double* x, double* r, int64_t n, KrylovScalars* sc, double* hist,
                         const VecWork& w, cudaStream_t s) {
  k_krylov_begin<<<w.grid, kThreads, 0, s>>>(b, x, r, n, sc, hist, w.slots, w.ticket);
  check_launch("krylov_begin");
}

void launch_fcg_gs(const double* z, const double* ap_ring, double* p_ring, int64_t n, KrylovScalars* sc,
                   const VecWork& w, cudaStream_t s) {
  k_fcg_gs_dots<<<w.grid, kThreads, 0, s>>>(z, ap_ring, n, sc, w.slots, w.ticket);
  k_fcg_update_p<<<w.grid, kThreads, 0, s>>>(z, p_ring, n, sc);
  check_launch("fcg_gs");
}

void launch_fcg_axpy(double* x, double* r, const double* p_ring, const double* ap_ring, int64_t n,
                     KrylovScalars* sc, double* hist, const VecWork& w, cudaStream_t s) {
  k_fcg_axpy<<<w.grid, kThreads, 0, s>>>(x, r, p_ring, ap_ring, n, sc, hist, w.slots, w.ticket);
  check_launch("fcg_axpy");
}

void launch_cg_begin(const double* b, const double* inv_diag, double* x, double* r, double* z, double* p, int64_t n,
                     KrylovScalars* sc, double* hist, const VecWork& w, cudaStream_t s) {
  k_cg_begin<<<w.grid, kThreads, 0, s>>>(b, inv_diag, x, r, z, p, n, sc, hist, w.slots, w.ticket);
  check_launch("cg_begin");
}

void launch_cg_axpy(double* x, double* r, double* z, const double* inv_diag, const double* p, const double* ap,
                    int64_t n, KrylovScalars* sc, double* hist, const VecWork& w, cudaStream_t s, bool general_m) {
  k_cg_axpy<<<w.grid, kThreads, 0, s>>>(x, r, z, inv_diag, p, ap, n, sc, hist, w.slots, w.ticket, general_m ? 1 : 0);
  check_launch("cg_axpy");
}

// ---------------------------------------------------------------- V-cycle (extension)
// Symmetric two-grid / multigrid cycle with damped-Jacobi pre- and post-smoothing
// (BASELINE cfg 1's "Jacobi smoothing (1 pre-sweep, 1 post-sweep)", north-star (2);
// not a reference routine).  Elementwise steps:
//   pre:  x1 = w dinv r                         (k_vc_pre)
//   r1 = r - y1   (y1 = A x1)                   (k_vc_sub, in place in y1)
//   x2 = x1 + e   (e = P e_c)                   (k_vc_add, in place in e)
//   post: z = x2 + w dinv (r - y2)  (y2 = A x2) (k_vc_post)
__global__ void __launch_bounds__(kThreads) k_vc_pre(const double* __restrict__ r, const double* __restrict__ dinv,
                                                     double w, double* __restrict__ x1, int64_t n, const int32_t* done) {
  if (done != nullptr && *done) return;
  grid_stride(n, [&](int64_t i) { x1[i] = w * (dinv[i] * r[i]); });
}
__global__ void __launch_bounds__(kThreads) k_vc_sub(const double* __restrict__ r, double* __restrict__ y, int64_t n,
                                                     const int32_t* done) {
  if (done != nullptr && *done) return;
  grid_stride(n, [&](int64_t i) { y[i] = r[i] - y[i]; });
}
__global__ void __launch_bounds__(kThreads) k_vc_add(const double* __restrict__ x1, double* __restrict__ e, int64_t n,
                                                     const int32_t* done) {
  if (done != nullptr && *done) return;
  grid_stride(n, [&](int64_t i) { e[i] = x1[i] + e[i]; });
}
// additive finest level: z = dinv r + w_i e_c(label_i) (Jacobi term first, then the
// prolonged coarse correction; one pass instead of pre + prolong + add)
__global__ void __launch_bounds__(kThreads) k_vc_jacobi_prolong(const double* __restrict__ r,
                                                                const double* __restrict__ dinv,
                                                                const int32_t* __restrict__ label,
                                                                const double* __restrict__ weight,
                                                                const double* __restrict__ ec, double* __restrict__ z,
                                                                int64_t n, const int32_t* done) {
  if (done != nullptr && *done) return;
  grid_stride(n, [&](int64_t i) { z[i] = dinv[i] * r[i] + weight[i] * ec[label[i]]; });
}
__global__ void __launch_bounds__(kThreads) k_vc_post(const double* __restrict__ x2, const double* __restrict__ r,
                                                      const double* __restrict__ y2, const double* __restrict__ dinv,
                                                      double w, double* __restrict__ z, int64_t n, const int32_t* done) {
  if (done != nullptr && *done) return;
  grid_stride(n, [&](int64_t i) { z[i] = x2[i] + w * (dinv[i] * (r[i] - y2[i])); });
}

// PCG with a general preconditioner (krylov.cpp:94-157 with z = M r): rz' = <r, z>
// (fixed-order grid reduction); begin: rz = rz', else beta = rz' / rz, rz = rz'.
__global__ void __launch_bounds__(kThreads) k_pcg_rz(const double* __restrict__ r, const double* __restrict__ z,
                                                     int64_t n, KrylovScalars* sc, int begin, double* slots,
                                                     unsigned* ticket) {
  if (sc->done) return;
  __shared__ double sh[kWarps];
  double rz = 0.0;
  grid_stride(n, [&](int64_t i) { rz += r[i] * z[i]; });
  const double b = block_sum(rz, sh);
  if (threadIdx.x == 0) slots[blockIdx.x] = b;
  if (grid_last(ticket)) {
    const double t = sum_slots(slots, gridDim.x, 1, 0, sh);
    if (threadIdx.x == 0) {
      if (!begin) sc->beta_cg = t / sc->rz;
      sc->rz = t;
    }
  }
}

// ---------------------------------------------------------------- batched pcg_vcycle
// k right-hand sides in lock step (BASELINE cfg 3's "16 right-hand sides solved as a
// batched block operator"): every block is row-major n x k, so each row of a
// block is k contiguous doubles (the block operator's layout).
// Per column the arithmetic is the single-RHS pcg_vcycle's; reductions are
// per-column fixed-order (CTA row ranges, then CTAs in order).
__global__ void __launch_bounds__(kThreads) k_bdot_partial(const double* __restrict__ a, const double* __restrict__ b,
                                                           int64_t n, int k, double* __restrict__ partial) {
  __shared__ double red[kThreads];
  const int rl_n = kThreads / k, t = threadIdx.x, rl = t / k, c = t % k;
  const int64_t rows_per = (n + gridDim.x - 1) / gridDim.x;
  const int64_t r0 = (int64_t)blockIdx.x * rows_per, r1 = (n < r0 + rows_per ? n : r0 + rows_per);
  double acc = 0.0;
  if (rl < rl_n)
    for (int64_t i = r0 + rl; i < r1; i += rl_n) acc += a[i * k + c] * b[i * k + c];
  red[t] = acc;
  __syncthreads();
  if (t < k) {
    double s = 0.0;
    for (int q = 0; q < rl_n; ++q) s += red[q * k + t];
    partial[(size_t)blockIdx.x * k + t] = s;
  }
}

// out[c] = the g block partials of column c summed: 16 sub-sums over every 16th
// block (4 loads in flight), added in sub order -- a fixed order
__global__ void __launch_bounds__(1024) k_bdot_final(const double* __restrict__ partial, int g, int k,
                                                     double* __restrict__ out) {
  __shared__ double sh[16][64];
  const int c = threadIdx.x & 63, sub = threadIdx.x >> 6;
  double s = 0.0;
  if (c < k)
    for (int b = sub; b < g; b += 64) {
      double v[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) v[u] = b + 16 * u < g ? partial[(size_t)(b + 16 * u) * k + c] : 0.0;
#pragma unroll
      for (int u = 0; u < 4; ++u) s += v[u];
    }
  sh[sub][c] = s;
  __syncthreads();
  if (sub == 0 && c < k) {
    double tot = sh[0][c];
#pragma unroll
    for (int u = 1; u < 16; ++u) tot += sh[u][c];
    out[c] = tot;
  }
}

// x += alpha p, r -= alpha Ap and the partials of <r, r> in one pass: the rows are dealt to
// blocks and threads exactly as k_bdot_partial deals them, so the partials (and the sums
// k_bdot_final forms from them) are those of the separate update + dot, bit for bit.
__global__ void __launch_bounds__(kThreads) k_bupdate_xr_dot(double* __restrict__ x, double* __restrict__ r,
                                                             const double* __restrict__ p,
                                                             const double* __restrict__ ap, const BlockScalars* sc,
                                                             int64_t n, int k, double* __restrict__ partial) {
  __shared__ double red[kThreads];
  const int rl_n = kThreads / k, t = threadIdx.x, rl = t / k, c = t % k;
  const int64_t rows_per = (n + gridDim.x - 1) / gridDim.x;
  const int64_t r0 = (int64_t)blockIdx.x * rows_per, r1 = (n < r0 + rows_per ? n : r0 + rows_per);
  double acc = 0.0;
  if (rl < rl_n) {
    const bool frozen = sc[c].done != 0;
    const double a = sc[c].alpha;
    for (int64_t i = r0 + rl; i < r1; i += rl_n) {
      const int64_t q = i * k + c;
      double rv = r[q];
      if (!frozen) {
        x[q] += a * p[q];
        rv = rv - a * ap[q];
        r[q] = rv;
      }
      acc += rv * rv;
    }
  }
  red[t] = acc;
  __syncthreads();
  if (t < k) {
    double s = 0.0;
    for (int q = 0; q < rl_n; ++q) s += red[q * k + t];
    partial[(size_t)blockIdx.x * k + t] = s;
  }
}

// z = D^-1 r + P e_c (the additive finest level) and the partials of <r, z> in one pass
// (same dealing of rows as k_bdot_partial)
__global__ void __launch_bounds__(kThreads) k_bvc_jacobi_prolong_dot(const double* __restrict__ r,
                                                                     const double* __restrict__ dinv,
                                                                     const int32_t* __restrict__ label,
                                                                     const double* __restrict__ weight,
                                                                     const double* __restrict__ ec,
                                                                     double* __restrict__ z, int64_t n, int k,
                                                                     double* __restrict__ partial) {
  __shared__ double red[kThreads];
  const int rl_n = kThreads / k, t = threadIdx.x, rl = t / k, c = t % k;
  const int64_t rows_per = (n + gridDim.x - 1) / gridDim.x;
  const int64_t r0 = (int64_t)blockIdx.x * rows_per, r1 = (n < r0 + rows_per ? n : r0 + rows_per);
  double acc = 0.0;
  if (rl < rl_n)
    for (int64_t i = r0 + rl; i < r1; i += rl_n) {
      const int64_t q = i * k + c;
      const double rv = r[q];
      const double zv = dinv[i] * rv + weight[i] * ec[(int64_t)label[i] * k + c];
      z[q] = zv;
      acc += rv * zv;
    }
  red[t] = acc;
  __syncthreads();
  if (t < k) {
    double s = 0.0;
    for (int q = 0; q < rl_n; ++q) s += red[q * k + t];
    partial[(size_t)blockIdx.x * k + t] = s;
  }
}

// begin: nb = ||rhs||, non-finite check, rz = <r, z>
__global__ void k_bpcg_begin(BlockScalars* sc, const double* rr, const double* rz, const double* nonfinite, int k,
                             double* hist) {
  const int c = threadIdx.x;
  if (c >= k) return;
  BlockScalars& s = sc[c];
  s.nb = sqrt(rr[c]);
  s.rz = rz[c];
  s.it = 0;
  s.converged = 0;
  s.status = nonfinite[c] > 0.0 ? 3 : 0;
  s.done = s.status != 0 ? 1 : 0;
  s.rel = 1.0;
  if (s.status == 0 && s.nb == 0.0) {
    s.converged = 1;
    s.done = 1;
    s.rel = 0.0;
    hist[c] = 0.0;
  }
}

// alpha = rz / <p, Ap>; <p, Ap> must be > 0 (krylov.cpp:128-132)
__global__ void k_bpcg_alpha(BlockScalars* sc, const double* pap, int k) {
  const int c = threadIdx.x;
  if (c >= k || sc[c].done) return;
  BlockScalars& s = sc[c];
  s.pap = pap[c];
  if (!(s.pap > 0.0)) {
    s.status = 2;
    s.done = 1;
    s.alpha = 0.0;
    return;
  }
  s.alpha = s.rz / s.pap;
}

__global__ void __launch_bounds__(kThreads) k_bupdate_xr(double* __restrict__ x, double* __restrict__ r,
                                                         const double* __restrict__ p, const double* __restrict__ ap,
                                                         const BlockScalars* sc, int64_t n, int k) {
  grid_stride(n * k, [&](int64_t q) {
    const int c = (int)(q % k);
    if (sc[c].done) return;
    const double a = sc[c].alpha;
    x[q] += a * p[q];
    r[q] = r[q] - a * ap[q];
  });
}

// ||r|| / ||rhs||, history, stop test (krylov.cpp:136-143)
__global__ void k_bpcg_conv(BlockScalars* sc, const double* rr, int k, double* hist) {
  const int c = threadIdx.x;
  if (c >= k || sc[c].done) return;
  BlockScalars& s = sc[c];
  const double rel = sqrt(rr[c]) / s.nb;
  hist[(size_t)s.it * k + c] = rel;
  s.rel = rel;
  s.it += 1;
  if (rel <= s.tol) {
    s.converged = 1;
    s.done = 1;
  } else if (s.it >= s.max_iters) {
    s.done = 1;
  }
}

__global__ void k_bpcg_beta(BlockScalars* sc, const double* rz, int k) {
  const int c = threadIdx.x;
  if (c >= k || sc[c].done) return;
  sc[c].beta = rz[c] / sc[c].rz;
  sc[c].rz = rz[c];
}

// p = z + beta p for running columns; finished columns' p is zeroed (their Ap = 0)
__global__ void __launch_bounds__(kThreads) k_bupdate_p(double* __restrict__ p, const double* __restrict__ z,
                                                        const BlockScalars* sc, int64_t n, int k) {
  grid_stride(n * k, [&](int64_t q) {
    const int c = (int)(q % k);
    p[q] = sc[c].done ? 0.0 : z[q] + sc[c].beta * p[q];
  });
}

// V-cycle blocks (rows scaled by the level's Jacobi diagonal)
__global__ void __launch_bounds__(kThreads) k_bvc_pre(const double* __restrict__ r, const double* __restrict__ dinv,
                                                      double w, double* __restrict__ x1, int64_t n, int k) {
  grid_stride(n * k, [&](int64_t q) { x1[q] = w * (dinv[q / k] * r[q]); });
}
__global__ void __launch_bounds__(kThreads) k_bvc_post(const double* __restrict__ x2, const double* __restrict__ r,
                                                       const double* __restrict__ y2, const double* __restrict__ dinv,
                                                       double w, double* __restrict__ z, int64_t n, int k) {
  grid_stride(n * k, [&](int64_t q) { z[q] = x2[q] + w * (dinv[q / k] * (r[q] - y2[q])); });
}
__global__ void __launch_bounds__(kThreads) k_bsub(const double* __restrict__ r, double* __restrict__ y, int64_t nk) {
  grid_stride(nk, [&](int64_t q) { y[q] = r[q] - y[q]; });
}
__global__ void __launch_bounds__(kThreads) k_bvc_jacobi_prolong(const double* __restrict__ r,
                                                                 const double* __restrict__ dinv,
                                                                 const int32_t* __restrict__ label,
                                                                 const double* __restrict__ weight,
                                                                 const double* __restrict__ ec,
                                                                 double* __restrict__ z, int64_t n, int k) {
  grid_stride(n * k, [&](int64_t q) {
    const int64_t i = q / k;
    z[q] = dinv[i] * r[q] + weight[i] * ec[(int64_t)label[i] * k + q % k];
  });
}
__global__ void __launch_bounds__(kThreads) k_badd(const double* __restrict__ x1, double* __restrict__ e, int64_t nk) {
  grid_stride(nk, [&](int64_t q) { e[q] = x1[q] + e[q]; });
}
// rc[s][c] = sum over the members i of s (increasing) of w_i y[i][c]
// a warp per cluster, lane (h, c): the members e = h (mod 2) in order for column
// c0 + c (4 loads in flight), the two sub-sums added h = 0 first -- a fixed order
__global__ void __launch_bounds__(kThreads) k_brestrict(const int32_t* __restrict__ mptr,
                                                        const int32_t* __restrict__ members,
                                                        const double* __restrict__ weight,
                                                        const double* __restrict__ y, double* __restrict__ rc,
                                                        int64_t nc, int k) {
  const int lane = threadIdx.x & 31, h = lane >> 4, c = lane & 15;
  const int64_t nw = ((int64_t)gridDim.x * kThreads) >> 5;
  for (int64_t s = ((int64_t)blockIdx.x * kThreads + threadIdx.x) >> 5; s < nc; s += nw) {
    const int e0 = mptr[s], e1 = mptr[s + 1];
    for (int c0 = 0; c0 < k; c0 += 16) {
      const bool okc = c0 + c < k;
      double acc = 0.0;
      for (int e = e0 + h; e < e1; e += 8) {
        double wv[4], yv[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const bool ok = okc && e + 2 * u < e1;
          const int i = ok ? members[e + 2 * u] : 0;
          wv[u] = ok ? weight[i] : 0.0;
          yv[u] = ok ? y[(int64_t)i * k + c0 + c] : 0.0;
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) acc += wv[u] * yv[u];
      }
      const double other = __shfl_xor_sync(0xffffffffu, acc, 16);
      if (h == 0 && okc) rc[s * k + c0 + c] = acc + other;
    }
  }
}
// e[i][c] = w_i ec[label_i][c]
__global__ void __launch_bounds__(kThreads) k_bprolong(const int32_t* __restrict__ label,
                                                       const double* __restrict__ weight,
                                                       const double* __restrict__ ec, double* __restrict__ e,
                                                       int64_t nf, int k) {
  grid_stride(nf * k, [&](int64_t q) {
    const int64_t i = q / k;
    e[q] = weight[i] * ec[(int64_t)label[i] * k + q % k];
  });
}
// ec = A_c^-1 rc for k columns (row-major nc x nc inverse): a warp per row i, lane
// (h, c) sums the j = h (mod 2) terms of column c0 + c in order (4 in flight), h = 0
// first -- a fixed order
__global__ void __launch_bounds__(kThreads) k_bgemm_inv(const double* __restrict__ ainv, const double* __restrict__ rc,
                                                        double* __restrict__ ec, int64_t nc, int k) {
  const int lane = threadIdx.x & 31, h = lane >> 4, c = lane & 15;
  const int64_t nw = ((int64_t)gridDim.x * kThreads) >> 5;
  for (int64_t i = ((int64_t)blockIdx.x * kThreads + threadIdx.x) >> 5; i < nc; i += nw) {
    const double* row = ainv + i * nc;
    for (int c0 = 0; c0 < k; c0 += 16) {
      const bool okc = c0 + c < k;
      double acc = 0.0;
      for (int64_t j = h; j < nc; j += 8) {
        double av[4], rv[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const bool ok = okc && j + 2 * u < nc;
          av[u] = ok ? row[j + 2 * u] : 0.0;
          rv[u] = ok ? rc[(j + 2 * u) * k + c0 + c] : 0.0;
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) acc += av[u] * rv[u];
      }
      const double other = __shfl_xor_sync(0xffffffffu, acc, 16);
      if (h == 0 && okc) ec[i * k + c0 + c] = acc + other;
    }
  }
}
// column-major (n x k) <-> row-major (n x k)
__global__ void __launch_bounds__(kThreads) k_bcol2row(const double* __restrict__ cm, double* __restrict__ rm,
                                                       int64_t n, int k) {
  grid_stride(n * k, [&](int64_t q) { rm[q] = cm[(q % k) * n + q / k]; });
}
__global__ void __launch_bounds__(kThreads) k_brow2col(const double* __restrict__ rm, double* __restrict__ cm,
                                                       int64_t n, int k) {
  grid_stride(n * k, [&](int64_t q) { cm[(q % k) * n + q / k] = rm[q]; });
}
__global__ void __launch_bounds__(kThreads) k_bnonfinite(const double* __restrict__ r, int64_t n, int k,
                                                         double* __restrict__ bad) {
  // one CTA per column: count of non-finite entries (order irrelevant: integers)
  const int c = blockIdx.x;
  __shared__ double sh[kWarps];
  double cnt = 0.0;
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x) cnt += isfinite(r[i * k + c]) ? 0.0 : 1.0;
  cnt = block_sum(cnt, sh);
  if (threadIdx.x == 0) bad[c] = cnt;
}

void launch_bdots(const double* a, const double* b, int64_t n, int k, double* partial, int g, double* out,
                  cudaStream_t s) {
  k_bdot_partial<<<g, kThreads, 0, s>>>(a, b, n, k, partial);
  k_bdot_final<<<1, 1024, 0, s>>>(partial, g, k, out);
  check_launch("bdots");
}
void launch_bpcg_begin(BlockScalars* sc, const double* rr, const double* rz, const double* bad, int k, double* hist,
                       cudaStream_t s) {
  k_bpcg_begin<<<1, 64, 0, s>>>(sc, rr, rz, bad, k, hist);
  check_launch("bpcg_begin");
}
void launch_bpcg_alpha(BlockScalars* sc, const double* pap, int k, cudaStream_t s) {
  k_bpcg_alpha<<<1, 64, 0, s>>>(sc, pap, k);
}
void launch_bdot_final(const double* partial, int g, int k, double* out, cudaStream_t s) {
  k_bdot_final<<<1, 1024, 0, s>>>(partial, g, k, out);
}
void launch_bupdate_xr_dot(double* x, double* r, const double* p, const double* ap, const BlockScalars* sc, int64_t n,
                           int k, double* partial, int g, double* rr, cudaStream_t s) {
  k_bupdate_xr_dot<<<g, kThreads, 0, s>>>(x, r, p, ap, sc, n, k, partial);
  k_bdot_final<<<1, 1024, 0, s>>>(partial, g, k, rr);
}
void launch_bvc_jacobi_prolong_dot(const double* r, const double* dinv, const int32_t* label, const double* weight,
                                   const double* ec, double* z, int64_t n, int k, double* partial, int g, double* rz,
                                   cudaStream_t s) {
  k_bvc_jacobi_prolong_dot<<<g, kThreads, 0, s>>>(r, dinv, label, weight, ec, z, n, k, partial);
  k_bdot_final<<<1, 1024, 0, s>>>(partial, g, k, rz);
}
void launch_bupdate_xr(double* x, double* r, const double* p, const double* ap, const BlockScalars* sc, int64_t n,
                       int k, cudaStream_t s) {
  k_bupdate_xr<<<grid_for(n * k, 148 * 8), kThreads, 0, s>>>(x, r, p, ap, sc, n, k);
}
void launch_bpcg_conv(BlockScalars* sc, const double* rr, int k, double* hist, cudaStream_t s) {
  k_bpcg_conv<<<1, 64, 0, s>>>(sc, rr, k, hist);
}
void launch_bpcg_beta(BlockScalars* sc, const double* rz, int k, cudaStream_t s) {
  k_bpcg_beta<<<1, 64, 0, s>>>(sc, rz, k);
}
void launch_bupdate_p(double* p, const double* z, const BlockScalars* sc, int64_t n, int k, cudaStream_t s) {
  k_bupdate_p<<<grid_for(n * k, 148 * 8), kThreads, 0, s>>>(p, z, sc, n, k);
  check_launch("bpcg_update");
}
void launch_bvc_pre(const double* r, const double* dinv, double w, double* x1, int64_t n, int k, cudaStream_t s) {
  k_bvc_pre<<<grid_for(n * k, 148 * 8), kThreads, 0, s>>>(r, dinv, w, x1, n, k);
}
void launch_bvc_post(const double* x2, const double* r, const double* y2, const double* dinv, double w, double* z,
                     int64_t n, int k, cudaStream_t s) {
  k_bvc_post<<<grid_for(n * k, 148 * 8), kThreads, 0, s>>>(x2, r, y2, dinv, w, z, n, k);
}
void launch_bsub(const double* r, double* y, int64_t nk, cudaStream_t s) {
  k_bsub<<<grid_for(nk, 148 * 8), kThreads, 0, s>>>(r, y, nk);
}
void launch_badd(const double* x1, double* e, int64_t nk, cudaStream_t s) {
  k_badd<<<grid_for(nk, 148 * 8), kThreads, 0, s>>>(x1, e, nk);
}
void launch_brestrict(const int32_t* mptr, const int32_t* members, const double* weight, const double* y, double* rc,
                      int64_t nc, int k, cudaStream_t s) {
  k_brestrict<<<grid_for(nc * 32, 148 * 8), kThreads, 0, s>>>(mptr, members, weight, y, rc, nc, k);
}
void launch_bprolong(const int32_t* label, const double* weight, const double* ec, double* e, int64_t nf, int k,
                     cudaStream_t s) {
  k_bprolong<<<grid_for(nf * k, 148 * 8), kThreads, 0, s>>>(label, weight, ec, e, nf, k);
}
void launch_bgemm_inv(const double* ainv, const double* rc, double* ec, int64_t nc, int k, cudaStream_t s) {
  k_bgemm_inv<<<grid_for(nc * 32, 148 * 8), kThreads, 0, s>>>(ainv, rc, ec, nc, k);
}
void launch_bcol2row(const double* cm, double* rm, int64_t n, int k, cudaStream_t s) {
  k_bcol2row<<<grid_for(n * k, 148 * 8), kThreads, 0, s>>>(cm, rm, n, k);
}
void launch_brow2col(const double* rm, double* cm, int64_t n, int k, cudaStream_t s) {
  k_brow2col<<<grid_for(n * k, 148 * 8), kThreads, 0, s>>>(rm, cm, n, k);
}
void launch_bnonfinite(const double* r, int64_t n, int k, double* bad, cudaStream_t s) {
  k_bnonfinite<<<k, kThreads, 0, s>>>(r, n, k, bad);
  check_launch("bnonfinite");
}

void launch_vc_pre(const double* r, const double* dinv, double w, double* x1, int64_t n, const int32_t* done,
                   cudaStream_t s) {
  k_vc_pre<<<grid_for(n, 148 * 4), kThreads, 0, s>>>(r, dinv, w, x1, n, done);
  check_launch("vc_pre");
}
void launch_vc_sub(const double* r, double* y, int64_t n, const int32_t* done, cudaStream_t s) {
  k_vc_sub<<<grid_for(n, 148 * 4), kThreads, 0, s>>>(r, y, n, done);
  check_launch("vc_sub");
}
void launch_vc_add(const double* x1, double* e, int64_t n, const int32_t* done, cudaStream_t s) {
  k_vc_add<<<grid_for(n, 148 * 4), kThreads, 0, s>>>(x1, e, n, done);
  check_launch("vc_add");
}
void launch_vc_jacobi_prolong(const double* r, const double* dinv, const int32_t* label, const double* weight,
                              const double* ec, double* z, int64_t n, const int32_t* done, cudaStream_t s) {
  k_vc_jacobi_prolong<<<grid_for(n, 148 * 4), kThreads, 0, s>>>(r, dinv, label, weight, ec, z, n, done);
  check_launch("vc_jacobi_prolong");
}
void launch_bvc_jacobi_prolong(const double* r, const double* dinv, const int32_t* label, const double* weight,
                               const double* ec, double* z, int64_t n, int k, cudaStream_t s) {
  k_bvc_jacobi_prolong<<<grid_for(n * k, 148 * 8), kThreads, 0, s>>>(r, dinv, label, weight, ec, z, n, k);
}
void launch_vc_post(const double* x2, const double* r, const double* y2, const double* dinv, double w, double* z,
                    int64_t n, const int32_t* done, cudaStream_t s) {
  k_vc_post<<<grid_for(n, 148 * 4), kThreads, 0, s>>>(x2, r, y2, dinv, w, z, n, done);
  check_launch("vc_post");
}
void launch_pcg_rz(const double* r, const double* z, int64_t n, KrylovScalars* sc, bool begin, const VecWork& w,
                   cudaStream_t s) {
  k_pcg_rz<<<w.grid, kThreads, 0, s>>>(r, z, n, sc, begin ? 1 : 0, w.slots, w.ticket);
  check_launch("pcg_rz");
}

void launch_cg_update_p(double* p, const double* z, int64_t n, const KrylovScalars* sc, cudaStream_t s) {
  k_cg_update_p<<<vec_grid(n), kThreads, 0, s>>>(p, z, n, sc);
  check_launch("cg_update_p");
}

void launch_restrict(const int32_t* mptr, const int32_t* members, const double* weight, const double* fine,
                     double* coarse, int64_t n_coarse, const int32_t* done, cudaStream_t s) {
  k_restrict<<<grid_for(n_coarse, 148 * 4), kThreads, 0, s>>>(mptr, members, weight, fine, coarse, n_coarse, done);
  check_launch("restrict");
}

void launch_prolong(const int32_t* label, const double* weight, const double* coarse, double* fine, int64_t n_fine,
                    const int32_t* done, cudaStream_t s) {
  k_prolong<<<vec_grid(n_fine), kThreads, 0, s>>>(label, weight, coarse, fine, n_fine, done);
  check_launch("prolong");
}

void launch_dense_gemv(const double* a, const double* x, double* y, int64_t n, const int32_t* done, cudaStream_t s) {
  k_dense_gemv<<<grid_for(n * 32, 148 * 8), kThreads, 0, s>>>(a, x, y, n, done);
  check_launch("dense_gemv");
}

void launch_scale_by_lambda(const double* w, double* v, int64_t n, const KrylovScalars* sc, cudaStream_t s) {
  k_scale_by_lambda<<<vec_grid(n), kThreads, 0, s>>>(w, v, n, sc);
  check_launch("scale_by_lambda");
}

void launch_diag_gram(const SparseDev& xt, const XtSchedule& sch, double beta, double* out, cudaStream_t s) {
  const int64_t f = sch.features;
  if (xt.val == nullptr)
    k_diag_gram<true><<<grid_for(f, 148 * 8), kThreads, 0, s>>>(xt.ptr, xt.val, f, beta, out);
  else
    k_diag_gram<false><<<grid_for(f, 148 * 8), kThreads, 0, s>>>(xt.ptr, xt.val, f, beta, out);
  check_launch("diag_gram");
}

void launch_fill(double* p, double v, int64_t n, cudaStream_t s) {
  if (n == 0) return;
  k_fill<<<vec_grid(n), kThreads, 0, s>>>(p, v, n);
  check_launch("fill");
}

void launch_copy_inner_count(const KrylovScalars* inner, KrylovScalars* outer, uint64_t* inner_hist,
                             cudaStream_t s) {
  k_copy_inner_count<<<1, 1, 0, s>>>(inner, outer, inner_hist);
  check_launch("copy_inner_count");
}


namespace {
template <int MODE>
void dense_sweep(const DenseDev& d, const double* v, const double* u, double* y, const int32_t* done,
                 const KrylovScalars* sc, int ring_stride, cudaStream_t s) {
  const size_t smem = static_cast<size_t>(kDenseStages) * kDenseTileBytes;
  const int grid = d.n_cta;
  if (d.fp32) {
    allow_smem(k_dense_ata<float, MODE>, kDenseStages * kDenseTileBytes);
    k_dense_ata<float, MODE><<<grid, kThreads, smem, s>>>(d, v, u, y, done, sc, ring_stride);
  } else {
    allow_smem(k_dense_ata<double, MODE>, kDenseStages * kDenseTileBytes);
    k_dense_ata<double, MODE><<<grid, kThreads, smem, s>>>(d, v, u, y, done, sc, ring_stride);
  }
}

void dense_finish(const DenseDev& d, Epi epi, const XtArgs& a, cudaStream_t s) {
  const dim3 g(d.fin_grid), b(kThreads);
  switch (epi) {
    case Epi::Plain: k_dense_finish<Epi::Plain><<<g, b, 0, s>>>(d, a); break;
    case Epi::Axpby: k_dense_finish<Epi::Axpby><<<g, b, 0, s>>>(d, a); break;
    case Epi::Fcg: k_dense_finish<Epi::Fcg><<<g, b, 0, s>>>(d, a); break;
    case Epi::Cg: k_dense_finish<Epi::Cg><<<g, b, 0, s>>>(d, a); break;
    case Epi::Rich: k_dense_finish<Epi::Rich><<<g, b, 0, s>>>(d, a); break;
    case Epi::Gram: k_dense_finish<Epi::Gram><<<g, b, 0, s>>>(d, a); break;
  }
}
}  // namespace

void launch_dense_ata(const DenseDev& d, const double* v, int ring_stride, const KrylovScalars* sc, Epi epi,
                      const XtArgs& a, cudaStream_t s) {
  if (d.rows == 0 || d.cols == 0) return;
  dense_sweep<0>(d, v, nullptr, nullptr, a.done, sc, ring_stride, s);
  dense_finish(d, epi, a, s);
  check_launch("dense_ata");
}

void launch_dense_spmv(const DenseDev& d, const double* v, double* y, cudaStream_t s) {
  if (d.rows == 0) return;
  dense_sweep<2>(d, v, nullptr, y, nullptr, nullptr, 0, s);
  check_launch("dense_spmv");
}

void launch_dense_xt(const DenseDev& d, const double* u, Epi epi, const XtArgs& a, cudaStream_t s) {
  if (d.cols == 0) return;
  dense_sweep<1>(d, nullptr, u, nullptr, a.done, nullptr, 0, s);
  dense_finish(d, epi, a, s);
  check_launch("dense_xt");
}

void launch_dense_diag(const DenseDev& d, double beta, double* out, cudaStream_t s) {
  if (d.cols == 0) return;
  dense_sweep<3>(d, nullptr, nullptr, nullptr, nullptr, nullptr, 0, s);
  XtArgs a;
  a.out = out;
  dense_finish(d, Epi::Plain, a, s);
  k_add_const<<<grid_for(d.cols, 148), kThreads, 0, s>>>(out, beta, d.cols);
  check_launch("dense_diag");
}


// RMG_BLOCK_HOT: V rows kept in shared memory by the K1 pass (0 disables)
int64_t block_hot_rows() {
  static int64_t rows = -1;
  if (rows < 0) {
    const char* e = std::getenv("RMG_BLOCK_HOT");
    rows = e != nullptr ? std::max<int64_t>(0, std::atoll(e)) : 0;  // measured slower on cfg 3
    rows = std::min<int64_t>(rows, 1700);  // <= 212 KB of shared memory
  }
  return rows;
}

template <bool PAT, bool NARROW>
void spmm_hot(int grid, size_t smem, cudaStream_t s, const SparseDev& x, const double* vk, double* t,
              const BlockXtSchedule& bs, int k, int c0, int kc, int n_hot) {
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(k_spmm_sell<PAT, NARROW, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, 1700 * 128);
    attr = true;
  }
  k_spmm_sell<PAT, NARROW, true><<<grid, 512, smem, s>>>(x.sell_off, x.sell_row, x.sell_len, x.idx, x.idx16, x.val, vk,
                                                         t, bs.slice0, bs.n_slices, k, c0, kc, n_hot, 0);
}

// RMG_BLOCK_K1V2=0: the round-2 split K1 (k_spmm_hot + cold SELL pass) instead of the
// record-streaming fused pass (read once: the layouts are built accordingly)
int block_k1v2_mode() {
  static int mode = -1;
  if (mode < 0) {
    const char* e = std::getenv("RMG_BLOCK_K1V2");
    mode = e != nullptr ? std::max(0, std::min(2, std::atoi(e))) : 2;
  }
  return mode;
}

constexpr int kK1Threads = 768, kK1Depth = 3;  // measured: 512 / 7 1149 us, 640 / 5 1132, 768 / 3 1120 per apply

template <bool PAT, bool VEC>
void spmm_k1v3(int sms, cudaStream_t s, const BlockK1v2& h, const double* vk, int k, int c0, int kc, int64_t s0,
               int64_t s1, double* t) {
  static bool attr = false;
  const size_t smem = static_cast<size_t>(h.H1 + 1) * 128 +
                      static_cast<size_t>(kK1Threads / 32) * (kK1Depth + 1) * (PAT ? 128 : 384);
  if (!attr) {
    cudaFuncSetAttribute(k_spmm_k1v3<PAT, VEC, kK1Threads, kK1Depth>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         227 * 1024);
    attr = true;
  }
  k_spmm_k1v3<PAT, VEC, kK1Threads, kK1Depth><<<sms, kK1Threads, smem, s>>>(h, vk, k, c0, kc, s0, s1, t);
}

void launch_ridge_block(const SparseDev& x, const SparseDev& xt, const BlockXtSchedule* chunks, int n_chunks,
                        const BlockHot& hot, const BlockHotK1& hot1, const BlockK1v2& k1v2, const double* v,
                        double* out, double beta, int k, double* t, double* vp, cudaStream_t s, bool xt_only) {
  if (x.rows == 0 || x.cols == 0 || k <= 0) return;
  if (x.sell_off == nullptr) throw std::runtime_error("block operator: needs the SELL layout of X");
  // TMA gather passes (spmm_tma.cu) when V and T rows are 16-byte aligned
  if (xt_only && beta != 0.0) throw std::runtime_error("block X^T pass: beta must be 0");
  if (!xt_only && n_chunks > 0 && chunks[0].tk1.units != nullptr && tma_spmm_ok(v, k) && tma_spmm_ok(t, k)) {
    for (int c0 = 0; c0 < k; c0 += kBlockCols) {
      const int kc = std::min(kBlockCols, k - c0);
      for (int c = 0; c < n_chunks; ++c) {
        const BlockXtSchedule& bs = chunks[c];
        const int first = c == 0, last = c + 1 == n_chunks;
        launch_spmm_tma_rows(bs.tk1, v, x.cols, k, c0, kc, t, s);
        launch_spmm_tma_xt(bs.tk2, t, x.rows, k, c0, kc, out, v, beta, bs.seg, first, last, s);
        if (bs.n_multi > 0)
          k_block_finish<<<static_cast<int>((static_cast<int64_t>(bs.n_multi) * 32 + 255) / 256), 256, 0, s>>>(
              bs, v, out, beta, k, c0, kc, first, last);
      }
    }
    check_launch("ridge_block_tma");
    return;
  }
  const double* vk = v;
  if (!xt_only && x.col_inv != nullptr) {  // relabeled columns: V rows into label order
    k_vperm_block<<<grid_for(x.cols * k, 148 * 8), kThreads, 0, s>>>(v, x.col_inv, vp, x.cols, k);
    vk = vp;
  }
  for (int c0 = 0; c0 < k; c0 += kBlockCols) {
    const int kc = std::min(kBlockCols, k - c0);
    for (int c = 0; c < n_chunks; ++c) {
      const BlockXtSchedule& bs = chunks[c];
      const int first = c == 0, last = c + 1 == n_chunks;
      const int g1 = grid_for(bs.n_slices * 32, 148 * 8);
      const int64_t units = static_cast<int64_t>(bs.n_short) + bs.n_items;  // one half-warp each
      const int g2 = static_cast<int>(std::max<int64_t>(1, (units * 16 + kThreads - 1) / kThreads));
      if (xt_only) {
        // t holds the caller's N x k block: only the X^T half runs
      } else if (bs.n_slices > 0 && k1v2.H1 > 0 && x.col_inv != nullptr) {
        // K1 fused: hot labels from shared memory, cold ones gathered, records streamed
        int sms = 148;
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
        const int64_t s0 = bs.slice0 * 4, s1 = std::min<int64_t>(k1v2.n_slices8, (bs.slice0 + bs.n_slices) * 4);
        const bool vec = kc == 16 && (k & 1) == 0;
        if (k1v2.pattern) {
          if (vec)
            spmm_k1v3<true, true>(sms, s, k1v2, vk, k, c0, kc, s0, s1, t);
          else
            spmm_k1v3<true, false>(sms, s, k1v2, vk, k, c0, kc, s0, s1, t);
        } else {
          if (vec)
            spmm_k1v3<false, true>(sms, s, k1v2, vk, k, c0, kc, s0, s1, t);
          else
            spmm_k1v3<false, false>(sms, s, k1v2, vk, k, c0, kc, s0, s1, t);
        }
      } else if (bs.n_slices > 0 && hot1.H1 > 0 && x.col_inv != nullptr) {
        // K1 split: hot labels from shared memory (T written), cold SELL pass adds
        const int64_t r0 = bs.slice0 * 32, r1 = std::min<int64_t>(x.rows, (bs.slice0 + bs.n_slices) * 32);
        static bool attr1 = false;
        if (!attr1) {
          cudaFuncSetAttribute(k_spmm_hot<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, 210 * 1024);
          cudaFuncSetAttribute(k_spmm_hot<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, 210 * 1024);
          attr1 = true;
        }
        int sms = 148;
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
        const size_t hsm = static_cast<size_t>(hot1.H1) * 16 * sizeof(double);
        if (hot1.val == nullptr)
          k_spmm_hot<true><<<sms, 1024, hsm, s>>>(hot1, vk, k, c0, kc, r0, r1, t);
        else
          k_spmm_hot<false><<<sms, 1024, hsm, s>>>(hot1, vk, k, c0, kc, r0, r1, t);
        const SparseDev& xc = hot1.cold;
        const int gc = grid_for(bs.n_slices * 32, 148 * 8);
        if (xc.val == nullptr) {
          if (xc.idx16 != nullptr)
            k_spmm_sell<true, true, false><<<gc, kThreads, 0, s>>>(xc.sell_off, xc.sell_row, xc.sell_len, xc.idx,
                                                                   xc.idx16, xc.val, v, t, bs.slice0, bs.n_slices, k,
                                                                   c0, kc, 0, 1);
          else
            k_spmm_sell<true, false, false><<<gc, kThreads, 0, s>>>(xc.sell_off, xc.sell_row, xc.sell_len, xc.idx,
                                                                    xc.idx16, xc.val, v, t, bs.slice0, bs.n_slices, k,
                                                                    c0, kc, 0, 1);
        } else {
          if (xc.idx16 != nullptr)
            k_spmm_sell<false, true, false><<<gc, kThreads, 0, s>>>(xc.sell_off, xc.sell_row, xc.sell_len, xc.idx,
                                                                    xc.idx16, xc.val, v, t, bs.slice0, bs.n_slices, k,
                                                                    c0, kc, 0, 1);
          else
            k_spmm_sell<false, false, false><<<gc, kThreads, 0, s>>>(xc.sell_off, xc.sell_row, xc.sell_len, xc.idx,
                                                                     xc.idx16, xc.val, v, t, bs.slice0, bs.n_slices,
                                                                     k, c0, kc, 0, 1);
        }
      } else if (bs.n_slices > 0) {
        // hot V rows in shared memory when the columns are relabeled by popularity
        const int n_hot = x.col_inv != nullptr ? static_cast<int>(std::min<int64_t>(x.cols, block_hot_rows())) : 0;
        const size_t hsm = static_cast<size_t>(n_hot) * 16 * sizeof(double);
        if (n_hot > 0) {
          int sms = 148;
          cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
          const int gh = static_cast<int>(std::min<int64_t>(sms, (bs.n_slices + 15) / 16));
          if (x.val == nullptr) {
            if (x.idx16 != nullptr)
              spmm_hot<true, true>(gh, hsm, s, x, vk, t, bs, k, c0, kc, n_hot);
            else
              spmm_hot<true, false>(gh, hsm, s, x, vk, t, bs, k, c0, kc, n_hot);
          } else {
            if (x.idx16 != nullptr)
              spmm_hot<false, true>(gh, hsm, s, x, vk, t, bs, k, c0, kc, n_hot);
            else
              spmm_hot<false, false>(gh, hsm, s, x, vk, t, bs, k, c0, kc, n_hot);
          }
        } else if (x.val == nullptr) {
          if (x.idx16 != nullptr)
            k_spmm_sell<true, true, false><<<g1, kThreads, 0, s>>>(x.sell_off, x.sell_row, x.sell_len, x.idx, x.idx16,
                                                                   x.val, vk, t, bs.slice0, bs.n_slices, k, c0, kc, 0, 0);
          else
            k_spmm_sell<true, false, false><<<g1, kThreads, 0, s>>>(x.sell_off, x.sell_row, x.sell_len, x.idx,
                                                                    x.idx16, x.val, vk, t, bs.slice0, bs.n_slices, k,
                                                                    c0, kc, 0, 0);
        } else {
          if (x.idx16 != nullptr)
            k_spmm_sell<false, true, false><<<g1, kThreads, 0, s>>>(x.sell_off, x.sell_row, x.sell_len, x.idx,
                                                                    x.idx16, x.val, vk, t, bs.slice0, bs.n_slices, k,
                                                                    c0, kc, 0, 0);
          else
            k_spmm_sell<false, false, false><<<g1, kThreads, 0, s>>>(x.sell_off, x.sell_row, x.sell_len, x.idx,
                                                                     x.idx16, x.val, vk, t, bs.slice0, bs.n_slices, k,
                                                                     c0, kc, 0, 0);
        }
      }
      if (units > 0) {
        if (xt.val == nullptr)
          k_xt_block<true><<<g2, kThreads, 0, s>>>(xt.ptr, xt.idx, xt.val, bs, t, v, out, beta, k, c0, kc, first, last);
        else
          k_xt_block<false><<<g2, kThreads, 0, s>>>(xt.ptr, xt.idx, xt.val, bs, t, v, out, beta, k, c0, kc, first,
                                                    last);
      }
      if (bs.n_multi > 0)
        k_block_finish<<<static_cast<int>((static_cast<int64_t>(bs.n_multi) * 32 + 255) / 256), 256, 0, s>>>(
            bs, v, out, beta, k, c0, kc, first, last);
    }
    if (hot.H > 0) {  // hot features: from shared-memory T blocks, then folded
      const size_t smem = static_cast<size_t>(hot.R + 1) * 128 +
                          static_cast<size_t>(kHotBlkThreads / 32) * (kHotBlkDepth + 1) * (hot.pattern ? 128 : 384);
      static bool attr = false;
      if (!attr) {
        cudaFuncSetAttribute(k_xt_hotblk<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
        cudaFuncSetAttribute(k_xt_hotblk<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
        attr = true;
      }
      if (hot.pattern)
        k_xt_hotblk<true><<<hot.nblk, kHotBlkThreads, smem, s>>>(hot, t, k, c0, kc, x.rows);
      else
        k_xt_hotblk<false><<<hot.nblk, kHotBlkThreads, smem, s>>>(hot, t, k, c0, kc, x.rows);
      k_hot_fold<<<hot.H, kFoldSubs * 16, 0, s>>>(hot, v, out, beta, k, c0, kc);
    }
  }
  check_launch("ridge_block");
}

}  // namespace rmg
