// Persistent inner solver for small coarse levels.
//
// A coarse level k >= 1 of the hierarchy is solved by an inner FCG (or CG)
// to tolerance 1e-6 at every outer iteration (krylov.cpp:395-410).  On cfg 2
// that is F_1 = 2000 unknowns and ~150 inner iterations per outer step: the
// work per iteration is tiny and launch/sync latency dominated.  B200 layout:
//   * the Galerkin operator is held densely, A_k = X_k^T X_k + beta_k I
//     (mathematically GalerkinOperator::apply, coarsening.cpp:174-185);
//   * with a direct coarsest level below, the level-k preconditioner
//     (krylov.cpp:379-420) is the fixed linear map
//         z = omega r + Q (P^T r),   Q = (I - omega A_k) P A_{k+1}^{-1}  (n x nc)
//     with Q precomputed once.  The level's unknowns are held in next-level
//     cluster order, so P^T r is a sum of per-CTA segment partials: each CTA
//     scans its owned rows by cluster right after its r update (before the
//     barrier that already ends the iteration) and every CTA gathers the
//     ~grid + nc partials at the next z step.  Per iteration a CTA streams
//     its n_c-wide rows of Q (22 KB on cfg 2) instead of n-wide rows of the
//     dense M = Q P^T (224 KB; the fallback when nc exceeds the scratch);
//   * one cooperative launch runs the whole inner solve: <= 148 CTAs x 256
//     threads, each CTA owns a contiguous block of rows, keeps its rows of A_k
//     resident in shared memory when they fit (2000 x 2000 fp64 = 32 MB
//     = 143 x 219 KB) and streams its rows of M from L2;
//   * 4 grid barriers per iteration; every other step is spread over the
//     CTA's threads (measured with tools/microbench_*.cu: serial per-row
//     sections and 1024-thread CTAs were barrier-stall bound).
// Reductions are deterministic: every CTA publishes a per-block partial and
// every CTA re-reduces all partials in the same fixed order; the FCG direction
// update subtracts the Gram-Schmidt terms in the reference's order.
#include <cooperative_groups.h>

#include <algorithm>
#include <cstdlib>
#include <stdexcept>
#include <string>

#include "dense_level.cuh"

namespace cg = cooperative_groups;

namespace rmg {

namespace {

constexpr int kT = 256;
constexpr int kW = kT / 32;
// partial slots per block: [0] ||b||^2, [1] #non-finite, [2..33] GS, [34] pap, [35] pr, [36] rr;
// 64 doubles = 512 B per CTA so every CTA's slots start on their own L2 line group
constexpr int kPS = 80;
constexpr int kGS = 2, kPAP = 34, kPR = 35, kRR = 36;
// two-barrier kernel: ||r||^2 and the Gram-Schmidt dots are one contiguous run
constexpr int kRR2 = 40, kGS2 = 41;  // 41..71
constexpr int kMaxQ = 16;  // n <= 4096 columns = 16 per thread
constexpr int kMaxUse = 32;

__device__ __forceinline__ double wsum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Block sum of one value per thread, result broadcast to every thread.
__device__ __forceinline__ double bsum_all(double v, double* sh) {
  v = wsum(v);
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  __syncthreads();
  if (lane == 0) sh[wid] = v;
  __syncthreads();
  double r = 0.0;
#pragma unroll
  for (int w = 0; w < kW; ++w) r += sh[w];
  return r;
}

// Cross-CTA partials are slot-major, partials[slot * stride + cta]: a reduced
// quantity is one contiguous run of gridDim.x doubles (coalesced for the warp
// that sums it); measured: the CTA-major layout (one line per CTA) put a
// placement-dependent 25% on every inner iteration.
__device__ __forceinline__ int slot_stride() { return (gridDim.x + 31) & ~31; }

// out[q] = sum over blocks b (fixed order) of partials[first + q][b], q < count,
// one warp per quantity; ends with __syncthreads so every thread may read out.
__device__ __forceinline__ void grid_sums(const double* partials, int first, int count, double* out) {
  // All loads of a warp's (up to 4) quantities are issued before any add, so
  // the sums cost one L2 round trip instead of one per quantity; per lane the
  // order (b = lane, lane + 32, ...) and the warp tree are unchanged.
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int stride = slot_stride(), nb = gridDim.x;
  for (int q0 = wid; q0 < count; q0 += 4 * kW) {
    double x[4][8];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int q = q0 + j * kW;
      const double* row = partials + (size_t)(first + q) * stride;  // slot-major: grid contiguous doubles
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int b = lane + 32 * u;
        x[j][u] = (q < count && b < nb) ? __ldcg(row + b) : 0.0;
      }
    }
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      double acc = 0.0;
#pragma unroll
      for (int u = 0; u < 8; ++u)
        if (lane + 32 * u < nb) acc += x[j][u];
      acc = wsum(acc);
      if (lane == 0 && q0 + j * kW < count) out[q0 + j * kW] = acc;
    }
  }
  __syncthreads();
}

// Row sums of (rows x v) for the nr owned rows; rows is nr x n row-major
// (shared or global), v held as vc[q] = v[tid + q*kT].  Result in out[lr]
// (fixed-order combine of the kW warp partials).
template <bool GLOBAL>
__device__ __forceinline__ void gemv_rows(const double* rows, int nr, int n, const double (&vc)[kMaxQ], double* red,
                                          double* out) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, tid = threadIdx.x;
  for (int lr0 = 0; lr0 < nr; lr0 += 4) {
    double acc[4] = {0.0, 0.0, 0.0, 0.0};
    // branch-free over the 4 rows (clamped to the last owned row; surplus
    // sums are discarded) so all 4 x kMaxQ loads can be in flight at once
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const double* row = rows + (size_t)min(lr0 + u, nr - 1) * n;
#pragma unroll
      for (int q = 0; q < kMaxQ; ++q) {
        const int c = tid + q * kT;
        if (c < n) acc[u] += (GLOBAL ? __ldg(row + c) : row[c]) * vc[q];
      }
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const double s = wsum(acc[u]);
      if (lane == 0 && lr0 + u < nr) red[(lr0 + u) * kW + wid] = s;
    }
  }
  __syncthreads();
  if (tid < nr) {
    double s = 0.0;
#pragma unroll
    for (int w = 0; w < kW; ++w) s += red[tid * kW + w];
    out[tid] = s;
  }
  __syncthreads();
}

// Low-rank preconditioner: partial sums of w r over the owned rows, one per
// (CTA, cluster) segment, by warp 0 (owned rows <= 28 = lanes).  Segmented
// inclusive warp scan in cluster order; the segment's last lane stores it.
// The per-lane layout (weight, head / end flags, segment slot) is constant for
// the solve and computed once.
struct SegLane {
  double w = 0.0;
  bool head = false, end = false;
  int slot = -1;
};

__device__ __forceinline__ SegLane segment_layout(const DenseKrylovArgs& a, int row0, int nr) {
  SegLane L;
  const int lane = threadIdx.x & 31;
  const bool own = lane < nr;
  const int cl = own ? a.cid[row0 + lane] : -1;
  const int prevc = __shfl_up_sync(0xffffffffu, cl, 1);
  const int nextc = __shfl_down_sync(0xffffffffu, cl, 1);
  L.head = own && (lane == 0 || prevc != cl);
  L.end = own && (lane == nr - 1 || nextc != cl);
  const unsigned heads = __ballot_sync(0xffffffffu, L.head);
  L.slot = a.cta_seg0[blockIdx.x] + __popc(heads & ((2u << lane) - 1u)) - 1;
  L.w = own ? a.wts[row0 + lane] : 0.0;
  return L;
}

__device__ __forceinline__ void segment_partials(const SegLane& L, double ri, double* dst) {
  const int lane = threadIdx.x & 31;
  double v = L.w * ri;
  bool f = L.head;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const double y = __shfl_up_sync(0xffffffffu, v, d);
    const bool g = __shfl_up_sync(0xffffffffu, f, d);
    if (lane >= d && !f) {
      v += y;
      f = g;
    }
  }
  if (L.end) dst[L.slot] = v;
}

// Narrow GEMV for the low-rank preconditioner (nc <= kT columns, nr <= 28
// rows): thread tid owns column tid; its rows' entries q[] are loaded by the
// caller ahead of the cluster sums (one overlapped L2 round trip instead of
// one per 4-row chunk).  Result in out[lr] (fixed-order warp combine).
__device__ __forceinline__ void gemv_narrow(const double (&q)[28], int nr, double sv, double* red, double* out) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, tid = threadIdx.x;
#pragma unroll
  for (int lr = 0; lr < 28; ++lr) {
    if (lr >= nr) break;
    const double s = wsum(q[lr] * sv);
    if (lane == 0) red[lr * kW + wid] = s;
  }
  __syncthreads();
  if (tid < nr) {
    double s = 0.0;
#pragma unroll
    for (int w = 0; w < kW; ++w) s += red[tid * kW + w];
    out[tid] = s;
  }
  __syncthreads();
}


// Warp reduce-scatter of NR (16 or 32) per-lane row partials: after it lane L
// holds the warp sum of row L >> (NR == 16 ? 1 : 0) in acc[0] (16: lanes 2r and
// 2r + 1 both hold row r).  NR - 1 shuffles instead of 5 NR for NR warp trees;
// fixed order, deterministic.
template <int NR>
__device__ __forceinline__ double warp_rows_sum(double (&acc)[NR]) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int w = NR / 2, off = 16; w >= 1; w >>= 1, off >>= 1) {
    const bool hi = (lane & off) != 0;
#pragma unroll
    for (int k = 0; k < w; ++k) {
      const double send = hi ? acc[k] : acc[k + w];
      const double keep = hi ? acc[k + w] : acc[k];
      acc[k] = keep + __shfl_xor_sync(0xffffffffu, send, off);
    }
  }
  if (NR == 16) acc[0] += __shfl_xor_sync(0xffffffffu, acc[0], 1);
  return acc[0];
}

// Row sums of (rows x v) for nr <= 32 owned rows, all rows' loads in flight at
// once and one reduce-scatter per warp (gemv_rows does 4 rows and 4 warp trees
// at a time).  Same contract as gemv_rows.
template <bool GLOBAL, int NQ>
__device__ __forceinline__ void gemv_rows_rs(const double* rows, int nr, int n, const double (&vc)[NQ], double* red,
                                             double* out) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, tid = threadIdx.x;
  for (int lr0 = 0; lr0 < nr; lr0 += 16) {
    double acc[16];
#pragma unroll
    for (int u = 0; u < 16; ++u) acc[u] = 0.0;
#pragma unroll
    for (int q = 0; q < NQ; ++q) {
      const int c = tid + q * kT;
      if (c < n) {
#pragma unroll
        for (int u = 0; u < 16; ++u) {
          const double* row = rows + (size_t)min(lr0 + u, nr - 1) * n;
          acc[u] += (GLOBAL ? __ldg(row + c) : row[c]) * vc[q];
        }
      }
    }
    const double sr = warp_rows_sum<16>(acc);
    const int lr = lr0 + (lane >> 1);
    if ((lane & 1) == 0 && lr < nr) red[lr * kW + wid] = sr;
  }
  __syncthreads();
  if (tid < nr) {
    double s = 0.0;
#pragma unroll
    for (int w = 0; w < kW; ++w) s += red[tid * kW + w];
    out[tid] = s;
  }
  __syncthreads();
}

// gemv_rows_rs with column pairs (n even): thread tid owns columns 2 tid + 2 kT p
// and the next one, read as one 16-byte load (half the load instructions); the
// pairs' products are added in column order.
template <bool GLOBAL, int NP>
__device__ __forceinline__ void gemv_rows_rs2(const double* rows, int nr, int n, const double (&vc)[2 * NP],
                                              double* red, double* out) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, tid = threadIdx.x;
  for (int lr0 = 0; lr0 < nr; lr0 += 16) {
    double acc[16];
#pragma unroll
    for (int u = 0; u < 16; ++u) acc[u] = 0.0;
#pragma unroll
    for (int p = 0; p < NP; ++p) {
      const int c = 2 * tid + p * 2 * kT;
      if (c < n) {
#pragma unroll
        for (int u = 0; u < 16; ++u) {
          const double* row = rows + (size_t)min(lr0 + u, nr - 1) * n;
          const double2 x = GLOBAL ? __ldg(reinterpret_cast<const double2*>(row + c))
                                   : *reinterpret_cast<const double2*>(row + c);
          acc[u] += x.x * vc[2 * p];
          acc[u] += x.y * vc[2 * p + 1];
        }
      }
    }
    const double sr = warp_rows_sum<16>(acc);
    const int lr = lr0 + (lane >> 1);
    if ((lane & 1) == 0 && lr < nr) red[lr * kW + wid] = sr;
  }
  __syncthreads();
  if (tid < nr) {
    double s = 0.0;
#pragma unroll
    for (int w = 0; w < kW; ++w) s += red[tid * kW + w];
    out[tid] = s;
  }
  __syncthreads();
}

// gemv_narrow with the reduce-scatter (nr <= RM: 16 or 28).
template <int RM>
__device__ __forceinline__ void gemv_narrow_rs(const double (&q)[RM], int nr, double sv, double* red, double* out) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, tid = threadIdx.x;
  if (RM <= 16) {
    double acc[16];
#pragma unroll
    for (int u = 0; u < 16; ++u) acc[u] = q[u < RM ? u : 0] * sv;
    const double s = warp_rows_sum<16>(acc);
    if ((lane & 1) == 0 && (lane >> 1) < nr) red[(lane >> 1) * kW + wid] = s;
  } else {
    double acc[32];
#pragma unroll
    for (int u = 0; u < 32; ++u) acc[u] = u < RM ? q[u < RM ? u : 0] * sv : 0.0;
    const double s = warp_rows_sum<32>(acc);
    if (lane < nr) red[lane * kW + wid] = s;
  }
  __syncthreads();
  if (tid < nr) {
    double s = 0.0;
#pragma unroll
    for (int w = 0; w < kW; ++w) s += red[tid * kW + w];
    out[tid] = s;
  }
  __syncthreads();
}

// Optional phase timing (diagnostics): %globaltimer of CTA 0 at phase marks
// of the first 16 iterations, when args.timing != nullptr.
__device__ __forceinline__ void tmark(const DenseKrylovArgs& a, int it, int idx) {
  if (a.timing != nullptr && it < 16 && blockIdx.x == 0 && threadIdx.x == 0) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    a.timing[it * 16 + idx] = t;
  }
}

template <bool SMEM>
__global__ void __launch_bounds__(kT, 1) k_dense_krylov(DenseKrylovArgs a) {
  cg::grid_group grid = cg::this_grid();
  extern __shared__ double smem[];
  const int n = a.n, R = a.rows_per_cta;
  const int row0 = blockIdx.x * R;
  const int row1 = min(n, row0 + R);
  const int nr = max(0, row1 - row0);
  // shared layout: [A rows: R*n if SMEM][red: R*kW][zs: R][v: R][contrib: R*kMaxUse][gsum: 64][coef: kMaxUse][sh: kW]
  double* As = smem;
  double* red = smem + (SMEM ? (size_t)R * n : 0);
  double* zs = red + (size_t)R * kW;
  double* vv = zs + R;
  double* contrib = vv + R;
  double* gsum = contrib + (size_t)R * kMaxUse;
  double* coef = gsum + 64;
  double* sh = coef + kMaxUse;
  const int tid = threadIdx.x;
  const int pstride = slot_stride();
  auto part = [&](int slot) -> double& { return a.partials[(size_t)slot * pstride + blockIdx.x]; };
  KrylovScalars* sc = a.sc;
  const double* Arows = SMEM ? As : a.A + (size_t)row0 * n;
  const double* Mrows = a.M + (size_t)row0 * (a.lowrank ? a.nc : n);
  auto orig = [&](int i) { return a.perm != nullptr ? a.perm[i] : i; };

  if (SMEM) {
    for (int idx = tid; idx < nr * n; idx += kT) As[idx] = a.A[(size_t)row0 * n + idx];
  }
  // ---- begin: x = 0, r = b, ||b|| (krylov.cpp:164-176)
  double bb = 0.0, bad = 0.0;
  for (int i = row0 + tid; i < row1; i += kT) {
    const double bi = a.b[orig(i)];
    a.x[i] = 0.0;
    a.r[i] = bi;
    bb += bi * bi;
    if (!isfinite(bi)) bad += 1.0;
  }
  SegLane seg;
  if (a.lowrank && tid < 32) {
    seg = segment_layout(a, row0, nr);
    segment_partials(seg, tid < nr ? a.b[orig(row0 + tid)] : 0.0, a.spart);
  }
  bb = bsum_all(bb, sh);
  bad = bsum_all(bad, sh);
  if (tid == 0) {
    part(0) = bb;
    part(1) = bad;
  }
  grid.sync();
  grid_sums(a.partials, 0, 2, gsum);
  const double nb = sqrt(gsum[0]);
  const double nbad = gsum[1];
  if (nbad > 0.0 || nb == 0.0) {
    if (blockIdx.x == 0 && tid == 0) {
      sc->it = 0;
      sc->status = nbad > 0.0 ? 3 : 0;
      sc->converged = nbad > 0.0 ? 0 : 1;
      sc->done = 1;
      sc->rel = nbad > 0.0 ? 1.0 : 0.0;
      sc->nb = nb;
      if (nbad == 0.0) a.hist[0] = 0.0;
    }
    if (a.x_out != a.x)
      for (int i = row0 + tid; i < row1; i += kT) a.x_out[orig(i)] = 0.0;
    return;
  }
  const int keep = a.keep, RING = keep + 1;
  const double omega = a.omega;
  double rz = nb * nb;  // CG: <r, z> with z = r
  double beta_cg = 0.0;
  int it = 0;
  bool converged = false;
  int status = 0;
  double rel = 1.0;
  for (; it < a.max_iters; ++it) {
    const int slot = it % RING;
    double* p_now = a.p_ring + (size_t)slot * n;
    double* ap_now = a.ap_ring + (size_t)slot * n;
    tmark(a, it, 0);
    // ---- z = M^{-1} r for the owned rows: omega r + M r (FCG) or r (CG)
    if (a.fcg) {
      if (a.dbg & 1) {
        if (tid < nr) vv[tid] = 0.0;
        __syncthreads();
      } else if (a.lowrank) {  // S = P^T r from the segment partials, then Q S
        if (a.nc <= kT) {
          double q[28];  // this thread's column of the owned rows of Q, in flight first
#pragma unroll
          for (int lr = 0; lr < 28; ++lr)
            q[lr] = (lr < nr && tid < a.nc) ? __ldg(Mrows + (size_t)lr * a.nc + tid) : 0.0;
          for (int g = tid; g < a.n_segments; g += kT) contrib[g] = __ldcg(a.spart + g);  // one coalesced pass
          __syncthreads();
          double sum = 0.0;
          if (tid < a.nc)
            for (int g = __ldg(a.cseg + tid); g < __ldg(a.cseg + tid + 1); ++g) sum += contrib[g];
          gemv_narrow(q, nr, sum, red, vv);
        } else {
          for (int g = tid; g < a.n_segments; g += kT) contrib[g] = __ldcg(a.spart + g);
          __syncthreads();
          double sv[kMaxQ];
#pragma unroll
          for (int q = 0; q < kMaxQ; ++q) {
            const int c = tid + q * kT;
            double sum = 0.0;
            if (c < a.nc)
              for (int g = __ldg(a.cseg + c); g < __ldg(a.cseg + c + 1); ++g) sum += contrib[g];
            sv[q] = sum;
          }
          gemv_rows<true>(Mrows, nr, a.nc, sv, red, vv);
        }
      } else {
        double rc[kMaxQ];
#pragma unroll
        for (int q = 0; q < kMaxQ; ++q) {
          const int c = tid + q * kT;
          rc[q] = c < n ? __ldcg(a.r + c) : 0.0;
        }
        gemv_rows<true>(Mrows, nr, n, rc, red, vv);
      }
      if (tid < nr) zs[tid] = omega * a.r[row0 + tid] + vv[tid];
    } else {
      if (tid < nr) zs[tid] = a.r[row0 + tid];
    }
    __syncthreads();
    tmark(a, it, 1);
    if (a.fcg) {
      // ---- classical Gram-Schmidt of z against the newest use = min(m_i, |hist|)
      // directions (krylov.cpp:189-197); coefficients from z, oldest -> newest
      const int mi = it == 0 ? 0 : max(1, it % (keep + 1));
      const int use = min(mi, min(it, keep));
      if (use > 0) {
        const int lane = tid & 31, wid = tid >> 5;
        // nr <= 28 (n <= 4096 over >= 148 CTAs): one element per lane; the
        // loads of a warp's (up to 4) directions are issued together
        double y[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const int q = wid + j * kW;
          const double* aph = a.ap_ring + (size_t)((it - use + q) % RING) * n;
          y[j] = (q < use && lane < nr) ? zs[lane] * __ldcg(aph + row0 + lane) : 0.0;
        }
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const double acc = wsum(y[j]);
          if (lane == 0 && wid + j * kW < use) part(kGS + wid + j * kW) = acc;
        }
        tmark(a, it, 2);
        grid.sync();  // B1
        tmark(a, it, 3);
        grid_sums(a.partials, kGS, use, gsum);
        if (tid < use) coef[tid] = gsum[tid] / __ldcg(a.pap_ring + (it - use + tid) % RING);
        __syncthreads();
        tmark(a, it, 4);
        for (int e = tid; e < nr * use; e += kT) {  // c_q p_q(row), all pairs in parallel
          const int lr = e / use, q = e - lr * use;
          contrib[lr * kMaxUse + q] = coef[q] * __ldcg(a.p_ring + (size_t)((it - use + q) % RING) * n + row0 + lr);
        }
        __syncthreads();
        if (tid < nr) {  // p = z - c_0 p_0 - c_1 p_1 - ... (reference order)
          double pi = zs[tid];
          for (int q = 0; q < use; ++q) pi -= contrib[tid * kMaxUse + q];
          zs[tid] = pi;
        }
      }
    } else if (it > 0) {  // CG: p = z + beta p_prev (krylov.cpp:145-153)
      const double* pprev = a.p_ring + (size_t)((it - 1) % RING) * n;
      if (tid < nr) zs[tid] = zs[tid] + beta_cg * __ldcg(pprev + row0 + tid);
    }
    if (tid < nr) p_now[row0 + tid] = zs[tid];
    tmark(a, it, 5);
    grid.sync();  // B2: p complete
    tmark(a, it, 6);
    // ---- Ap = A p for the owned rows; <p,Ap>, <p,r> (krylov.cpp:199-208)
    {
      double pc[kMaxQ];
#pragma unroll
      for (int q = 0; q < kMaxQ; ++q) {
        const int c = tid + q * kT;
        pc[q] = c < n ? __ldcg(p_now + c) : 0.0;
      }
      if (a.dbg & 2) {
        if (tid < nr) vv[tid] = zs[tid];  // ablation: A = I keeps pap > 0
        __syncthreads();
      } else if (SMEM) {
        gemv_rows<false>(Arows, nr, n, pc, red, vv);
      } else {
        gemv_rows<true>(Arows, nr, n, pc, red, vv);
      }
      tmark(a, it, 7);
      double dpap = 0.0, dpr = 0.0;
      if (tid < nr) {
        const double s = vv[tid];
        ap_now[row0 + tid] = s;
        dpap = zs[tid] * s;
        dpr = zs[tid] * a.r[row0 + tid];
      }
      dpap = bsum_all(dpap, sh);
      dpr = bsum_all(dpr, sh);
      if (tid == 0) {
        part(kPAP) = dpap;
        part(kPR) = dpr;
      }
    }
    tmark(a, it, 8);
    grid.sync();  // B3
    tmark(a, it, 9);
    grid_sums(a.partials, kPAP, 2, gsum);
    tmark(a, it, 10);
    const double pap = gsum[0], pr = gsum[1];
    if (a.fcg ? pap == 0.0 : false) {
      status = 1;
      break;
    }
    if (a.fcg ? pap < 0.0 : !(pap > 0.0)) {
      status = 2;
      break;
    }
    const double alpha = a.fcg ? pr / pap : rz / pap;
    if (blockIdx.x == 0 && tid == 0) a.pap_ring[slot] = pap;
    double rr = 0.0, ri = 0.0;
    if (tid < nr) {
      const int i = row0 + tid;
      a.x[i] += alpha * zs[tid];
      ri = a.r[i] - alpha * vv[tid];
      a.r[i] = ri;
      rr = ri * ri;
    }
    if (a.lowrank && tid < 32) segment_partials(seg, ri, a.spart);
    rr = bsum_all(rr, sh);
    if (tid == 0) part(kRR) = rr;
    tmark(a, it, 11);
    grid.sync();  // B4
    tmark(a, it, 12);
    grid_sums(a.partials, kRR, 1, gsum);
    tmark(a, it, 13);
    const double rrs = gsum[0];
    rel = sqrt(rrs) / nb;
    if (blockIdx.x == 0 && tid == 0) a.hist[it] = rel;
    if (rel <= a.tol) {
      converged = true;
      ++it;
      break;
    }
    if (!a.fcg) {  // CG: rz' = <r, r>, beta = rz'/rz (every CTA computes the same value)
      beta_cg = rrs / rz;
      rz = rrs;
    }
  }
  if (a.x_out != a.x)  // solution back to the original order
    for (int i = row0 + tid; i < row1; i += kT) a.x_out[orig(i)] = a.x[i];
  if (blockIdx.x == 0 && tid == 0) {
    sc->it = it;
    sc->status = status;
    sc->converged = converged ? 1 : 0;
    sc->done = 1;
    sc->rel = rel;
    sc->nb = nb;
  }
}

// Two grid barriers per iteration, for the low-rank FCG
// preconditioner and for plain CG.  Same iteration as k_dense_krylov
// (krylov.cpp:164-220), regrouped around two exchanges:
//   B1 publishes z (whole vector), ||r||^2 and the Gram-Schmidt dots <z, Ap_q>;
//      then Ap = A z - sum_q c_q Ap_q (CG: A z + beta Ap_prev) from the own rows
//      of the stored Ap history, so p never has to be exchanged, and
//      p = z - sum_q c_q p_q in the reference's order;
//   B3 publishes <p, Ap>, <p, r> and the segment partials of P^T Ap; after it
//      every CTA has alpha, updates its rows of x and r, and forms
//      P^T r_new = sum over segments of (P^T r_old - alpha P^T Ap) partials
//      (both sets of partials are per-iteration, so nothing is carried over
//      iterations and no recurrence drift builds up).
// The convergence test of r_k (||r_k||^2 rides on B1 of iteration k) runs half
// an iteration after the update; the iteration logic, history and breakdown
// exits are those of k_dense_krylov.  The A z row sums are a different
// (fixed) summation order per variant -- the PAIR variant (even n, A in SMEM)
// has thread tid sum columns 2 tid, 2 tid + 1, 2 tid + 2 kT, ...; the others
// columns tid, tid + kT, ... -- so inner rounding depends on the variant
// (tests/test_gpu_parity.py::test_pair_variant_within_bars holds both to the bars).  Own-row work (nr <= 28) is warp 0:
// its reductions are warp sums.
// HM >= truncation (history directions held per lane); NQ = columns per thread
// (n <= NQ * kT) and RM >= owned rows: compile-time so the unrolled loop body
// stays small enough for the instruction cache (measured: no_inst stalls at
// NQ = 16 on n = 2000).
template <bool SMEM, int HM, int NQ, bool PAIR = false>
__global__ void __launch_bounds__(kT, 1) k_dense_krylov2(DenseKrylovArgs a) {
  constexpr int RM = NQ <= 8 ? 16 : 28;
  cg::grid_group grid = cg::this_grid();
  extern __shared__ double smem[];
  const int n = a.n, R = a.rows_per_cta;
  const int row0 = blockIdx.x * R;
  const int row1 = min(n, row0 + R);
  const int nr = max(0, row1 - row0);
  double* As = smem;  // same layout as k_dense_krylov
  double* red = smem + (SMEM ? (size_t)R * n : 0);
  double* zs = red + (size_t)R * kW;
  double* vv = zs + R;
  double* contrib = vv + R;
  double* gsum = contrib + (size_t)R * kMaxUse;
  double* coef = gsum + 64;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int pstride = slot_stride();
  auto part = [&](int slot) -> double& { return a.partials[(size_t)slot * pstride + blockIdx.x]; };
  KrylovScalars* sc = a.sc;
  const double* Arows = SMEM ? As : a.A + (size_t)row0 * n;
  const double* Qrows = a.M + (size_t)row0 * a.nc;
  auto orig = [&](int i) { return a.perm != nullptr ? a.perm[i] : i; };
  const bool own = wid == 0 && lane < nr;
  const int i = row0 + lane;  // warp 0: lane lr holds row row0 + lr
  const int nseg = a.n_segments;
  // a.spart: [P^T r partials, even iterations | odd iterations | P^T Ap partials]
  double* spart_ap = a.spart + 2 * nseg;

  if (SMEM) {
    for (int idx = tid; idx < nr * n; idx += kT) As[idx] = a.A[(size_t)row0 * n + idx];
  }
  // ---- begin: x = 0, r = b, ||b|| (krylov.cpp:164-176)
  double ri = 0.0, xi = 0.0, pi = 0.0, api = 0.0;
  SegLane seg;
  if (wid == 0) {
    ri = own ? a.b[orig(i)] : 0.0;
    const double bb = wsum(ri * ri);
    const double bad = wsum(own && !isfinite(ri) ? 1.0 : 0.0);
    if (lane == 0) {
      part(0) = bb;
      part(1) = bad;
    }
    if (a.lowrank) {
      seg = segment_layout(a, row0, nr);
      segment_partials(seg, ri, a.spart);
    }
  }
  double q[RM];  // this thread's column of the owned rows of Q, held for the whole solve
#pragma unroll
  for (int lr = 0; lr < RM; ++lr)
    q[lr] = (a.lowrank && a.nc <= kT && lr < nr && tid < a.nc) ? __ldg(Qrows + (size_t)lr * a.nc + tid) : 0.0;
  int cs0 = 0, cs1 = 0;  // this thread's cluster segments (nc <= kT)
  if (a.lowrank && a.nc <= kT && tid < a.nc) {
    cs0 = __ldg(a.cseg + tid);
    cs1 = __ldg(a.cseg + tid + 1);
  }
  grid.sync();
  grid_sums(a.partials, 0, 2, gsum);
  const double nb = sqrt(gsum[0]);
  const double nbad = gsum[1];
  if (nbad > 0.0 || nb == 0.0) {
    if (blockIdx.x == 0 && tid == 0) {
      sc->it = 0;
      sc->status = nbad > 0.0 ? 3 : 0;
      sc->converged = nbad > 0.0 ? 0 : 1;
      sc->done = 1;
      sc->rel = nbad > 0.0 ? 1.0 : 0.0;
      sc->nb = nb;
      if (nbad == 0.0) a.hist[0] = 0.0;
    }
    if (own) {
      a.x_out[orig(i)] = 0.0;
      if (a.x_out != a.x) a.x[i] = 0.0;
    }
    return;
  }
  const int keep = a.keep, RING = keep + 1;
  const double omega = a.omega;
  double rz = nb * nb;  // CG: <r, z> with z = r
  double beta_cg = 0.0;
  int iters = 0, status = 0;
  bool converged = false;
  double rel = 1.0;
  for (int it = 0;; ++it) {
    tmark(a, it, 0);
    // ======== phase 1: alpha, x/r update (direction it-1), z_it
    const int mi = it == 0 ? 0 : max(1, it % (keep + 1));
    const int use = a.fcg ? min(mi, min(it, keep)) : 0;
    double ygs[4];  // own rows of the Ap_q for the Gram-Schmidt dots, in flight first
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int qd = wid + j * kW;
      ygs[j] = (qd < use && lane < nr) ? __ldcg(a.ap_ring + (size_t)((it - use + qd) % RING) * n + i) : 0.0;
    }
    double sg[2] = {0.0, 0.0}, sa[2] = {0.0, 0.0};
    if (a.lowrank) {
      const double* sp = a.spart + (it > 0 ? ((it - 1) & 1) * nseg : 0);
#pragma unroll
      for (int u = 0; u < 2; ++u) {
        const int g = tid + u * kT;
        if (g < nseg) {
          sg[u] = __ldcg(sp + g);
          if (it > 0) sa[u] = __ldcg(spart_ap + g);
        }
      }
    }
    double alpha = 0.0;
    if (it > 0) {
      grid_sums(a.partials, kPAP, 2, gsum);
      const double pap = gsum[0], pr = gsum[1];
      if (a.fcg ? pap == 0.0 : false) {
        status = 1;
        iters = it - 1;
        break;
      }
      if (a.fcg ? pap < 0.0 : !(pap > 0.0)) {
        status = 2;
        iters = it - 1;
        break;
      }
      alpha = a.fcg ? pr / pap : rz / pap;
      if (blockIdx.x == 0 && tid == 0) a.pap_ring[(it - 1) % RING] = pap;
      if (own) {
        xi += alpha * pi;
        ri = ri - alpha * api;
      }
    }
    tmark(a, it, 1);
    double zi = ri;  // CG: z = r
    if (a.lowrank) {  // z = omega r + Q (P^T r)
#pragma unroll
      for (int u = 0; u < 2; ++u) {
        const int g = tid + u * kT;
        if (g < nseg) contrib[g] = it > 0 ? sg[u] - alpha * sa[u] : sg[u];
      }
      if (it > 0 && wid == 0) segment_partials(seg, own ? ri : 0.0, a.spart + (it & 1) * nseg);
      __syncthreads();
      if (a.nc <= kT) {
        double sum = 0.0;
        for (int g = cs0; g < cs1; ++g) sum += contrib[g];
        gemv_narrow_rs<RM>(q, nr, sum, red, vv);
      } else {
        double sv[kMaxQ];
#pragma unroll
        for (int qq = 0; qq < kMaxQ; ++qq) {
          const int c = tid + qq * kT;
          double sum = 0.0;
          if (c < a.nc)
            for (int g = __ldg(a.cseg + c); g < __ldg(a.cseg + c + 1); ++g) sum += contrib[g];
          sv[qq] = sum;
        }
        gemv_rows<true>(Qrows, nr, a.nc, sv, red, vv);
      }
      if (own) zi = omega * ri + vv[lane];
    }
    tmark(a, it, 2);
    // ---- publish z, ||r||^2, Gram-Schmidt dots <z, Ap_q> (krylov.cpp:189-197)
    if (wid == 0) {
      if (own) {
        a.zfull[i] = zi;
        zs[lane] = zi;
      }
      const double rr = wsum(own ? ri * ri : 0.0);
      if (lane == 0) part(kRR2) = rr;
    }
    if (use > 0) {
      __syncthreads();
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const double acc = wsum(lane < nr ? zs[lane] * ygs[j] : 0.0);
        if (lane == 0 && wid + j * kW < use) part(kGS2 + wid + j * kW) = acc;
      }
    }
    tmark(a, it, 3);
    grid.sync();  // B1
    tmark(a, it, 4);
    // ======== phase 2: convergence of r_it; direction it
    double pc[NQ];
    if constexpr (PAIR) {  // columns 2 tid + 2 kT p and the next (gemv_rows_rs2)
#pragma unroll
      for (int p2 = 0; p2 < NQ / 2; ++p2) {
        const int c = 2 * tid + p2 * 2 * kT;
        const double2 zz = c < n ? __ldcg(reinterpret_cast<const double2*>(a.zfull + c)) : make_double2(0.0, 0.0);
        pc[2 * p2] = zz.x;
        pc[2 * p2 + 1] = zz.y;
      }
    } else {
#pragma unroll
      for (int qq = 0; qq < NQ; ++qq) {
        const int c = tid + qq * kT;
        pc[qq] = c < n ? __ldcg(a.zfull + c) : 0.0;
      }
    }
    double den = 1.0;
    if (tid < use) den = __ldcg(a.pap_ring + (it - use + tid) % RING);
    // own rows of the history: warp 0 loads the p_q, warp 1 the Ap_q
    double h[HM];
    {
      const bool hw = wid < 2 && lane < nr;
      const double* hb = wid == 0 ? a.p_ring : a.ap_ring;
      const int nh = a.fcg ? use : (it > 0 ? 1 : 0);
      int hs = (it - nh) % RING;
#pragma unroll
      for (int qd = 0; qd < HM; ++qd) {
        h[qd] = (hw && qd < nh) ? __ldcg(hb + (size_t)hs * n + i) : 0.0;
        hs = hs + 1 == RING ? 0 : hs + 1;
      }
    }
    grid_sums(a.partials, kRR2, 1 + use, gsum);
    tmark(a, it, 5);
    const double rrs = gsum[0];
    if (it > 0) {
      rel = sqrt(rrs) / nb;
      if (blockIdx.x == 0 && tid == 0) a.hist[it - 1] = rel;
      if (rel <= a.tol) {
        converged = true;
        iters = it;
        break;
      }
      if (!a.fcg) {  // CG: rz' = <r, r>, beta = rz'/rz
        beta_cg = rrs / rz;
        rz = rrs;
      }
    }
    if (it >= a.max_iters) {
      iters = it;
      break;
    }
    if (tid < use) coef[tid] = gsum[1 + tid] / den;
    // A z for the owned rows (ends with __syncthreads: coef and vv visible)
    if constexpr (PAIR)
      gemv_rows_rs2<!SMEM, NQ / 2>(Arows, nr, n, pc, red, vv);
    else
      gemv_rows_rs<!SMEM, NQ>(Arows, nr, n, pc, red, vv);
    tmark(a, it, 6);
    if (wid < 2) {  // warp 0: p = z - c_0 p_0 - c_1 p_1 - ... (reference order); warp 1: Ap alike
      double v = wid == 0 ? zi : (lane < nr ? vv[lane] : 0.0);
      if (a.fcg) {
#pragma unroll
        for (int qd = 0; qd < HM; ++qd)
          if (qd < use) v = v - __dmul_rn(coef[qd], h[qd]);
      } else if (it > 0) {  // CG: p = z + beta p_prev (krylov.cpp:145-153)
        v = v + beta_cg * h[0];
      }
      if (wid == 0) {
        pi = own ? v : 0.0;
      } else if (lane < nr) {
        vv[lane] = v;
      }
    }
    __syncthreads();
    if (wid == 0) {
      const int slot = it % RING;
      api = own ? vv[lane] : 0.0;
      if (own) {
        a.p_ring[(size_t)slot * n + i] = pi;
        a.ap_ring[(size_t)slot * n + i] = api;
      }
      const double dpap = wsum(pi * api);
      const double dpr = wsum(pi * ri);
      if (lane == 0) {
        part(kPAP) = dpap;
        part(kPR) = dpr;
      }
      if (a.lowrank) segment_partials(seg, api, spart_ap);
    }
    tmark(a, it, 7);
    grid.sync();  // B3
  }
  if (own) {  // solution back to the original order
    a.x_out[orig(i)] = xi;
    if (a.x_out != a.x) a.x[i] = xi;
    a.r[i] = ri;
  }
  if (blockIdx.x == 0 && tid == 0) {
    sc->it = iters;
    sc->status = status;
    sc->converged = converged ? 1 : 0;
    sc->done = 1;
    sc->rel = rel;
    sc->nb = nb;
  }
}

}  // namespace

DenseKrylovPlan plan_dense_krylov(int n, int nc, int device) {
  (void)nc;
  DenseKrylovPlan p;
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
  int max_smem = 0;
  cudaDeviceGetAttribute(&max_smem, cudaDevAttrMaxSharedMemoryPerBlockOptin, device);
  p.rows_per_cta = std::max(1, (n + sms - 1) / sms);
  p.grid = (n + p.rows_per_cta - 1) / p.rows_per_cta;
  const size_t R = p.rows_per_cta;
  const size_t extra = (R * kW + 2 * R + R * kMaxUse + 64 + kMaxUse + kW) * sizeof(double);
  const size_t with_a = extra + R * n * sizeof(double);
  p.smem_a = with_a <= (size_t)max_smem;
  if (const char* e = std::getenv("RMG_DENSE_SMEM")) p.smem_a = p.smem_a && e[0] != '0';
  p.smem_bytes = p.smem_a ? with_a : extra;
  p.partial_stride = kPS * ((p.grid + 31) / 32 * 32) / std::max(1, p.grid);
  p.max_clusters = p.rows_per_cta * kMaxUse;
  return p;
}

bool dense_two_barrier(const DenseKrylovArgs& a) {
  static const bool off = std::getenv("RMG_DENSE_4B") != nullptr;
  return !off && a.dbg == 0 && (a.fcg == 0 || (a.lowrank != 0 && a.n_segments <= 2 * kT)) && a.zfull != nullptr;
}

void launch_dense_krylov(const DenseKrylovPlan& plan, const DenseKrylovArgs& args, cudaStream_t s) {
  if (args.n > kMaxQ * kT) throw std::runtime_error("dense inner solver: level above 4096 unknowns");
  if (args.keep + 1 > kMaxUse) throw std::runtime_error("dense inner solver: truncation above 31");
  if (args.lowrank && args.n_segments > plan.max_clusters)
    throw std::runtime_error("dense inner solver: more cluster segments than shared scratch");
  if (plan.rows_per_cta > 32 || plan.grid > 256)  // one GS element per lane; grid_sums unroll
    throw std::runtime_error("dense inner solver: too few SMs for this level");
  void* fn = plan.smem_a ? (void*)k_dense_krylov<true> : (void*)k_dense_krylov<false>;
  if (dense_two_barrier(args)) {
    const bool small = args.n <= 8 * kT && plan.rows_per_cta <= 16;
    const bool h20 = args.keep <= 20;
    static const bool no_pair = std::getenv("RMG_DENSE_NO_PAIR") != nullptr;
    const bool pair = !no_pair && args.n % 2 == 0 && plan.smem_a && h20;
    if (pair)
      fn = small ? (void*)k_dense_krylov2<true, 20, 8, true> : (void*)k_dense_krylov2<true, 20, kMaxQ, true>;
    else if (small)
      fn = h20 ? (plan.smem_a ? (void*)k_dense_krylov2<true, 20, 8> : (void*)k_dense_krylov2<false, 20, 8>)
               : (plan.smem_a ? (void*)k_dense_krylov2<true, kMaxUse - 1, 8> : (void*)k_dense_krylov2<false, kMaxUse - 1, 8>);
    else
      fn = h20 ? (plan.smem_a ? (void*)k_dense_krylov2<true, 20, kMaxQ> : (void*)k_dense_krylov2<false, 20, kMaxQ>)
               : (plan.smem_a ? (void*)k_dense_krylov2<true, kMaxUse - 1, kMaxQ>
                              : (void*)k_dense_krylov2<false, kMaxUse - 1, kMaxQ>);
  }
  cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)plan.smem_bytes);
  if (e != cudaSuccess) throw std::runtime_error(std::string("dense inner solver attribute: ") + cudaGetErrorString(e));
  DenseKrylovArgs a = args;
  a.rows_per_cta = plan.rows_per_cta;
  void* kargs[] = {&a};
  e = cudaLaunchCooperativeKernel(fn, dim3(plan.grid), dim3(kT), kargs, plan.smem_bytes, s);
  if (e != cudaSuccess) throw std::runtime_error(std::string("dense inner solver launch: ") + cudaGetErrorString(e));
}

}  // namespace rmg
