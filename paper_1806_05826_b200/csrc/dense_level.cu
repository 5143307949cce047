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
//         z = omega r + Q (P^T r),   Q = (I - omega A_k) P A_{k+1}^{-1}
//     so it is precomputed once (n x n_c);
//   * one cooperative launch runs the whole inner solve: 148 CTAs x 1024
//     threads, each CTA owns a contiguous block of rows, keeps its rows of A_k
//     resident in shared memory when they fit (2000 x 2000 fp64 = 32 MB
//     = 148 x 216 KB), and the iteration synchronizes with 4 grid barriers.
// Reductions are deterministic: every CTA publishes a per-block partial and
// every CTA re-reduces all partials in block order.
#include <cooperative_groups.h>

#include <algorithm>
#include <stdexcept>
#include <string>

#include "dense_level.cuh"

namespace cg = cooperative_groups;

namespace rmg {

namespace {

constexpr int kT = 1024;
constexpr int kW = kT / 32;
constexpr int kPS = 40;  // partial slots per block: [0] ||b||^2, [1..31] GS, [34] pap, [35] pr, [36] rr

__device__ __forceinline__ double wsum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Block sum, result broadcast to every thread.
__device__ __forceinline__ double bsum_all(double v, double* sh) {
  v = wsum(v);
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  __syncthreads();
  if (lane == 0) sh[wid] = v;
  __syncthreads();
  if (wid == 0) {
    double r = lane < kW ? sh[lane] : 0.0;
    r = wsum(r);
    if (lane == 0) sh[kW] = r;
  }
  __syncthreads();
  return sh[kW];
}

// Sum of slot `c` over all blocks in block order (same value in every CTA).
__device__ __forceinline__ double all_blocks(const double* part, int c, double* sh) {
  double acc = 0.0;
  for (int b = threadIdx.x; b < (int)gridDim.x; b += kT) acc += __ldcg(part + (size_t)b * kPS + c);
  return bsum_all(acc, sh);
}

template <bool SMEM>
__global__ void __launch_bounds__(kT, 1) k_dense_krylov(DenseKrylovArgs a) {
  cg::grid_group grid = cg::this_grid();
  extern __shared__ double smem[];
  const int n = a.n, nc = a.nc, R = a.rows_per_cta;
  const int row0 = blockIdx.x * R;
  const int row1 = min(n, row0 + R);
  const int nr = max(0, row1 - row0);
  // shared layout: [A rows: R*n if SMEM][rc: nc][red: R*kW][zs: R][sh: kW+1]
  double* As = smem;
  double* rc = smem + (SMEM ? (size_t)R * n : 0);
  double* red = rc + nc;
  double* zs = red + (size_t)R * kW;
  double* sh = zs + R;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  double* part = a.partials + (size_t)blockIdx.x * kPS;
  KrylovScalars* sc = a.sc;

  if (SMEM) {
    for (int idx = tid; idx < nr * n; idx += kT) As[idx] = a.A[(size_t)row0 * n + idx];
  }
  // ---- begin: x = 0, r = b, ||b|| (krylov.cpp:164-176)
  double bb = 0.0, bad = 0.0;
  for (int i = row0 + tid; i < row1; i += kT) {
    const double bi = a.b[i];
    a.x[i] = 0.0;
    a.r[i] = bi;
    bb += bi * bi;
    if (!isfinite(bi)) bad += 1.0;
  }
  bb = bsum_all(bb, sh);
  bad = bsum_all(bad, sh);
  if (tid == 0) {
    part[0] = bb;
    part[1] = bad;
  }
  grid.sync();
  const double nb = sqrt(all_blocks(a.partials, 0, sh));
  const double nbad = all_blocks(a.partials, 1, sh);
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
    return;
  }
  if (!a.fcg && blockIdx.x == 0 && tid == 0) a.cg_rz_shared[0] = nb * nb;  // rz = <r, z> = ||b||^2
  const int keep = a.keep, RING = keep + 1;
  const double omega = a.omega;
  int it = 0;
  bool converged = false;
  int status = 0;
  double rel = 1.0;
  for (; it < a.max_iters; ++it) {
    const int slot = it % RING;
    double* p_now = a.p_ring + (size_t)slot * n;
    double* ap_now = a.ap_ring + (size_t)slot * n;
    // ---- z = M^{-1} r for the owned rows
    if (a.fcg) {
      for (int s = tid; s < nc; s += kT) {  // r_c = P^T r, members in increasing order
        double acc = 0.0;
        for (int q = a.mptr[s]; q < a.mptr[s + 1]; ++q) {
          const int i = a.members[q];
          const double ri = __ldcg(a.r + i);
          if (ri != 0.0) acc += a.weight[i] * ri;
        }
        rc[s] = acc;
      }
      __syncthreads();
      for (int lr = wid; lr < nr; lr += kW) {  // z_i = omega r_i + Q_i . r_c
        const double* qrow = a.Q + (size_t)(row0 + lr) * nc;
        double acc = 0.0;
        for (int s = lane; s < nc; s += 32) acc += qrow[s] * rc[s];
        acc = wsum(acc);
        if (lane == 0) zs[lr] = omega * a.r[row0 + lr] + acc;
      }
    } else {  // plain CG: z = r
      for (int lr = tid; lr < nr; lr += kT) zs[lr] = a.r[row0 + lr];
    }
    __syncthreads();
    if (a.fcg) {
      // ---- Gram-Schmidt against the newest use = min(m_i, |hist|) directions (krylov.cpp:189-197)
      const int mi = it == 0 ? 0 : max(1, it % (keep + 1));
      const int use = min(mi, min(it, keep));
      for (int q = wid; q < use; q += kW) {
        const double* aph = a.ap_ring + (size_t)((it - use + q) % RING) * n;
        double acc = 0.0;
        for (int lr = lane; lr < nr; lr += 32) acc += zs[lr] * __ldcg(aph + row0 + lr);
        acc = wsum(acc);
        if (lane == 0) part[1 + q] = acc;
      }
      grid.sync();  // B1
      for (int q = 0; q < use; ++q) {
        const double cq = all_blocks(a.partials, 1 + q, sh) / __ldcg(a.pap_ring + (it - use + q) % RING);
        if (tid < nr) zs[tid] -= cq * __ldcg(a.p_ring + (size_t)((it - use + q) % RING) * n + row0 + tid);
      }
      // zs now holds p for the owned rows
    } else if (it > 0) {
      // CG: p = z + beta p_prev  (krylov.cpp:145-153), beta from the previous iteration
      const double bcg = __ldcg(a.cg_beta_shared);
      const double* pprev = a.p_ring + (size_t)((it - 1) % RING) * n;
      if (tid < nr) zs[tid] += bcg * __ldcg(pprev + row0 + tid);
    }
    __syncthreads();
    for (int lr = tid; lr < nr; lr += kT) p_now[row0 + lr] = zs[lr];
    grid.sync();  // B2: p complete
    // ---- Ap = A p for the owned rows; pap, pr (krylov.cpp:199-208)
    {
      constexpr int MAXQ = 4;  // n <= 4096
      double pc[MAXQ];
#pragma unroll
      for (int q = 0; q < MAXQ; ++q) {
        const int c = tid + q * kT;
        pc[q] = c < n ? __ldcg(p_now + c) : 0.0;
      }
      for (int lr = 0; lr < nr; ++lr) {
        const double* arow = SMEM ? As + (size_t)lr * n : a.A + (size_t)(row0 + lr) * n;
        double acc = 0.0;
#pragma unroll
        for (int q = 0; q < MAXQ; ++q) {
          const int c = tid + q * kT;
          if (c < n) acc += arow[c] * pc[q];
        }
        acc = wsum(acc);
        if (lane == 0) red[lr * kW + wid] = acc;
      }
      __syncthreads();
      double dpap = 0.0, dpr = 0.0;
      if (tid < nr) {
        double s = 0.0;
        for (int w = 0; w < kW; ++w) s += red[tid * kW + w];
        ap_now[row0 + tid] = s;
        red[tid * kW] = s;  // keep Ap_i for the update below
        dpap = zs[tid] * s;
        dpr = zs[tid] * a.r[row0 + tid];
      }
      dpap = bsum_all(dpap, sh);
      dpr = bsum_all(dpr, sh);
      if (tid == 0) {
        part[34] = dpap;
        part[35] = dpr;
      }
    }
    grid.sync();  // B3
    const double pap = all_blocks(a.partials, 34, sh);
    const double pr = all_blocks(a.partials, 35, sh);
    if (a.fcg ? (pap == 0.0) : false) {
      status = 1;
      break;
    }
    if (a.fcg ? (pap < 0.0) : !(pap > 0.0)) {
      status = 2;
      break;
    }
    // FCG: alpha = <p,r>/pap.  CG: alpha = rz/pap with rz = <r,z> = <r,r> kept in cg_rz
    const double alpha = a.fcg ? pr / pap : __ldcg(a.cg_rz_shared + (it & 1)) / pap;
    if (blockIdx.x == 0 && tid == 0) a.pap_ring[slot] = pap;
    double rr = 0.0;
    if (tid < nr) {
      const int i = row0 + tid;
      a.x[i] += alpha * zs[tid];
      const double ri = a.r[i] - alpha * red[tid * kW];
      a.r[i] = ri;
      rr = ri * ri;
    }
    rr = bsum_all(rr, sh);
    if (tid == 0) part[36] = rr;
    grid.sync();  // B4
    const double rrs = all_blocks(a.partials, 36, sh);
    rel = sqrt(rrs) / nb;
    if (blockIdx.x == 0 && tid == 0) {
      a.hist[it] = rel;
      if (!a.fcg) {  // CG: rz' = <r,r>, beta = rz'/rz
        a.cg_beta_shared[0] = rrs / __ldcg(a.cg_rz_shared + (it & 1));
        a.cg_rz_shared[(it + 1) & 1] = rrs;
      }
    }
    if (rel <= a.tol) {
      converged = true;
      ++it;
      break;
    }
    if (!a.fcg) grid.sync();  // CG: beta visible to every CTA
  }
  if (blockIdx.x == 0 && tid == 0) {
    sc->it = it;
    sc->status = status;
    sc->converged = converged ? 1 : 0;
    sc->done = 1;
    sc->rel = rel;
    sc->nb = nb;
  }
}

}  // namespace

DenseKrylovPlan plan_dense_krylov(int n, int nc, int device) {
  DenseKrylovPlan p;
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
  int max_smem = 0;
  cudaDeviceGetAttribute(&max_smem, cudaDevAttrMaxSharedMemoryPerBlockOptin, device);
  p.rows_per_cta = std::max(1, (n + sms - 1) / sms);
  p.grid = (n + p.rows_per_cta - 1) / p.rows_per_cta;
  const size_t extra = ((size_t)nc + (size_t)p.rows_per_cta * kW + p.rows_per_cta + kW + 1) * sizeof(double);
  const size_t with_a = extra + (size_t)p.rows_per_cta * n * sizeof(double);
  p.smem_a = with_a <= (size_t)max_smem;
  p.smem_bytes = p.smem_a ? with_a : extra;
  p.partial_stride = kPS;
  return p;
}

void launch_dense_krylov(const DenseKrylovPlan& plan, const DenseKrylovArgs& args, cudaStream_t s) {
  if (args.n > 4096) throw std::runtime_error("dense inner solver: level above 4096 unknowns");
  void* fn = plan.smem_a ? (void*)k_dense_krylov<true> : (void*)k_dense_krylov<false>;
  cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)plan.smem_bytes);
  if (e != cudaSuccess) throw std::runtime_error(std::string("dense inner solver attribute: ") + cudaGetErrorString(e));
  DenseKrylovArgs a = args;
  a.rows_per_cta = plan.rows_per_cta;
  void* kargs[] = {&a};
  e = cudaLaunchCooperativeKernel(fn, dim3(plan.grid), dim3(kT), kargs, plan.smem_bytes, s);
  if (e != cudaSuccess) throw std::runtime_error(std::string("dense inner solver launch: ") + cudaGetErrorString(e));
}

}  // namespace rmg
