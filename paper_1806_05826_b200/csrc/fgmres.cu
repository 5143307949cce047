// Device parts of the flexible GMRES outer solver (krylov.cpp:229-328).
//
// The reference orthogonalizes w = A z_j against v_0..v_j with modified
// Gram-Schmidt: h_i = <w, v_i> with the current w, then w -= h_i v_i, one basis
// vector after the other.  Here one cooperative launch does the whole sweep:
// each CTA owns a contiguous block of rows of w, so the update is local and a
// sweep costs one grid barrier per basis vector (plus one for ||w||).  Dots are
// per-CTA fixed-order partials re-reduced by every CTA in CTA order
// (deterministic, no atomics).  Givens rotations, the residual estimate and the
// back substitution are the reference's own host arithmetic (runtime.cu).
#include <cooperative_groups.h>

#include <stdexcept>
#include <string>

#include "fgmres.cuh"

namespace cg = cooperative_groups;

namespace rmg {

namespace {

constexpr int kT = 256;
constexpr int kW = kT / 32;

__device__ __forceinline__ double wsum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

__device__ __forceinline__ double block_total(double v, double* sh) {
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

// sum over CTAs of partials[0 .. gridDim.x), fixed order, result in every thread
__device__ __forceinline__ double grid_total(const double* partials, double* sh) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  if (wid == 0) {
    double acc = 0.0;
    for (int b = lane; b < (int)gridDim.x; b += 32) acc += __ldcg(partials + b);
    acc = wsum(acc);
    if (lane == 0) sh[kW] = acc;
  }
  __syncthreads();
  const double r = sh[kW];
  __syncthreads();
  return r;
}

__global__ void __launch_bounds__(kT) k_mgs(double* w, const double* basis, int64_t n, int j, double* h,
                                            double* partials) {
  cg::grid_group grid = cg::this_grid();
  __shared__ double sh[kW + 1];
  const int64_t per = (n + gridDim.x - 1) / gridDim.x;
  const int64_t r0 = (int64_t)blockIdx.x * per, r1 = min(n, r0 + per);
  for (int i = 0; i <= j; ++i) {
    const double* vi = basis + (size_t)i * n;
    double d = 0.0;
    for (int64_t t = r0 + threadIdx.x; t < r1; t += kT) d += w[t] * vi[t];
    d = block_total(d, sh);
    double* slot = partials + (size_t)(i & 1) * gridDim.x;  // parity double buffer
    if (threadIdx.x == 0) slot[blockIdx.x] = d;
    grid.sync();
    const double hi = grid_total(slot, sh);
    if (blockIdx.x == 0 && threadIdx.x == 0) h[i] = hi;
    for (int64_t t = r0 + threadIdx.x; t < r1; t += kT) w[t] = w[t] - hi * vi[t];
  }
  double q = 0.0;
  for (int64_t t = r0 + threadIdx.x; t < r1; t += kT) q += w[t] * w[t];
  q = block_total(q, sh);
  double* slot = partials + (size_t)((j + 1) & 1) * gridDim.x;
  if (threadIdx.x == 0) slot[blockIdx.x] = q;
  grid.sync();
  const double nn = grid_total(slot, sh);
  if (blockIdx.x == 0 && threadIdx.x == 0) h[j + 1] = sqrt(nn);
}

__global__ void k_div(double* dst, const double* src, const double* den, int64_t n) {
  const double d = *den;
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < n; t += (int64_t)gridDim.x * blockDim.x)
    dst[t] = src[t] / d;
}

// x[t] = sum over jj in order of y[jj] * z_jj[t] (the reference's loop order,
// products and sums rounded separately: bit-equal to it for equal inputs)
__global__ void k_combine(double* x, const double* z, const double* y, int k, int64_t n) {
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < n; t += (int64_t)gridDim.x * blockDim.x) {
    double acc = 0.0;
    for (int jj = 0; jj < k; ++jj) acc = __dadd_rn(acc, __dmul_rn(y[jj], z[(size_t)jj * n + t]));
    x[t] = acc;
  }
}

int grid_sm(int64_t n) {
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  return static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(sms, (n + kT - 1) / kT)));
}

}  // namespace

int mgs_grid(int64_t n) { return grid_sm(n); }

void launch_mgs(double* w, const double* basis, int64_t n, int j, double* h, double* partials, cudaStream_t s) {
  const int grid = grid_sm(n);
  void* args[] = {&w, &basis, &n, &j, &h, &partials};
  const cudaError_t e = cudaLaunchCooperativeKernel((void*)k_mgs, dim3(grid), dim3(kT), args, 0, s);
  if (e != cudaSuccess) throw std::runtime_error(std::string("fgmres MGS launch: ") + cudaGetErrorString(e));
}

void launch_div(double* dst, const double* src, const double* den, int64_t n, cudaStream_t s) {
  k_div<<<grid_sm(n) * 4, kT, 0, s>>>(dst, src, den, n);
}

void launch_combine(double* x, const double* z, const double* y, int k, int64_t n, cudaStream_t s) {
  k_combine<<<grid_sm(n) * 4, kT, 0, s>>>(x, z, y, k, n);
}

}  // namespace rmg
