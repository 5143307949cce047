// Microbenchmark: the Ap = A p step of the persistent inner solver on B200,
// in isolation (cooperative launch over 143 CTAs, n = 2000, 14 rows per CTA,
// A rows resident in shared memory).  Each variant is its own template
// instantiation.  Times are per iteration, averaged over 1000.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/microbench_gemv tools/microbench_gemv.cu
#include <cooperative_groups.h>
#include <cstdio>
namespace cg = cooperative_groups;

constexpr int N = 2000, R = 14;

__device__ __forceinline__ double wsum(double v) {
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// SYNC: grid.sync + p store/load each iteration; LOADP: p loaded from global
// (else kept in registers); RED: 0 = warp shuffles per row + smem combine,
// 1 = per-thread partials to smem, then one warp per row sums them.
template <int T, bool SYNC, bool LOADP, int RED>
__global__ void __launch_bounds__(T, 1) k(int iters, const double* A, double* p, double* out) {
  cg::grid_group grid = cg::this_grid();
  constexpr int W = T / 32, Q = (N + T - 1) / T;
  extern __shared__ double sm[];
  double* As = sm;            // R*N
  double* red = sm + R * N;   // R*W (RED 0) or reused
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int row0 = blockIdx.x * R;
  const int nr = min(R, max(0, N - row0));
  for (int i = tid; i < nr * N; i += T) As[i] = A[(size_t)row0 * N + i];
  __syncthreads();
  double vc[Q];
#pragma unroll
  for (int q = 0; q < Q; ++q) vc[q] = 1.0 + tid;
  double tot = 0;
  for (int it = 0; it < iters; ++it) {
    if (SYNC) {
      if (tid < nr) p[row0 + tid] = it + tid;
      grid.sync();
    }
    if (LOADP) {
#pragma unroll
      for (int q = 0; q < Q; ++q) vc[q] = tid + q * T < N ? __ldcg(p + tid + q * T) : 0.0;
    }
    if (RED == 0) {
      for (int lr0 = 0; lr0 < nr; lr0 += 4) {
        double acc[4] = {0, 0, 0, 0};
#pragma unroll
        for (int u = 0; u < 4; ++u)
          if (lr0 + u < nr) {
#pragma unroll
            for (int q = 0; q < Q; ++q)
              if (tid + q * T < N) acc[u] += As[(lr0 + u) * N + tid + q * T] * vc[q];
          }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const double s = wsum(acc[u]);
          if (lane == 0 && lr0 + u < nr) red[(lr0 + u) * W + wid] = s;
        }
      }
      __syncthreads();
      if (tid < nr) {
        double s = 0;
        for (int w = 0; w < W; ++w) s += red[tid * W + w];
        tot += s;
      }
      __syncthreads();
    } else {
      // each warp owns whole rows: lanes stride the columns, p from registers is
      // not usable (different columns) -> p read from global/L1 per lane
      for (int lr = wid; lr < nr; lr += W) {
        double s = 0;
        for (int c = lane; c < N; c += 32) s += As[lr * N + c] * __ldcg(p + c);
        s = wsum(s);
        if (lane == 0) tot += s;
      }
      __syncthreads();
    }
  }
  if (tid == 0) out[blockIdx.x] = tot + vc[0];
}

template <int T, bool SYNC, bool LOADP, int RED>
void run(const char* name, const double* A, double* p, double* out) {
  const int grid = (N + R - 1) / R;
  const size_t smem = sizeof(double) * (R * N + R * (T / 32));
  auto fn = k<T, SYNC, LOADP, RED>;
  cudaFuncSetAttribute((void*)fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  int iters = 1000;
  void* args[] = {&iters, (void*)&A, (void*)&p, (void*)&out};
  cudaLaunchCooperativeKernel((void*)fn, dim3(grid), dim3(T), args, smem, 0);
  cudaEventRecord(a);
  cudaLaunchCooperativeKernel((void*)fn, dim3(grid), dim3(T), args, smem, 0);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  printf("%-44s %8.3f us/iter (%s)\n", name, ms * 1000.0 / iters, cudaGetErrorString(cudaGetLastError()));
}

// Closer to the solver: p written into a 21-slot ring (new address every
// iteration) and/or a second GEMV streaming a 32 MB matrix M from L2/HBM.
// RING: bit 0 = p ring, bit 1 = M stream.
template <int RING>
__global__ void __launch_bounds__(1024, 1) kr(int iters, const double* A, double* ring, const double* M, double* out) {
  cg::grid_group grid = cg::this_grid();
  constexpr int T = 1024, W = 32;
  extern __shared__ double sm[];
  double* As = sm;
  double* red = sm + R * N;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int row0 = blockIdx.x * R;
  const int nr = min(R, max(0, N - row0));
  for (int i = tid; i < nr * N; i += T) As[i] = A[(size_t)row0 * N + i];
  __syncthreads();
  double tot = 0;
  auto gemv = [&](const double* rows, bool global, double v0, double v1) {
    for (int lr0 = 0; lr0 < nr; lr0 += 4) {
      double acc[4] = {0, 0, 0, 0};
#pragma unroll
      for (int u = 0; u < 4; ++u)
        if (lr0 + u < nr) {
          const double* row = rows + (size_t)(lr0 + u) * N;
          acc[u] += (global ? __ldg(row + tid) : row[tid]) * v0;
          if (tid + T < N) acc[u] += (global ? __ldg(row + tid + T) : row[tid + T]) * v1;
        }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const double s = wsum(acc[u]);
        if (lane == 0 && lr0 + u < nr) red[(lr0 + u) * W + wid] = s;
      }
    }
    __syncthreads();
    if (tid < nr) {
      double s = 0;
      for (int w = 0; w < W; ++w) s += red[tid * W + w];
      tot += s;
    }
    __syncthreads();
  };
  for (int it = 0; it < iters; ++it) {
    double* p = ring + (RING & 1 ? (size_t)(it % 21) * N : 0);
    if (tid < nr) p[row0 + tid] = it + tid;
    grid.sync();
    const double v0 = __ldcg(p + tid), v1 = tid + T < N ? __ldcg(p + tid + T) : 0.0;
    if (RING & 2) gemv(M + (size_t)row0 * N, true, v0, v1);
    gemv(As, false, v0, v1);
  }
  if (tid == 0) out[blockIdx.x] = tot;
}

void run_ring(int v, const double* A, double* ring, const double* M, double* out) {
  const int grid = (N + R - 1) / R;
  const size_t smem = sizeof(double) * (R * N + R * 32);
  void* fns[] = {(void*)kr<0>, (void*)kr<1>, (void*)kr<2>, (void*)kr<3>};
  const char* names[] = {"ring-test: fixed p, no M", "ring-test: p ring, no M", "ring-test: fixed p, + M stream",
                         "ring-test: p ring + M stream"};
  cudaFuncSetAttribute(fns[v], cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  int iters = 1000;
  void* args[] = {&iters, (void*)&A, (void*)&ring, (void*)&M, (void*)&out};
  cudaLaunchCooperativeKernel(fns[v], dim3(grid), dim3(1024), args, smem, 0);
  cudaEventRecord(a);
  cudaLaunchCooperativeKernel(fns[v], dim3(grid), dim3(1024), args, smem, 0);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  printf("%-44s %8.3f us/iter (%s)\n", names[v], ms * 1000.0 / iters, cudaGetErrorString(cudaGetLastError()));
}

int main() {
  double *A, *p, *out;
  cudaMalloc(&A, sizeof(double) * N * N);
  cudaMalloc(&p, sizeof(double) * N);
  cudaMalloc(&out, sizeof(double) * 4096);
  cudaMemset(A, 0, sizeof(double) * N * N);
  cudaMemset(p, 0, sizeof(double) * N);
  run<1024, false, false, 0>("T1024 gemv only (p in regs)", A, p, out);
  run<1024, false, true, 0>("T1024 gemv + p load (no sync)", A, p, out);
  run<1024, true, false, 0>("T1024 gemv + sync (no p load)", A, p, out);
  run<1024, true, true, 0>("T1024 gemv + sync + p load", A, p, out);
  run<512, false, false, 0>("T512 gemv only", A, p, out);
  run<512, true, true, 0>("T512 gemv + sync + p load", A, p, out);
  run<256, false, false, 0>("T256 gemv only", A, p, out);
  run<256, true, true, 0>("T256 gemv + sync + p load", A, p, out);
  run<1024, true, true, 1>("T1024 warp-per-row + sync + p(global)", A, p, out);
  run<512, true, true, 1>("T512 warp-per-row + sync + p(global)", A, p, out);
  double *ring, *M;
  cudaMalloc(&ring, sizeof(double) * N * 21);
  cudaMalloc(&M, sizeof(double) * N * N);
  cudaMemset(ring, 0, sizeof(double) * N * 21);
  cudaMemset(M, 0, sizeof(double) * N * N);
  for (int v = 0; v < 4; ++v) run_ring(v, A, ring, M, out);
  return 0;
}
