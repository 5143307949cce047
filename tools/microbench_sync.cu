// Microbenchmark: cost of grid-wide synchronization primitives on B200
// (148 / 143 CTAs x 256 threads, cooperative launch), to size the persistent
// inner solver (dense_level.cu).  Build + run:
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/mb tools/microbench_sync.cu && /tmp/mb
#include <cooperative_groups.h>
#include <cstdio>
namespace cg = cooperative_groups;

__device__ __forceinline__ double wsum(double v) {
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// mode 0: grid.sync only; 1: grid.sync + one all-block reduction (like all_blocks)
// mode 2: custom flag barrier (atomic arrive + spin on generation)
// mode 3: monotonic counter: red.release.gpu arrive, ld.acquire.gpu poll until
//         (it + 1) * gridDim.x (no reset, no generation word)
__device__ __forceinline__ void red_release_add(unsigned* p, unsigned v) {
  asm volatile("red.release.gpu.global.add.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ unsigned ld_acquire(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

template <int NT>
__global__ void __launch_bounds__(NT, 1) k(int iters, int mode, double* part, unsigned* bar, double* out) {
  cg::grid_group grid = cg::this_grid();
  __shared__ double sh[33];
  double acc = 0.0;
  for (int it = 0; it < iters; ++it) {
    if (mode == 3) {
      __syncthreads();
      if (threadIdx.x == 0) {
        const unsigned target = (unsigned)(it + 1) * gridDim.x;
        red_release_add(bar + 2, 1u);
        while (ld_acquire(bar + 2) < target) {
        }
      }
      __syncthreads();
    } else if (mode == 2) {
      __syncthreads();
      if (threadIdx.x == 0) {
        volatile unsigned* gen = bar + 1;
        const unsigned g = *gen;
        __threadfence();
        const unsigned a = atomicAdd(bar, 1u);
        if (a == gridDim.x - 1) {
          bar[0] = 0;
          __threadfence();
          atomicAdd((unsigned*)gen, 1u);
        } else {
          while (*gen == g) {
          }
        }
        __threadfence();
      }
      __syncthreads();
    } else if (mode == 9 || mode == 10) {
      // 9: one 128 B line per CTA's partial; 10: partials written with st.global (L1
      // write-through) but read after the barrier with ld.acquire.gpu
      const int stride = mode == 9 ? 16 : 1;
      if (threadIdx.x == 0) part[(size_t)blockIdx.x * stride] = it + blockIdx.x;
      grid.sync();
      double v = 0.0;
      if (threadIdx.x < gridDim.x) {
        if (mode == 9) {
          v = __ldcg(part + (size_t)threadIdx.x * stride);
        } else {
          asm volatile("ld.relaxed.gpu.global.f64 %0, [%1];" : "=d"(v) : "l"(part + threadIdx.x) : "memory");
        }
      }
      v = wsum(v);
      if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = v;
      __syncthreads();
      if (threadIdx.x < 32) {
        double r = threadIdx.x < (NT / 32) ? sh[threadIdx.x] : 0.0;
        r = wsum(r);
        if (threadIdx.x == 0) sh[32] = r;
      }
      __syncthreads();
      acc += sh[32];
    } else if (mode == 12 || mode == 13) {
      // 12: the monotonic-counter barrier (tight spin, no backoff) + the constant block
      // reduction of mode 11; 13: the same with every warp's lane 0 polling (no
      // __syncthreads release inside the CTA)
      __syncthreads();
      const unsigned target = (unsigned)(it + 1) * gridDim.x;
      if (threadIdx.x == 0) red_release_add(bar + 2, 1u);
      if (mode == 12) {
        if (threadIdx.x == 0)
          while (ld_acquire(bar + 2) < target) {
          }
        __syncthreads();
      } else {
        if ((threadIdx.x & 31) == 0)
          while (ld_acquire(bar + 2) < target) {
          }
        __syncwarp();
      }
      double v = threadIdx.x < gridDim.x ? (double)threadIdx.x : 0.0;
      v = wsum(v);
      if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = v;
      __syncthreads();
      if (threadIdx.x < 32) {
        double r = threadIdx.x < (NT / 32) ? sh[threadIdx.x] : 0.0;
        r = wsum(r);
        if (threadIdx.x == 0) sh[32] = r;
      }
      __syncthreads();
      acc += sh[32];
    } else if (mode == 11) {
      // grid.sync + block reduction of a constant (no global load): the reduction's own cost
      grid.sync();
      double v = threadIdx.x < gridDim.x ? (double)threadIdx.x : 0.0;
      v = wsum(v);
      if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = v;
      __syncthreads();
      if (threadIdx.x < 32) {
        double r = threadIdx.x < (NT / 32) ? sh[threadIdx.x] : 0.0;
        r = wsum(r);
        if (threadIdx.x == 0) sh[32] = r;
      }
      __syncthreads();
      acc += sh[32];
    } else if (mode >= 4) {
      // mode 4 + log2(R): grid.sync + one all-block reduction read from R replicas of
      // the partials (CTA b reads replica b % R): fewer readers per L2 line
      const int R = 1 << (mode - 4);
      if (threadIdx.x < R) part[(size_t)threadIdx.x * 512 + blockIdx.x] = it + blockIdx.x;
      grid.sync();
      const double* src = part + (size_t)(blockIdx.x % R) * 512;
      double v = threadIdx.x < gridDim.x ? __ldcg(src + threadIdx.x) : 0.0;
      v = wsum(v);
      if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = v;
      __syncthreads();
      if (threadIdx.x < 32) {
        double r = threadIdx.x < (NT / 32) ? sh[threadIdx.x] : 0.0;
        r = wsum(r);
        if (threadIdx.x == 0) sh[32] = r;
      }
      __syncthreads();
      acc += sh[32];
    } else {
      if (threadIdx.x == 0) part[blockIdx.x] = it + blockIdx.x;
      grid.sync();
      if (mode == 1) {
        double v = threadIdx.x < gridDim.x ? __ldcg(part + threadIdx.x) : 0.0;
        v = wsum(v);
        if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = v;
        __syncthreads();
        if (threadIdx.x < 32) {
          double r = sh[threadIdx.x];
          r = wsum(r);
          if (threadIdx.x == 0) sh[32] = r;
        }
        __syncthreads();
        acc += sh[32];
      }
    }
  }
  if (threadIdx.x == 0 && blockIdx.x == 0) out[0] = acc;
}

int main() {
  double *part, *out;
  unsigned* bar;
  cudaMalloc(&part, 16 * 512 * 8);
  cudaMalloc(&out, 8);
  cudaMalloc(&bar, 16);
  cudaMemset(bar, 0, 16);
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (int mode = 0; mode < 14; ++mode) {
    for (int grid : {sms, 143, 74}) {
      int iters = 2000;
      void* args[] = {&iters, &mode, &part, &bar, &out};
      cudaMemset(bar, 0, 16);
      cudaLaunchCooperativeKernel((void*)k<256>, dim3(grid), dim3(256), args, 0, 0);
      cudaMemset(bar, 0, 16);
      cudaEventRecord(a);
      cudaLaunchCooperativeKernel((void*)k<256>, dim3(grid), dim3(256), args, 0, 0);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      printf("mode %d grid %3d: %.3f us per iteration (%s)\n", mode, grid, ms * 1000.0 / iters,
             cudaGetErrorString(cudaGetLastError()));
    }
  }
  return 0;
}
