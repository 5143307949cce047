// Microbenchmark: grid-wide "exchange" (barrier + every CTA reading what every
// other CTA published) on B200, 143 CTAs x 256 threads (the cfg 2 inner
// solver's grid), cooperative launch.  Compares:
//   mode 0: grid.sync, then one warp sums the 143 per-CTA partials
//   mode 1: sentinel slots: no barrier; a CTA first re-arms its slot of the
//           buffer used two exchanges later (3 rotating buffers), then stores
//           its partial; readers poll the slots until none holds the sentinel
//   mode 2: grid.sync, then every thread loads its 8 elements of a 2000-vector
//           (14 rows published per CTA) -- the solver's B1 exchange of z
//   mode 3: the same vector exchange through sentinel slots
// Build + run:
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/mb2 tools/microbench_sync2.cu && /tmp/mb2
#include <cooperative_groups.h>
#include <cstdint>
#include <cstdio>
namespace cg = cooperative_groups;

constexpr unsigned long long kSentinel = 0x7ff4dead5e5e5e5eull;  // a NaN payload no computation produces

__device__ __forceinline__ double wsum(double v) {
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ void st_relaxed(double* p, double v) {
  asm volatile("st.relaxed.gpu.global.f64 [%0], %1;" ::"l"(p), "d"(v) : "memory");
}
__device__ __forceinline__ unsigned long long ld_relaxed(const double* p) {
  unsigned long long v;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ void st_release(double* p, double v) {
  asm volatile("st.release.gpu.global.f64 [%0], %1;" ::"l"(p), "d"(v) : "memory");
}
__device__ __forceinline__ unsigned long long ld_acquire64(const double* p) {
  unsigned long long v;
  asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_u32(unsigned* p, unsigned v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ unsigned ld_acquire_u32(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

template <int NT>
__global__ void __launch_bounds__(NT, 1) k(int iters, int mode, double* part, double* vec, double* out, int n, unsigned* flags) {
  cg::grid_group grid = cg::this_grid();
  __shared__ double sh[33];
  const int tid = threadIdx.x, lane = tid & 31, nb = gridDim.x;
  const int R = (n + nb - 1) / nb, row0 = blockIdx.x * R, row1 = min(n, row0 + R);
  double acc = 0.0;
  for (int it = 0; it < iters; ++it) {
    const int cur = it % 3, nxt = (it + 1) % 3;
    if (mode >= 4) {
      // 4: sentinel, st.release publish (re-arm issued one exchange earlier), ld.acquire polls
      // 5: sentinel, relaxed everything, no fences (ordering lower bound, not a valid protocol)
      // 6: per-CTA flags: data, st.release flag; one warp polls 143 flags (ld.acquire), then loads
      if (mode == 6) {
        if (tid == 0) {
          part[blockIdx.x] = it + blockIdx.x;
          st_release_u32(flags + blockIdx.x, it + 1);
        }
        if (tid < 32) {
          for (int b = lane; b < nb; b += 32)
            while (ld_acquire_u32(flags + b) < (unsigned)(it + 1)) {
            }
        }
        __syncthreads();
        if (tid < 32) {
          double v = 0.0;
          for (int b = lane; b < nb; b += 32) v += __ldcg(part + b);
          v = wsum(v);
          if (tid == 0) sh[0] = v;
        }
      } else {
        double* P = part;
        const int m = nb;
        if (tid == 0) {
          // re-arm own slot of the next buffer (read last two exchanges ago), ordered
          // before this publish by its release
          st_relaxed(P + (size_t)nxt * m + blockIdx.x, __longlong_as_double(kSentinel));
          if (mode == 4) st_release(P + (size_t)cur * m + blockIdx.x, it + blockIdx.x);
          else st_relaxed(P + (size_t)cur * m + blockIdx.x, it + blockIdx.x);
        }
        const double* src = P + (size_t)cur * m;
        if (tid < 32) {
          double x[5];
          unsigned pending = 0;
#pragma unroll
          for (int u = 0; u < 5; ++u) {
            x[u] = 0.0;
            if (lane + 32 * u < nb) pending |= 1u << u;
          }
          while (pending) {
#pragma unroll
            for (int u = 0; u < 5; ++u)
              if (pending & (1u << u)) {
                const unsigned long long bits =
                    mode == 4 ? ld_acquire64(src + lane + 32 * u) : ld_relaxed(src + lane + 32 * u);
                if (bits != kSentinel) {
                  x[u] = __longlong_as_double(bits);
                  pending &= ~(1u << u);
                }
              }
          }
          double v = 0.0;
#pragma unroll
          for (int u = 0; u < 5; ++u) v += x[u];
          v = wsum(v);
          if (tid == 0) sh[0] = v;
        }
      }
      __syncthreads();
      acc += sh[0];
      __syncthreads();
    } else if (mode == 0 || mode == 2) {
      if (mode == 0) {
        if (tid == 0) part[blockIdx.x] = it + blockIdx.x;
      } else {
        for (int i = row0 + tid; i < row1; i += NT) vec[i] = it + i;
      }
      grid.sync();
      if (mode == 0) {
        if (tid < 32) {
          double v = 0.0;
          for (int b = lane; b < nb; b += 32) v += __ldcg(part + b);
          v = wsum(v);
          if (tid == 0) sh[0] = v;
        }
      } else {
        double v = 0.0;
        for (int i = tid; i < n; i += NT) v += __ldcg(vec + i);
        v = wsum(v);
        if (lane == 0) sh[tid >> 5] = v;
      }
      __syncthreads();
      acc += sh[0];
      __syncthreads();
    } else {
      double* P = mode == 1 ? part : vec;
      const int m = mode == 1 ? nb : n;
      // re-arm own slots of the buffer used at it + 1 (read last at it - 2, done by
      // every CTA before it published at it - 1), then publish at it
      if (mode == 1) {
        if (tid == 0) {
          st_relaxed(P + (size_t)nxt * m + blockIdx.x, __longlong_as_double(kSentinel));
          __threadfence();
          st_relaxed(P + (size_t)cur * m + blockIdx.x, it + blockIdx.x);
        }
      } else {
        for (int i = row0 + tid; i < row1; i += NT) st_relaxed(P + (size_t)nxt * m + i, __longlong_as_double(kSentinel));
        __syncthreads();
        if (tid == 0) __threadfence();
        __syncthreads();
        for (int i = row0 + tid; i < row1; i += NT) st_relaxed(P + (size_t)cur * m + i, it + i);
      }
      const double* src = P + (size_t)cur * m;
      if (mode == 1) {
        if (tid < 32) {
          double x[5];
          unsigned pending = 0;
#pragma unroll
          for (int u = 0; u < 5; ++u) {
            const int b = lane + 32 * u;
            x[u] = 0.0;
            if (b < nb) pending |= 1u << u;
          }
          while (pending) {
#pragma unroll
            for (int u = 0; u < 5; ++u)
              if (pending & (1u << u)) {
                const unsigned long long bits = ld_relaxed(src + lane + 32 * u);
                if (bits != kSentinel) {
                  x[u] = __longlong_as_double(bits);
                  pending &= ~(1u << u);
                }
              }
          }
          asm volatile("fence.acq_rel.gpu;" ::: "memory");  // pairs with the writers' fence
          double v = 0.0;
#pragma unroll
          for (int u = 0; u < 5; ++u) v += x[u];
          v = wsum(v);
          if (tid == 0) sh[0] = v;
        }
      } else {
        double x[8];
        unsigned pending = 0;
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          x[u] = 0.0;
          if (tid + u * NT < n) pending |= 1u << u;
        }
        while (pending) {
#pragma unroll
          for (int u = 0; u < 8; ++u)
            if (pending & (1u << u)) {
              const unsigned long long bits = ld_relaxed(src + tid + u * NT);
              if (bits != kSentinel) {
                x[u] = __longlong_as_double(bits);
                pending &= ~(1u << u);
              }
            }
        }
        asm volatile("fence.acq_rel.gpu;" ::: "memory");
        double v = 0.0;
#pragma unroll
        for (int u = 0; u < 8; ++u) v += x[u];
        v = wsum(v);
        if (lane == 0) sh[tid >> 5] = v;
      }
      __syncthreads();
      acc += sh[0];
      __syncthreads();
    }
  }
  if (tid == 0 && blockIdx.x == 0) out[0] = acc;
}

int main() {
  const int n = 2000;
  double *part, *vec, *out;
  cudaMalloc(&part, 3 * 4096 * 8);
  cudaMalloc(&vec, 3 * 4096 * 8);
  cudaMalloc(&out, 8);
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  const char* names[] = {"grid.sync + 143 partials", "sentinel slots, 143 partials", "grid.sync + 2000-vector",
                         "sentinel slots, 2000-vector", "sentinel, st.release/ld.acquire", "sentinel, no ordering",
                         "per-CTA release flags"};
  unsigned* flags;
  cudaMalloc(&flags, 4096 * 4);
  for (int mode = 0; mode < 7; ++mode) {
    for (int grid : {143, sms}) {
      int iters = 4000;
      int nn = n;
      void* args[] = {&iters, &mode, &part, &vec, &out, &nn, &flags};
      for (int rep = 0; rep < 2; ++rep) {
        // all slots start armed (sentinel) for the sentinel modes
        unsigned long long s = kSentinel;
        static unsigned long long h[3 * 4096];
        for (auto& x : h) x = s;
        cudaMemcpy(part, h, sizeof(h), cudaMemcpyHostToDevice);
        cudaMemcpy(vec, h, sizeof(h), cudaMemcpyHostToDevice);
        cudaMemset(flags, 0, 4096 * 4);
        cudaEventRecord(a);
        cudaLaunchCooperativeKernel((void*)k<256>, dim3(grid), dim3(256), args, 0, 0);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        double o;
        cudaMemcpy(&o, out, 8, cudaMemcpyDeviceToHost);
        if (rep == 1)
          printf("mode %d (%-28s) grid %3d: %.3f us per exchange (%s) out %.6g\n", mode, names[mode], grid,
                 ms * 1000.0 / iters, cudaGetErrorString(cudaGetLastError()), o);
      }
    }
  }
  return 0;
}
