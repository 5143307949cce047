// Microbenchmark: random 128-byte row gathers (the block operator's access:
// one row of a row-major n x 16 fp64 block per nonzero).  A half-warp reads one
// row (lane q: double q), every lane keeps U independent gathers in flight.
// Rows are drawn uniformly from a table of `rows` rows (L2-resident or not) or
// Zipf-like (rank^-1.1, label order: the popular rows share L1 lines).
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/microbench_gather tools/microbench_gather.cu
//   tools/microbench_gather
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <random>
#include <vector>

#define CK(x)                                                                  \
  do {                                                                         \
    cudaError_t e = (x);                                                       \
    if (e != cudaSuccess) {                                                    \
      std::printf("%s: %s\n", #x, cudaGetErrorString(e));                      \
      std::exit(1);                                                            \
    }                                                                          \
  } while (0)

template <int U, bool NC>
__global__ void __launch_bounds__(256) gather(const double* __restrict__ m, const int* __restrict__ idx, int64_t n_idx,
                                              double* __restrict__ out) {
  const int lane = threadIdx.x & 31, q = lane & 15, h = lane >> 4;
  const int64_t hw = ((int64_t)blockIdx.x * 256 + threadIdx.x) >> 4;  // half-warp id
  const int64_t nhw = ((int64_t)gridDim.x * 256) >> 4;
  double acc = 0.0;
  for (int64_t base = (hw >> 1) * 2 * U; base < n_idx; base += nhw * U) {
    int r[U];
#pragma unroll
    for (int u = 0; u < U; ++u) r[u] = idx[(base + 2 * u + h) % n_idx];
    double v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) v[u] = NC ? __ldg(m + (int64_t)r[u] * 16 + q) : m[(int64_t)r[u] * 16 + q];
#pragma unroll
    for (int u = 0; u < U; ++u) acc += v[u];
  }
  if (acc == 12345.678) out[0] = acc;
}

int main() {
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int64_t n_idx = 64 << 20;  // 64 M gathers = 8 GB of rows
  std::vector<int64_t> table_rows = {100000, 500000, 1000000, 8000000};
  int* d_idx;
  double* d_m;
  double* d_out;
  CK(cudaMalloc(&d_idx, n_idx * sizeof(int)));
  CK(cudaMalloc(&d_m, (int64_t)8000000 * 16 * 8));
  CK(cudaMalloc(&d_out, 8));
  CK(cudaMemset(d_m, 0, (int64_t)8000000 * 16 * 8));
  std::mt19937_64 rng(1);
  std::vector<int> h(n_idx);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int zipf = 0; zipf < 2; ++zipf) {
    for (int64_t rows : table_rows) {
      if (zipf) {  // inverse CDF of rank^-1.1 over `rows` ranks
        std::vector<double> cdf(rows);
        double s = 0;
        for (int64_t k = 0; k < rows; ++k) cdf[k] = (s += std::pow(double(k + 1), -1.1));
        std::uniform_real_distribution<double> U(0, s);
        for (auto& x : h) x = int(std::upper_bound(cdf.begin(), cdf.end(), U(rng)) - cdf.begin());
      } else {
        std::uniform_int_distribution<int64_t> U(0, rows - 1);
        for (auto& x : h) x = int(U(rng));
      }
      CK(cudaMemcpy(d_idx, h.data(), n_idx * sizeof(int), cudaMemcpyHostToDevice));
      for (int variant = 0; variant < 3; ++variant) {
        auto run = [&](int blocks_per_sm) {
          const int grid = sms * blocks_per_sm;
          if (variant == 0) gather<16, true><<<grid, 256>>>(d_m, d_idx, n_idx, d_out);
          if (variant == 1) gather<8, true><<<grid, 256>>>(d_m, d_idx, n_idx, d_out);
          if (variant == 2) gather<16, false><<<grid, 256>>>(d_m, d_idx, n_idx, d_out);
        };
        for (int bps : {4, 8}) {
          run(bps);
          CK(cudaDeviceSynchronize());
          cudaEventRecord(e0);
          run(bps);
          cudaEventRecord(e1);
          CK(cudaEventSynchronize(e1));
          float ms = 0;
          cudaEventElapsedTime(&ms, e0, e1);
          const double gb = double(n_idx) * 128 / 1e9;
          std::printf("%s rows=%8lld (%6.1f MB) U=%2d %s ctas/SM=%d: %7.3f ms  %6.2f TB/s of 128-B rows\n",
                      zipf ? "zipf   " : "uniform", (long long)rows, rows * 128 / 1e6, variant == 1 ? 8 : 16,
                      variant == 2 ? "ld  " : "ldg ", bps, ms, gb / ms / 1e3);
        }
      }
    }
  }
  return 0;
}
