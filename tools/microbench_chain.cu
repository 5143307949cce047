// Latency of a dependent FP64 accumulation chain on one thread (the shape of the
// reference's sequential dot / per-column scatter sums, sparse.cpp:114-123,184-189):
// acc = acc + a[i] * b[i] without contraction, operands streamed from L2/L1.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/microbench_chain tools/microbench_chain.cu
#include <cstdio>
#include <cuda_runtime.h>

__global__ void chain(const double* a, const double* b, int n, double* out, long long* cyc) {
  long long t0 = clock64();
  double acc = 0.0;
  for (int i = 0; i < n; ++i) acc = __dadd_rn(acc, __dmul_rn(a[i], b[i]));
  long long t1 = clock64();
  out[0] = acc;
  cyc[0] = t1 - t0;
}

// the same with 8 operands prefetched into registers per step (loads off the chain)
__global__ void chain_pf(const double* a, const double* b, int n, double* out, long long* cyc) {
  long long t0 = clock64();
  double acc = 0.0;
  int i = 0;
  for (; i + 8 <= n; i += 8) {
    double p[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) p[j] = __dmul_rn(a[i + j], b[i + j]);
#pragma unroll
    for (int j = 0; j < 8; ++j) acc = __dadd_rn(acc, p[j]);
  }
  for (; i < n; ++i) acc = __dadd_rn(acc, __dmul_rn(a[i], b[i]));
  long long t1 = clock64();
  out[0] = acc;
  cyc[0] = t1 - t0;
}

int main() {
  const int n = 1 << 16;
  double *a, *b, *out;
  long long* cyc;
  cudaMalloc(&a, n * 8);
  cudaMalloc(&b, n * 8);
  cudaMalloc(&out, 8);
  cudaMalloc(&cyc, 8);
  cudaMemset(a, 0, n * 8);
  cudaMemset(b, 0, n * 8);
  long long h;
  for (int rep = 0; rep < 3; ++rep) {
    chain<<<1, 1>>>(a, b, n, out, cyc);
    cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
    printf("chain: %.2f cycles per term\n", double(h) / n);
    chain_pf<<<1, 1>>>(a, b, n, out, cyc);
    cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
    printf("chain_pf: %.2f cycles per term\n", double(h) / n);
  }
  return 0;
}
