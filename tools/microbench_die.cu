// Microbenchmark: latency of an L2 load of a line just written by another SM,
// per reading SM and per line (B200 has two dies, each with its own L2 half).
// For each of 16 lines: CTA w (the writer, SM of CTA 0) stores, grid.sync, then
// every CTA's thread 0 times one ld.cg of that line with clock64.  Prints, per
// line, the mean latency over SMs [0, 74) and [74, 148) by %smid.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/mbd tools/microbench_die.cu && /tmp/mbd
#include <cooperative_groups.h>
#include <cstdio>
#include <vector>
namespace cg = cooperative_groups;

__global__ void k(double* buf, long long* lat, int* smid_out, int lines, int reps) {
  cg::grid_group grid = cg::this_grid();
  unsigned smid;
  asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
  if (threadIdx.x == 0) smid_out[blockIdx.x] = (int)smid;
  for (int l = 0; l < lines; ++l) {
    long long acc = 0;
    for (int r = 0; r < reps; ++r) {
      double* p = buf + (size_t)l * 16;  // one 128 B line per l
      if (blockIdx.x == 0 && threadIdx.x == 0) {
        asm volatile("st.global.cg.f64 [%0], %1;" ::"l"(p), "d"((double)(r + l)) : "memory");
        __threadfence();
      }
      grid.sync();
      if (threadIdx.x == 0) {
        const long long t0 = clock64();
        double v;
        asm volatile("ld.global.cg.f64 %0, [%1];" : "=d"(v) : "l"(p) : "memory");
        if (v < -1.0) acc += 1;  // consume
        asm volatile("" ::"d"(v));
        const long long t1 = clock64();
        acc += t1 - t0;
      }
      grid.sync();
    }
    if (threadIdx.x == 0) lat[(size_t)l * gridDim.x + blockIdx.x] = acc / reps;
  }
}

int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int lines = 16, reps = 50;
  double* buf;
  long long* lat;
  int* smid;
  cudaMalloc(&buf, (size_t)lines * 128 * 64);
  cudaMalloc(&lat, (size_t)lines * sms * sizeof(long long));
  cudaMalloc(&smid, sms * sizeof(int));
  int l_ = lines, r_ = reps;
  void* args[] = {&buf, &lat, &smid, &l_, &r_};
  cudaLaunchCooperativeKernel((void*)k, dim3(sms), dim3(32), args, 0, 0);
  cudaDeviceSynchronize();
  printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
  std::vector<long long> h((size_t)lines * sms);
  std::vector<int> s(sms);
  cudaMemcpy(h.data(), lat, h.size() * sizeof(long long), cudaMemcpyDeviceToHost);
  cudaMemcpy(s.data(), smid, s.size() * sizeof(int), cudaMemcpyDeviceToHost);
  for (int l = 0; l < lines; ++l) {
    double a = 0, b = 0;
    int na = 0, nb = 0;
    long long mn = 1 << 30, mx = 0;
    for (int c = 0; c < sms; ++c) {
      const long long v = h[(size_t)l * sms + c];
      if (s[c] < sms / 2) {
        a += v;
        ++na;
      } else {
        b += v;
        ++nb;
      }
      mn = v < mn ? v : mn;
      mx = v > mx ? v : mx;
    }
    printf("line %2d: smid<%d mean %.0f cyc, smid>=%d mean %.0f cyc (min %lld max %lld)\n", l, sms / 2, a / na,
           sms / 2, b / nb, mn, mx);
  }
  return 0;
}
