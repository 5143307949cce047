// k-means on the GPU with labels bit-identical to the reference (kmeans_gpu.cu).
#pragma once
#include <cuda_runtime.h>

#include <cstdint>

#include "host_setup.hpp"

namespace rmg {

// Whether kmeans_gpu can run this size (k <= 8192, int32 indices, N x k
// prototypes within device memory).
bool kmeans_gpu_supported(int64_t n, int64_t f, int64_t k, int64_t nnz);
// cols: the matrix as features x samples (the reference's columns), rows: the
// same matrix as samples x features.  Same result as kmeans(cols, ...).
Clustering kmeans_gpu(cudaStream_t s, const HostCsr& cols, const HostCsr& rows, int64_t k, uint64_t max_iters,
                      uint64_t seed);

}  // namespace rmg
