// Hierarchy setup for dense X on the device: clustering,
// coarsening and the coarse Gram matrices without a host CSR copy of X
// (BASELINE cfg 4 is 4M x 1024; its CSR view would be 67 GB of host memory).
// Every value equals the host restatement's (host_setup.cpp) bit for bit:
// the same operations, separately rounded, in the same order.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <vector>

#include "host_setup.hpp"
#include "kernels.cuh"

namespace rmg {

// out (n x ldo fp64, row-major, ldo >= cols, even) = the columns of x widened to
// fp64 and, when normalize, scaled to unit norm as normalized_columns
// (host_setup.cpp:79-90): norm_j = sqrt(sum over rows in order of x^2), x / norm_j.
void dense_columns_f64(cudaStream_t s, const DenseDev& x, bool normalize, double* out, int64_t ldo);

// kmeans (host_setup.cpp:205-340 / clustering.cpp:189-355) over the columns of the
// fp64 row-major xc (n x f, leading dimension ld, even): k-means++ seeding with
// the column distances on the device and the draws on the host, Lloyd
// iterations on the device, empty-cluster repair and convergence on the host.
Clustering kmeans_dense_gpu(cudaStream_t s, const double* xc, int64_t n, int64_t f, int64_t ld, int64_t k,
                            uint64_t max_iters, uint64_t seed);

// X_c = X P (coarsen, host_setup.cpp:424-452) into out (n x ldc fp64 row-major,
// columns >= nc zero): out[r][c] = sum over the members j of c in increasing
// order of x[r][j] * weight[j].
void coarsen_dense_gpu(cudaStream_t s, const DenseDev& x, const Aggregation& agg, double* out, int64_t ldc);

// X^T X (coarse_gram without the beta shift, host_setup.cpp:454-465): per entry,
// the products summed over rows in increasing order.  x must be fp64.
std::vector<double> gram_dense_gpu(cudaStream_t s, const DenseDev& x);

// Sketched clustering (RMG_CLUSTER_KMEANS_SKETCH): the columns of a
// level are projected to d <= 32 dimensions, S = G^T X (d x F, row-major, leading
// dimension ldS), G[r][c] = -1 or +1 from sketch_negative(seed, r, c, d) below, the
// columns of X unit-normalised first when norm != nullptr (x / norm_j, norms as
// normalized_columns).  Each S entry sums over the column's nonzeros in increasing
// row order.  The reference's k-means (kmeans_dense_gpu) then runs on S.
void sketch_sparse_gpu(cudaStream_t s, const SparseDev& xt, const double* norm, int d, uint64_t seed, double* S,
                       int64_t ldS, int64_t row0 = 0);
void sketch_dense_gpu(cudaStream_t s, const double* xc, int64_t n, int64_t f, int64_t ld, int d, uint64_t seed,
                      double* S, int64_t ldS, int64_t row0 = 0);

}  // namespace rmg
