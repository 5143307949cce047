// Device parts of the FGMRES outer solver (fgmres.cu; krylov.cpp:229-328).
#pragma once
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>

namespace rmg {

// CTAs of the cooperative MGS sweep (partials needs 2 x this many doubles)
int mgs_grid(int64_t n);
// Modified Gram-Schmidt of w against basis[0..j] (each n long, contiguous):
// h[i] = <w, v_i> (current w), w -= h[i] v_i; then h[j+1] = ||w||.
void launch_mgs(double* w, const double* basis, int64_t n, int j, double* h, double* partials, cudaStream_t s);
// dst = src / *den (device scalar), element-wise division as the reference
void launch_div(double* dst, const double* src, const double* den, int64_t n, cudaStream_t s);
// x = sum_{jj < k} y[jj] z_jj, per element in jj order (z: k x n, contiguous)
void launch_combine(double* x, const double* z, const double* y, int k, int64_t n, cudaStream_t s);

}  // namespace rmg
