// Dense Gram matrices of coarse levels.
//
// A coarse level X_k (N rows, n_k features) enters the solve only through
// A_k = X_k^T X_k + beta_k I.  When n_k^2 doubles are fewer bytes than one
// sweep pair over X_k (cfg 3: n_1 = 10 000 -> 800 MB against 1.15 GB of
// X_c1 per application), the V-cycle applies the dense G_k = X_k^T X_k
// instead: a GEMV (one RHS) or a skinny GEMM (k RHS) streaming G_k once.
//
// G_k is assembled on the device from the CSR of X_k and of X_k^T with the
// reference coarse Gram's arithmetic (krylov.cpp:350-365): entry (i, j) is
// the sum over the rows r holding both features, in increasing r, of the
// separately rounded products x_ri * x_rj -- bit-identical to the host
// restatement coarse_gram (host_setup.cpp), which also uses it for the
// coarsest Cholesky and the dense inner levels.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace rmg {

// G (n x n, row-major, leading dimension ldg) = X^T X, no beta.
//   X   : row CSR (xptr[N+1], xidx, xval or nullptr for a binary pattern)
//   X^T : feature CSR (tptr[n+1], tidx = rows ascending, tval or nullptr)
void sparse_gram_gpu(cudaStream_t s, const int32_t* xptr, const int32_t* xidx, const double* xval,
                     const int32_t* tptr, const int32_t* tidx, const double* tval, int64_t n, double* G,
                     int64_t ldg);

// y = G x + beta x (one right-hand side); no-op when *done != 0.
void launch_gram_gemv(const double* G, int64_t ldg, const double* x, double beta, double* y, int64_t n,
                      const int32_t* done, cudaStream_t s);

// Y = G V + beta V for row-major n x k blocks V, Y (leading dimension k), k <= 64,
// on the FP64 tensor cores (DMMA, split K; RMG_GRAM_GEMM=cuda: CUDA cores).
// scratch: gram_gemm_scratch(n) doubles (split-K partials).
int64_t gram_gemm_scratch(int64_t n);
void launch_gram_gemm(const double* G, int64_t ldg, const double* V, double beta, double* Y, int64_t n, int k,
                      double* scratch, cudaStream_t s);

// G (cols x cols, row-major, leading dimension ldg) = X^T X of a dense row-major X
// (rows x cols, leading dimension ldx elements, fp32 != 0: float storage) on the FP64
// tensor cores, split over row ranges with the partials summed in a fixed order.
// Synchronizes the stream.  (The dense multi-right-hand-side operator: DESIGN.md §4.16.)
void syrk_dense_dmma(cudaStream_t s, const void* X, int fp32, int64_t ldx, int64_t rows, int64_t cols, double* G,
                     int64_t ldg);

// out (cols x k, row-major) = X^T B for the dense X above and a column-major block
// b_cm (k vectors of `rows`), one sweep of X per 16 columns, on the FP64 tensor cores;
// per-CTA partials summed in a fixed order.  scratch: xtb_scratch(rows, cols) doubles.
int64_t xtb_scratch(int64_t rows, int64_t cols);
void launch_xtb_dmma(cudaStream_t s, const void* X, int fp32, int64_t ldx, int64_t rows, int64_t cols,
                     const double* b_cm, int k, double* out, double* scratch);

// X_c = X P on the device (coarsening.cpp:112-148), bit-identical to the host
// restatement: per row, the products x_ri * w_i (separately rounded) of each
// coarse column summed from 0.0 in increasing fine-column order, the row's coarse
// columns ascending, explicit zeros from exact cancellation kept.  Row r's entries
// land at [xptr[r], xptr[r] + count[r]) of cidx / cval (a row of X_c has at most
// as many entries as the same row of X).
void coarsen_rows_gpu(cudaStream_t s, const int32_t* xptr, const int32_t* xidx, const double* xval, int64_t n,
                      const int32_t* label, const double* weight, int32_t* count, int32_t* cidx, double* cval);

}  // namespace rmg
