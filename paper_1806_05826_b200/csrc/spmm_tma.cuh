// Block operator gathers by TMA: Y[row] = sum_e val_e * M[idx_e]
// over CSR units, M a row-major n_rows x ld fp64 block (16-column passes), the
// rows of M fetched into shared memory with cp.async.bulk.tensor ... tile::gather4
// (four 128-byte rows per instruction, completion on an mbarrier) instead of one
// register-held load per lane: a warp keeps 3 x 64 gathered rows in flight with
// no register cost, so the pass runs at L2 gather throughput rather than at the
// load-latency x occupancy product of the register-gather kernels.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "kernels.cuh"

namespace rmg {

// Opt-in (RMG_BLOCK_TMA=1, read when a matrix is uploaded and at launch):
// measured slower than the register-gather passes on cfg 3.
bool tma_spmm_enabled();
// true when enabled and M (ld doubles per row, 16-byte aligned rows) can be read by TMA
bool tma_spmm_ok(const void* m, int ld);

// K1: T[row * ld + c0 + q] = sum over the unit's entries of val * M[idx * ld + c0 + q]
void launch_spmm_tma_rows(const TmaSpmm& u, const double* M, int64_t m_rows, int ld, int c0, int kc, double* T,
                          cudaStream_t s);
// X^T pass with the chunked epilogue of k_xt_block (first / last chunk, beta V,
// segment partials for items of long rows)
void launch_spmm_tma_xt(const TmaSpmm& u, const double* M, int64_t m_rows, int ld, int c0, int kc, double* out,
                        const double* V, double beta, double* seg, int first, int last, cudaStream_t s);

}  // namespace rmg
