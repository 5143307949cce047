// Persistent cooperative inner solver for small coarse levels (dense_level.cu).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "kernels.cuh"

namespace rmg {

struct DenseKrylovArgs {
  int n = 0, nc = 0, rows_per_cta = 1;
  int fcg = 1;                 // 1: FCG with z = omega r + M r; 0: plain CG (inner_cg)
  int keep = 20, max_iters = 500;
  double tol = 1e-6, omega = 0.0;
  const double* A = nullptr;   // n x n row-major, A = X_k^T X_k + beta_k I
  const double* M = nullptr;   // n x n row-major, (I - omega A) P A_{k+1}^{-1} P^T
  const double* b = nullptr;   // rhs
  double* x = nullptr;
  double* r = nullptr;
  double* p_ring = nullptr;
  double* ap_ring = nullptr;
  double* pap_ring = nullptr;  // [keep + 1]
  double* partials = nullptr;  // [grid * partial_stride]
  double* cg_rz_shared = nullptr;    // [2]
  double* cg_beta_shared = nullptr;  // [1]
  double* hist = nullptr;
  KrylovScalars* sc = nullptr;
  unsigned long long* timing = nullptr;  // diagnostics: [16 iterations][16 marks]
  int dbg = 0;  // diagnostics ablation (RMG_DENSE_DBG): 1 skip M r, 2 skip A p
};

struct DenseKrylovPlan {
  int grid = 1, rows_per_cta = 1, partial_stride = 40;
  bool smem_a = false;
  size_t smem_bytes = 0;
};

DenseKrylovPlan plan_dense_krylov(int n, int nc, int device);
void launch_dense_krylov(const DenseKrylovPlan& plan, const DenseKrylovArgs& args, cudaStream_t s);

}  // namespace rmg
