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
  const double* M = nullptr;   // dense: n x n row-major, (I - omega A) P A_{k+1}^{-1} P^T
  // low-rank FCG preconditioner (lowrank = 1): M r = Q (P^T r) with M = Q (n x nc,
  // row-major); unknowns held in next-level-cluster order (perm[i] = original
  // index of position i) so P^T r is a sum of per-CTA segment partials.
  int lowrank = 0;
  const int32_t* perm = nullptr;
  const int32_t* cid = nullptr;       // [n] cluster of position i (nondecreasing)
  const double* wts = nullptr;        // [n] aggregation weight of position i
  const int32_t* cta_seg0 = nullptr;  // [grid] first segment of each CTA
  const int32_t* cseg = nullptr;      // [nc + 1] segments of cluster c: [cseg[c], cseg[c+1])
  double* spart = nullptr;            // [3 n_segments] partial sums of w r (2 parities), of w Ap
  double* zfull = nullptr;            // [n] preconditioned residual (two-barrier kernel)
  int n_segments = 0;
  const double* b = nullptr;   // rhs (original order)
  double* x = nullptr;         // solution (solver order)
  double* x_out = nullptr;     // solution in the original order (== x when perm == nullptr)
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
  int max_clusters = 0;  // low-rank preconditioner: cluster segments the shared scratch holds
};

DenseKrylovPlan plan_dense_krylov(int n, int nc, int device);
void launch_dense_krylov(const DenseKrylovPlan& plan, const DenseKrylovArgs& args, cudaStream_t s);
// true when launch_dense_krylov runs the two-barrier kernel for these args
bool dense_two_barrier(const DenseKrylovArgs& a);

}  // namespace rmg
