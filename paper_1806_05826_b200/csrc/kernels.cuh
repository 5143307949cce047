// Device kernels of the ridgemg_b200 solve path (sm_100a).
//
// Layout in HBM:
//   X    : CSR over samples  (ptr int32[N+1], idx int32[nnz], val fp64[nnz] or none)
//   X^T  : CSR over features (ptr int32[F+1], idx int32[nnz], val fp64[nnz] or none),
//          plus an nnz-balanced work-item schedule (Xt_Schedule) that splits
//          Zipf-heavy feature columns into fixed segments.
//   all vectors fp64, Krylov history as two contiguous rings [(m+1) x F].
// Every reduction is fixed-order (per-block tree + last-block sequential
// combine over slots), so results are run-to-run bit reproducible.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace rmg {

// Per-solve device scalars (one instance per Krylov solver / level).
struct KrylovScalars {
  double nb;        // ||rhs||
  double alpha;     // step length
  double pap;       // <p, Ap> of the current iteration
  double pr;        // <p, r>
  double rz;        // CG: <r, z>
  double beta_cg;   // CG: rz_next / rz
  double rel;       // ||r|| / ||rhs|| after the last iteration
  double tol;
  double lambda;    // power iteration
  int32_t it;       // iterations completed
  int32_t max_iters;
  int32_t done;     // 1 -> every kernel of this solver is a no-op
  int32_t converged;
  int32_t status;   // 0 ok, 1 <p,Ap> == 0, 2 <p,Ap> < 0 (or !>0 for CG), 3 non-finite rhs
  int32_t keep;     // FCG truncation m (ring has keep+1 slots)
  int32_t use;      // FCG: directions orthogonalized against in this iteration
  int32_t pad;
  double coeff[32]; // FCG Gram-Schmidt coefficients, oldest -> newest
  double pap_ring[33];
};

enum : int { kMaxKeep = 31 };

// Value storage of a sparse orientation.
enum class Val : int { Pattern = 0, F64 = 1 };

struct SparseDev {
  int64_t rows = 0, cols = 0, nnz = 0;
  const int32_t* ptr = nullptr;
  const int32_t* idx = nullptr;
  const uint16_t* idx16 = nullptr;  // narrow column indices when cols <= 65536 (K1)
  const double* val = nullptr;  // nullptr -> binary pattern
  int width = 8;                // lanes per row (4, 8, 16, 32)
  const int32_t* col_inv = nullptr;  // relabeled columns: original column of label j (K1 v-permute)
  double* vperm = nullptr;           // [cols] scratch: v in label order
  // SELL-32 (K1): slice s holds 32 rows column-major at [sell_off[s], sell_off[s+1])
  const int32_t* sell_off = nullptr;  // [n_slices + 1]
  const int32_t* sell_row = nullptr;  // [n_slices * 32] row of each slot (-1: padding)
  const int32_t* sell_len = nullptr;  // [n_slices * 32] elements of each slot
  int64_t n_slices = 0;
};

// Work items for the X^T pass, by row-length class of the X^T CSR:
//   short : {q_begin, q_end, -1, slot}  rows perm[q_begin..q_end), W lanes each
//   medium: {q_begin, q_end, -2, slot}  rows perm[..], one warp each
//   long  : {long_id, nz_begin, nz_end, seg_id}  one fixed segment, whole CTA
// (The epilogue-only pass k_xt_finish reads precomputed sums from `partial`.)
struct XtSchedule {
  const int4* items = nullptr;
  const int32_t* perm = nullptr;  // rows grouped by class (short, medium)
  int n_items = 0;
  int64_t features = 0;           // F
  double* partial = nullptr;      // k_xt_finish: precomputed sums s_j
  double* fin_slots = nullptr;    // k_xt_finish: dot slots
  unsigned* fin_ticket = nullptr;
  int fin_grid = 1;
  const int32_t* long_col = nullptr;
  const int32_t* long_first_seg = nullptr;
  const int32_t* long_nseg = nullptr;
  const int32_t* long_slot = nullptr;
  int n_long = 0, n_segs = 0, n_slots = 0;
  double* seg_partial = nullptr;  // [n_segs]
  unsigned* col_ticket = nullptr; // [n_long]
  double* slots = nullptr;        // [n_slots * 2]
  unsigned* grid_ticket = nullptr;
  int width = 8;                  // lanes per short column
  int stream_t = 0;               // gathers of t bypass L1 (large N, no reuse: the hybrid cold pass)
};

// Epilogue of the X^T pass, s_j = sum_r X(r,j) t_r:
enum class Epi : int {
  Plain = 0,   // out_j = s_j                                  (spmv_transpose)
  Axpby = 1,   // out_j = s_j + beta v_j                       (ridge / Galerkin apply)
  Fcg = 2,     // out_j = s_j + beta p_j; <p,Ap>, <p,r> -> alpha  (krylov.cpp:199-208)
  Cg = 3,      // out_j = s_j + beta p_j; <p,Ap> -> alpha = rz/pap (krylov.cpp:126-134)
  Rich = 4,    // out_j = z1_j + omega (r_j - (s_j + beta z1_j))   (krylov.cpp:417-418)
  Gram = 5     // out_j = s_j; ||out||^2 -> lambda               (krylov.cpp:80-81)
};

struct XtArgs {
  const double* t = nullptr;   // gathered N-vector
  const double* v = nullptr;   // p / z1 / w (beta term)
  const double* r = nullptr;   // residual (Fcg dots, Rich)
  double* out = nullptr;
  double beta = 0.0, omega = 0.0;
  KrylovScalars* sc = nullptr; // Fcg / Cg / Gram finalization
  const int32_t* done = nullptr;
  int ring_stride = 0;         // Fcg/Cg: v/out are ring bases, offset by (it % (keep+1)) * stride
};

// Hybrid X^T pass: the hot features (dense enough that a
// sample block holds several of their nonzeros) are summed per sample block
// from an SMEM copy of the block's slice of t; the rest uses the segmented K2.
constexpr int kHotBlockMax = 13824;  // samples per block: 108 KB of t in SMEM, 2 CTAs per SM
struct HotXtDev {
  const int32_t* ptr = nullptr;     // [nblk * H + 1], row (b, h) = b * H + h
  const uint16_t* idx16 = nullptr;  // sample offset inside block b
  const double* val = nullptr;      // nullptr: binary pattern
  const int32_t* feat = nullptr;    // [H] feature of hot row h
  double* partial = nullptr;        // [nblk * H]
  double* red2 = nullptr;           // [S * H]
  int H = 0, hA = 0, nblk = 0, B = 0, S = 1;
  int64_t N = 0;
};

// Dense X (row-major, fp64 or fp32 storage, fp64 arithmetic) for dense inputs
// (DESIGN.md §4.6): the operator X^T X is one fused sweep over X.
struct DenseDev {
  const void* data = nullptr;
  int fp32 = 0;            // 1: float storage
  int64_t ld = 0;          // elements per stored row (>= cols)
  int64_t rows = 0, cols = 0;
  double* partial = nullptr;  // [cols x n_cta] column-major per-CTA partial sums
  int n_cta = 0;
  double* fin_slots = nullptr;
  unsigned* fin_ticket = nullptr;
  int fin_grid = 1;
};
constexpr int kDenseMaxCols = 1024;  // 32 register partials per lane

// Block operator (BASELINE cfg 3: k right-hand sides as one SpMM; DESIGN.md
// §4.8): V, T and out are row-major blocks (F x k, N x k, F x k), so every
// gathered row of V or T is k contiguous doubles (one 128 B line at k = 16).
// A unit of work of the TMA gather passes (spmm_tma.cuh): (row of Y, first
// entry, one past the last entry, segment slot or -1).  Units are whole CSR
// rows, or <= 512-entry items of long rows whose segment partials
// k_block_finish combines.
struct TmaSpmm {
  const int4* units = nullptr;
  int n_units = 0;
  const int32_t* idx = nullptr;  // column (K1) / sample (X^T pass) indices
  const double* val = nullptr;   // nullptr: binary pattern
};

// The samples are split into chunks whose T slice (rows x 16 columns) stays in
// L2: per chunk, K1 writes its T rows, then the X^T pass over
// the same samples gathers them back from L2 and accumulates into out.
struct BlockXtSchedule {
  const int32_t* short_rows = nullptr;  // rows of X^T with <= 512 nonzeros in the chunk: one unit each
  int n_short = 0;
  const int4* items = nullptr;          // (row, k0, k1, seg) items of longer rows
  int n_items = 0;
  const int4* multi = nullptr;          // (row, first_seg, n_seg, -) rows split into several items
  int n_multi = 0;
  double* seg = nullptr;                // [n_items x 16] segment partials (seg >= 0)
  const int32_t* e_begin = nullptr;     // per X^T row: first entry whose sample lies in the chunk
  const int32_t* e_end = nullptr;       // per X^T row: one past its last entry in the chunk
  int64_t slice0 = 0, n_slices = 0;     // K1: the SELL slices holding the chunk's samples
  TmaSpmm tk1, tk2;                     // the same chunk as TMA gather units (K1 rows, X^T units)
};

// ---------------------------------------------------------------- launchers
void launch_spmv_rows(const SparseDev& x, const double* v, double* t, const int32_t* done,
                      cudaStream_t s);
void launch_spmv_rows_ring(const SparseDev& x, const double* v_ring, int ring_stride,
                           const KrylovScalars* sc, double* t, cudaStream_t s);
void launch_xt(const SparseDev& xt, const XtSchedule& sch, Epi epi, const XtArgs& a,
               cudaStream_t s);
void launch_chunk_combine(const double* part, int nchunks, int64_t F, const int32_t* list, int64_t nlist, double* out,
                          const int32_t* done, const KrylovScalars* sc, cudaStream_t s);
// dense X: out = epilogue(X^T (X v)) in one sweep (v may live in a ring: sc != nullptr)
void launch_dense_ata(const DenseDev& d, const double* v, int ring_stride, const KrylovScalars* sc, Epi epi,
                      const XtArgs& a, cudaStream_t s);
// dense X: y = X v (rows), out = X^T u (+ epilogue), out = beta + diag(X^T X)
void launch_dense_spmv(const DenseDev& d, const double* v, double* y, cudaStream_t s);
void launch_dense_xt(const DenseDev& d, const double* u, Epi epi, const XtArgs& a, cudaStream_t s);
void launch_dense_diag(const DenseDev& d, double beta, double* out, cudaStream_t s);
// out = X^T (X V) + beta V for a row-major F x k block (k <= 64); x: the K1
// layout (SELL), xt: X^T CSR (int32 sample indices), t: N x k scratch, vp:
// F x k scratch (relabeled columns).  Per column the arithmetic order is fixed.
// Hot features of the block X^T pass: summed per sample block of R
// rows from a shared-memory copy of the block's T rows, one 16-double partial per
// (block, hot feature), folded in block order; the cold features keep the chunked
// gather pass.
struct BlockHot {
  int H = 0, R = 0, nblk = 0;
  // per sample block: the hot features' entries cut into segments of <= 64, sorted by
  // length, 8 segments to a slice, stored as records like K1's (BlockK1v2; the label
  // is the row inside the block, padding = R, a zero row of the staged block)
  const int32_t* boff = nullptr;   // [nblk + 1] first slice of each block
  const int32_t* off = nullptr;    // [n_slices + 1] first record of each slice
  const int32_t* rec = nullptr;    // records (96 ints each; pattern: 32)
  const int32_t* feat = nullptr;   // [H] the hot features (most popular first)
  const int32_t* fptr = nullptr;   // [H + 1] each hot feature's partials ...
  const int32_t* fidx = nullptr;   // ... as rows of part, in (block, segment) order
  double* part = nullptr;          // [n_slices * 8][16] one partial per segment
  bool pattern = false;
};
// K1 split the same way: the H1 most popular labels' V rows staged in
// shared memory per persistent CTA and summed per row from a row-major CSR of the
// hot entries; the cold entries form a second SELL-32 layout (original columns)
// whose pass adds onto T.
struct BlockHotK1 {
  int H1 = 0;
  const int32_t* ptr = nullptr;    // [N + 1] hot entries of each row
  const uint16_t* lab = nullptr;   // popularity label (< H1)
  const double* val = nullptr;     // nullptr: binary pattern
  SparseDev cold;                  // the remaining entries, SELL-32, original column indices
};
// K1, third layout ("chunk-interleaved records"): slices of 8 rows
// (sorted by hot / cold length inside 1024-row windows), a 4-lane group per row.  A
// record holds 4 entries of each of the slice's 8 rows: int32 label[8][4], then (valued
// matrices) double value[8][4].  A slice's records are contiguous: first the nhot
// records of its hot entries (label < H1, in label order = descending popularity,
// padded with label H1 = a zero row of the shared-memory block, value 0), then the
// records of its cold entries (label >= H1, padded with -1, value 0).
struct BlockK1v2 {
  int H1 = 0;
  int64_t n_slices8 = 0;
  const int32_t* off = nullptr;    // [n_slices8 + 1] first record of each slice
  const int32_t* nhot = nullptr;   // [n_slices8] hot records of each slice
  const int32_t* srow = nullptr;   // [n_slices8 * 8] the sample in each slot (-1: none)
  const int32_t* rec = nullptr;    // records (96 ints each; pattern: 32)
  bool pattern = false;
};
void launch_ridge_block(const SparseDev& x, const SparseDev& xt, const BlockXtSchedule* chunks, int n_chunks,
                        const BlockHot& hot, const BlockHotK1& hot1, const BlockK1v2& k1v2, const double* v,
                        double* out, double beta, int k, double* t, double* vp, cudaStream_t s, bool xt_only = false);
// hot part of the hybrid X^T pass: writes sums[feat[h]] for every hot row h
void launch_xt_hot(const HotXtDev& h, const double* t, const int32_t* done, const KrylovScalars* sc, double* sums,
                   cudaStream_t s);
// Epilogue (+ deterministic dots) over precomputed sums s_j = (X^T t)_j, e.g.
// after an all-reduce of per-rank partial sums (row-sharded operator).
void launch_xt_epilogue(const double* sums, int64_t features, Epi epi, const XtArgs& a, double* fin_slots,
                        unsigned* fin_ticket, int fin_grid, cudaStream_t s);

// Krylov vector work (all read their dynamic scalars from KrylovScalars)
struct VecWork {
  double* slots = nullptr;     // [grid * 32]
  unsigned* ticket = nullptr;
  int grid = 1;
};
int vec_grid(int64_t n);
void launch_krylov_begin(const double* b, double* x, double* r, int64_t n, KrylovScalars* sc,
                         double* hist, const VecWork& w, cudaStream_t s);
void launch_fcg_gs(const double* z, const double* ap_ring, double* p_ring, int64_t n,
                   KrylovScalars* sc, const VecWork& w, cudaStream_t s);
void launch_fcg_axpy(double* x, double* r, const double* p_ring, const double* ap_ring, int64_t n,
                     KrylovScalars* sc, double* hist, const VecWork& w, cudaStream_t s);
void launch_cg_begin(const double* b, const double* inv_diag, double* x, double* r, double* z,
                     double* p, int64_t n, KrylovScalars* sc, double* hist, const VecWork& w,
                     cudaStream_t s);
void launch_cg_axpy(double* x, double* r, double* z, const double* inv_diag, const double* p,
                    const double* ap, int64_t n, KrylovScalars* sc, double* hist,
                    const VecWork& w, cudaStream_t s, bool general_m = false);
// symmetric Jacobi-smoothed V-cycle steps and general-preconditioner PCG (kernels.cu)
void launch_vc_pre(const double* r, const double* dinv, double w, double* x1, int64_t n, const int32_t* done,
                   cudaStream_t s);
void launch_vc_sub(const double* r, double* y, int64_t n, const int32_t* done, cudaStream_t s);
void launch_vc_add(const double* x1, double* e, int64_t n, const int32_t* done, cudaStream_t s);
// additive finest level (pcg_vcycle_additive): z = dinv r + w_i e_c(label_i)
void launch_vc_jacobi_prolong(const double* r, const double* dinv, const int32_t* label, const double* weight,
                              const double* ec, double* z, int64_t n, const int32_t* done, cudaStream_t s);
void launch_bvc_jacobi_prolong(const double* r, const double* dinv, const int32_t* label, const double* weight,
                               const double* ec, double* z, int64_t n, int k, cudaStream_t s);
void launch_vc_post(const double* x2, const double* r, const double* y2, const double* dinv, double w, double* z,
                    int64_t n, const int32_t* done, cudaStream_t s);
// batched pcg_vcycle (k right-hand sides in lock step; row-major n x k blocks)
struct BlockScalars {
  double nb, rz, alpha, beta, rel, pap, tol;
  int32_t it, max_iters, done, converged, status, pad;
};
void launch_bdots(const double* a, const double* b, int64_t n, int k, double* partial, int g, double* out,
                  cudaStream_t s);
void launch_bpcg_begin(BlockScalars* sc, const double* rr, const double* rz, const double* bad, int k, double* hist,
                       cudaStream_t s);
void launch_bpcg_alpha(BlockScalars* sc, const double* pap, int k, cudaStream_t s);
void launch_bupdate_xr(double* x, double* r, const double* p, const double* ap, const BlockScalars* sc, int64_t n,
                       int k, cudaStream_t s);
// the same update with the <r, r> partials formed in the same pass (+ their fixed-order sum into rr)
void launch_bupdate_xr_dot(double* x, double* r, const double* p, const double* ap, const BlockScalars* sc, int64_t n,
                           int k, double* partial, int g, double* rr, cudaStream_t s);
// z = D^-1 r + P e_c with the <r, z> partials formed in the same pass (+ their sum into rz)
void launch_bvc_jacobi_prolong_dot(const double* r, const double* dinv, const int32_t* label, const double* weight,
                                   const double* ec, double* z, int64_t n, int k, double* partial, int g, double* rz,
                                   cudaStream_t s);
void launch_bpcg_conv(BlockScalars* sc, const double* rr, int k, double* hist, cudaStream_t s);
void launch_bpcg_beta(BlockScalars* sc, const double* rz, int k, cudaStream_t s);
void launch_bupdate_p(double* p, const double* z, const BlockScalars* sc, int64_t n, int k, cudaStream_t s);
void launch_bvc_pre(const double* r, const double* dinv, double w, double* x1, int64_t n, int k, cudaStream_t s);
void launch_bvc_post(const double* x2, const double* r, const double* y2, const double* dinv, double w, double* z,
                     int64_t n, int k, cudaStream_t s);
void launch_bsub(const double* r, double* y, int64_t nk, cudaStream_t s);
void launch_badd(const double* x1, double* e, int64_t nk, cudaStream_t s);
void launch_brestrict(const int32_t* mptr, const int32_t* members, const double* weight, const double* y, double* rc,
                      int64_t nc, int k, cudaStream_t s);
void launch_bprolong(const int32_t* label, const double* weight, const double* ec, double* e, int64_t nf, int k,
                     cudaStream_t s);
void launch_bgemm_inv(const double* ainv, const double* rc, double* ec, int64_t nc, int k, cudaStream_t s);
void launch_bcol2row(const double* cm, double* rm, int64_t n, int k, cudaStream_t s);
void launch_brow2col(const double* rm, double* cm, int64_t n, int k, cudaStream_t s);
void launch_bnonfinite(const double* r, int64_t n, int k, double* bad, cudaStream_t s);
void launch_pcg_rz(const double* r, const double* z, int64_t n, KrylovScalars* sc, bool begin, const VecWork& w,
                   cudaStream_t s);
void launch_cg_update_p(double* p, const double* z, int64_t n, const KrylovScalars* sc,
                        cudaStream_t s);

// Aggregation (adjusted average, coarsening.cpp:30-55,82-100)
void launch_restrict(const int32_t* mptr, const int32_t* members, const double* weight,
                     const double* fine, double* coarse, int64_t n_coarse, const int32_t* done,
                     cudaStream_t s);
void launch_prolong(const int32_t* label, const double* weight, const double* coarse,
                    double* fine, int64_t n_fine, const int32_t* done, cudaStream_t s);
// dense y = A x (row-major n x n), coarsest direct solve through A_c^{-1}
void launch_dense_gemv(const double* a, const double* x, double* y, int64_t n,
                       const int32_t* done, cudaStream_t s);
// out = v / nrm (power iteration renormalization, krylov.cpp:84)
void launch_scale_by_lambda(const double* w, double* v, int64_t n, const KrylovScalars* sc,
                            cudaStream_t s);
void launch_diag_gram(const SparseDev& xt, const XtSchedule& sch, double beta, double* out, cudaStream_t s);
void launch_fill(double* p, double v, int64_t n, cudaStream_t s);
void launch_copy_inner_count(const KrylovScalars* inner, KrylovScalars* outer,
                             uint64_t* inner_hist, cudaStream_t s);

}  // namespace rmg
