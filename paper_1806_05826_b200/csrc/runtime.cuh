// Host orchestration of the ridgemg_b200 solve path (device-resident data,
// host-sequenced kernels).  The C ABI in capi.cu wraps these classes.
#pragma once

#include <cuda_runtime.h>
#include <nccl.h>

#include <memory>
#include <mutex>
#include <string>
#include <vector>

#include "dense_level.cuh"
#include "host_setup.hpp"
#include "kernels.cuh"
#include "ridgemg_b200.h"

namespace rmg {

#define RMG_CK(expr)                                                                           \
  do {                                                                                         \
    const cudaError_t rmg_e_ = (expr);                                                         \
    if (rmg_e_ != cudaSuccess)                                                                 \
      throw ::rmg::CudaError(std::string(#expr) + " failed: " + cudaGetErrorString(rmg_e_)); \
  } while (0)

template <class T>
class DBuf {
 public:
  DBuf() = default;
  explicit DBuf(size_t n) { alloc(n); }
  DBuf(const DBuf&) = delete;
  DBuf& operator=(const DBuf&) = delete;
  DBuf(DBuf&& o) noexcept : p_(o.p_), n_(o.n_) {
    o.p_ = nullptr;
    o.n_ = 0;
  }
  DBuf& operator=(DBuf&& o) noexcept {
    if (this != &o) {
      release();
      p_ = o.p_;
      n_ = o.n_;
      o.p_ = nullptr;
      o.n_ = 0;
    }
    return *this;
  }
  ~DBuf() { release(); }
  void alloc(size_t n) {
    release();
    n_ = n;
    if (n) RMG_CK(cudaMalloc(&p_, n * sizeof(T)));
  }
  void release() {
    if (p_) cudaFree(p_);
    p_ = nullptr;
    n_ = 0;
  }
  void upload(const T* h, size_t n, cudaStream_t s) {
    if (n > n_) alloc(n);
    if (n) RMG_CK(cudaMemcpyAsync(p_, h, n * sizeof(T), cudaMemcpyHostToDevice, s));
  }
  T* get() const { return p_; }
  size_t size() const { return n_; }

 private:
  T* p_ = nullptr;
  size_t n_ = 0;
};

struct Context {
  // every C-ABI call that touches this context holds it: workspaces (matrix
  // scratch, method Krylov state) are per object and all device work is on one
  // stream, so serializing calls costs no GPU parallelism (krylov.hpp:172-175:
  // prepared methods accept concurrent solves)
  std::recursive_mutex mu;
  int device = 0;
  cudaStream_t stream = nullptr;
  bool own_stream = false;
  KrylovScalars* pinned_sc = nullptr;  // host mirror for per-iteration readback
  uint64_t launches = 0;               // kernels issued (diagnostics)
  // graphs are captured on this private stream (the caller's stream may be the
  // legacy default stream, which cannot capture) and launched on `stream`
  cudaStream_t capture_stream = nullptr;
  explicit Context(int dev);
  ~Context();
  void sync();
  KrylovScalars read(const KrylovScalars* dev);
  // read two scalar blocks with one synchronization (outer + inner solver)
  void read2(const KrylovScalars* a, KrylovScalars* ha, const KrylovScalars* b, KrylovScalars* hb);
};

// One orientation of a sparse matrix on the device.
struct DeviceSparse {
  SparseDev view;
  DBuf<int32_t> ptr, idx, col_inv, sell_off, sell_row, sell_len;
  DBuf<uint16_t> idx16;
  DBuf<double> val, vperm;
  // relabel: renumber columns by descending popularity (K1 gathers)
  void upload(const HostCsr& h, bool pattern, cudaStream_t s, bool narrow16 = false, bool relabel = false);
  // K1 layout: SELL-32 slices, rows length-sorted in 1024-row
  // windows, each row's elements in descending column popularity.
  void upload_sell(const HostCsr& h, bool pattern, cudaStream_t s, bool narrow16, bool relabel);
};

struct DeviceSchedule {
  XtSchedule view;
  DBuf<int4> items;
  DBuf<int32_t> perm, long_col, long_first, long_nseg, long_slot;
  DBuf<double> seg_partial, slots;
  DBuf<unsigned> col_ticket, grid_ticket;
  // xt: X^T CSR; features F; skip: rows left out of the schedule (the hot
  // rows of the hybrid pass)
  void build(const HostCsr& xt, cudaStream_t s, int64_t features, const std::vector<char>* skip = nullptr);
};


// In-situ timing of one level's operator kernels (CUDA events on the
// launching stream around K1 and K2 of every application).
struct OpProfile {
  std::vector<cudaEvent_t> pool;  // triples (before K1, between, after K2)
  size_t used = 0;
  uint64_t count = 0;
  double ms_k1 = 0.0, ms_k2 = 0.0;
  OpProfile() = default;
  OpProfile(const OpProfile&) = delete;
  OpProfile& operator=(const OpProfile&) = delete;
  ~OpProfile();
  void mark(cudaStream_t s);   // records the next event of the current triple
  void collect();              // after a stream sync: accumulate finished triples
  void reset();
};

// NCCL communicator over the GPUs of one node (one process per GPU).
// Sums over ranks: NCCL over NVLink, or host-staged (several ranks on one device,
// where NCCL refuses duplicate devices): the vector is copied to pinned host
// memory, `host_fn` replaces it by the sum over the ranks, and it is copied back.
typedef int (*HostAllreduceFn)(void* user, double* buf, uint64_t count);
struct Comm {
  ncclComm_t comm = nullptr;
  int nranks = 1, rank = 0;
  HostAllreduceFn host_fn = nullptr;
  void* host_user = nullptr;
  double* pinned = nullptr;
  size_t pinned_n = 0;
  Comm(int nranks, int rank, const ncclUniqueId& id, int device);
  Comm(int nranks, int rank, HostAllreduceFn fn, void* user);
  ~Comm();
  Comm(const Comm&) = delete;
  Comm& operator=(const Comm&) = delete;
  void allreduce(const double* send, double* recv, int64_t count, cudaStream_t s);
};

// nnz-balanced contiguous row blocks: bounds[r]..bounds[r+1] for rank r.
std::vector<int64_t> partition_rows(const std::vector<int64_t>& row_offsets, int nranks);

// X (N x F) and X^T on the device, with the X^T schedule and an N-vector scratch.
// With a communicator, only this rank's nnz-balanced row block of X lives on
// the device and every X^T pass ends in an all-reduce of the F-vector
// (north star: row sharding over NVLink); `host` keeps the full matrix for
// the (replicated) hierarchy setup.
// Hybrid X^T pass: sample-blocked hot features + segmented cold rest.
struct HotXt {
  HotXtDev view;
  DBuf<int32_t> ptr, feat;
  DBuf<uint16_t> idx16;
  DBuf<double> val, partial, red2;
  DeviceSchedule cold;  // segmented schedule over the cold rows only
  // when t outgrows the L2 (N > 8 M): the cold rows split by sample chunk, one
  // pass per chunk over its L2-resident t slice, partials combined in chunk order
  std::vector<DeviceSparse> chunk_x;
  std::vector<DeviceSchedule> chunk_sched;
  DBuf<double> chunk_part;  // [chunks][F]
  DBuf<int32_t> cold_list;  // the cold features (combine targets)
  int64_t n_cold = 0;
  // the cold pass runs on a side stream, concurrently with the hot pass
  // (RMG_XT_SERIAL=1: one stream)
  cudaStream_t side = nullptr;
  cudaEvent_t fork = nullptr, join = nullptr;
  ~HotXt() {
    if (fork) cudaEventDestroy(fork);
    if (join) cudaEventDestroy(join);
    if (side) cudaStreamDestroy(side);
  }
};

// Dense X on the device: row-major, fp64 or fp32 storage.
struct DenseInput {
  const void* data = nullptr;  // host, row-major n x f, leading dimension ld
  int fp32 = 0;
  int64_t ld = 0;
};
struct DenseStore {
  DenseDev view;
  DBuf<char> data;
  DBuf<double> partial, fin_slots;
  DBuf<unsigned> fin_ticket;
};

struct Matrix {
  Context* ctx = nullptr;
  HostCsr host;  // canonical CSR kept for setup (clustering, coarsening)
  bool pattern = false;
  DeviceSparse x, xt;
  DeviceSchedule sched;
  DBuf<double> t;             // X v scratch
  DBuf<KrylovScalars> gram_sc;  // power-iteration scalars
  Comm* comm = nullptr;       // row-sharded when non-null
  int64_t row0 = 0, row1 = 0; // this rank's rows of X (global numbering)
  DBuf<double> part, red, fin_slots;
  DBuf<unsigned> fin_ticket;
  int fin_grid = 1;
  std::unique_ptr<HotXt> hot;  // hybrid X^T pass when N is large (nullptr otherwise)
  std::unique_ptr<DenseStore> dense;  // dense inputs: X row-major on the device, no CSR copies
  // block operator (cfg 3): schedule of the X^T pass over row-major F x k blocks
  // one schedule per sample chunk: its X^T entry ranges, units and segments
  struct BlockChunkBufs {
    DBuf<int32_t> sh;
    DBuf<int4> it, mu, u1, u2;  // + the TMA passes' units (K1 rows, X^T rows and items)
  };
  DBuf<int32_t> bx_idx;        // X as a row CSR for the TMA K1 (entries in column order)
  DBuf<double> bx_val;
  BlockHot bhot;               // hot features of the block X^T pass (H = 0: none)
  BlockHotK1 bhot1;            // hot labels of the block K1 (H1 = 0: none)
  DBuf<int32_t> bh1_ptr;
  DBuf<uint16_t> bh1_lab;
  DBuf<double> bh1_val;
  DeviceSparse bh1_cold;
  BlockK1v2 bk1v2;             // chunk-interleaved K1 layout (H1 = 0: none)
  DBuf<int32_t> bk_off, bk_nhot, bk_srow, bk_rec;
  DBuf<int32_t> bh_boff, bh_off, bh_rec, bh_feat, bh_fptr, bh_fidx;
  DBuf<double> bh_part;
  std::vector<BlockChunkBufs> bchunk_bufs;
  std::vector<BlockXtSchedule> bviews;
  DBuf<int32_t> bbounds;       // (chunks + 1) x F entry offsets into X^T
  int64_t bchunk_rows = 0;
  DBuf<double> bseg, bt, bvp;  // + scratch T (N x k) and permuted V (F x k), kept across calls
  void build_block_schedule(const HostCsr& x, const HostCsr& ht);
  void build_block_hot(const HostCsr& ht, const std::vector<int32_t>& feat, int64_t R, int64_t nblk);
  void build_k1v2(const HostCsr& xr, const std::vector<int32_t>& rank, int64_t h1);
  // out = X^T (X V) + beta V, V and out row-major F x k (device pointers)
  void apply_block(const double* v, double* out, double beta, int k, bool sync = true);
  void ensure_block_gram();    // dense X: G = X^T X on the FP64 tensor cores, once
  void ensure_block_schedule();  // CSR X: the block layouts, on the first block call
  bool block_built = false;
  DBuf<double> bgram, bgram_scratch;
  int64_t bgram_ld = 0;
  // out (F x k, row-major) = X^T B for k columns given column-major (B_cm: k vectors of N): the block X^T pass
  void xt_block_cm(const double* b_cm, double* out, int k);
  // defer_operator: a coarse level of a V-cycle hierarchy that may never apply X_k (it enters
  // additively, or its Gram matrix is kept dense): the K1 layout and the hot X^T blocks are
  // built by ensure_operator() on the first application instead (never inside a graph capture:
  // build_vcycle applies every level that smooths once, at prepare)
  Matrix(Context* c, HostCsr h, bool detect_pattern, Comm* comm = nullptr, const DenseInput* din = nullptr,
         bool defer_operator = false);
  // per-rank input: `local` holds rows [row0, row0 + local.n) of an n_global-row X
  // (row offsets rebased); every setup step on it is sharded (rmg_matrix_create_csr_rows)
  Matrix(Context* c, HostCsr local, int64_t n_global, int64_t row0, bool detect_pattern, Comm* comm,
         bool defer_operator = false);
  bool defer_op = false, op_ready = true;
  void ensure_operator();
  void upload_k1(const HostCsr& local);
  int64_t n_global = -1;
  bool rows_only = false;  // host holds only this rank's rows
  void init_sparse(const HostCsr& local);
  void alloc_comm_buffers();
  // dense X without a host CSR (setup on the device): from host
  // rows, or from a device buffer already padded to ld (coarse levels)
  Matrix(Context* c, int64_t n, int64_t f, const DenseInput& din);
  Matrix(Context* c, int64_t n, int64_t f, DBuf<char>&& data, int fp32, int64_t ld);
  // per-rank dense input: rows [row0, row0 + n_local) of an n_global x f X (host rows,
  // or a device buffer padded to ld for coarse levels); setup on it is sharded
  Matrix(Context* c, int64_t n_global, int64_t row0, int64_t n_local, int64_t f, const DenseInput& din, Comm* comm);
  Matrix(Context* c, int64_t n_global, int64_t row0, int64_t n_local, int64_t f, DBuf<char>&& data, int fp32,
         int64_t ld, Comm* comm);
  bool host_ok = true;  // host holds the CSR view
  const HostCsr& host_csr();  // built from the device copy on first use
  bool device_setup() const { return dense != nullptr && comm == nullptr && !host_ok; }
  std::vector<double> gram_cache;  // X^T X of a device-resident level (beta-independent)
  void init_dense(DBuf<char>&& data, int fp32, int64_t ld, int64_t rows);
  void init_dense_from_host(const void* data, int fp32, int64_t ld_in, int64_t rows);
  void build_hot(const HostCsr& ht, int64_t n_samples);
  int64_t n_local() const { return row1 - row0; }
  void allreduce_sums(double* sendbuf, double* recvbuf, int64_t count);
  int64_t n() const { return n_global >= 0 ? n_global : host.n; }
  int64_t f() const { return host.f; }
  int64_t nnz() const { return host_ok ? host.nnz() : host.n * host.f; }
  // t = X v then the X^T epilogue; v may live in a ring (sc != nullptr)
  void apply(const double* v, Epi epi, const XtArgs& args, OpProfile* prof = nullptr);
  void apply_ring(const double* v_ring, int stride, const KrylovScalars* sc, Epi epi, const XtArgs& args,
                  OpProfile* prof = nullptr);
  void spmv(const double* v, double* y);
  void spmv_t(const double* u, double* y);
  void gram_diagonal(double beta, double* out);
  double lambda_max(double tol, uint64_t max_iters, uint64_t seed, uint64_t* iters, bool* conv);
};

// Solver workspace for one level.
struct KrylovWork {
  int64_t n = 0;
  int keep = 20;
  DBuf<double> b, x, r, z, z1, p_ring, ap_ring, hist, inv_diag;
  DBuf<uint64_t> inner_hist;
  DBuf<KrylovScalars> sc;
  DBuf<double> slots;
  DBuf<unsigned> ticket;
  VecWork vw;
  KrylovWork(int64_t n, int keep, uint64_t max_iters, double tol, cudaStream_t s);
  void set_params(double tol, uint64_t max_iters, int keep_m, cudaStream_t s);
  uint64_t max_iters = 0;
};

struct LevelSpecHost {
  rmg_level_spec spec{};
  std::vector<int64_t> labels;  // imported labels (copied)
};

struct CoarseLevelDev {
  std::unique_ptr<Matrix> mat;  // X_k, k >= 1
  Aggregation agg;              // level k-1 -> k
  DBuf<int32_t> label, mptr, members;
  DBuf<double> weight;
  DeviceSparse pt;           // P^T as CSR (clusters x fine features), for the restriction
  DeviceSchedule pt_sched;   // nnz-balanced: giant clusters are split into segments
  double beta = 0.0;
};

// Dense persistent inner solve of one coarse level (dense_level.cu).
struct DenseInner {
  DenseKrylovPlan plan;
  bool fcg = true;
  double omega = 0.0;
  int nc = 0;
  DBuf<double> A, Q, pap_ring, partials, cg_shared;
  DBuf<unsigned long long> timing;  // RMG_DENSE_TIMING diagnostics
  // low-rank preconditioner (dense_level.cu): unknowns in next-level cluster order
  bool lowrank = false;
  int n_segments = 0;
  DBuf<int32_t> perm, cid, cta_seg0, cseg;
  DBuf<double> wts, spart, xp, zfull;
  std::vector<float> tuned_ms;      // partials placement candidates (ms per 40 iterations)
  int tuned_pick = 0;
};

struct SolveResult {
  uint64_t iterations = 0;
  bool converged = false;
  double wall = 0.0;
  double final_rel = 0.0;
  std::vector<double> hist;
  std::vector<uint64_t> inner;
};

class Method {
 public:
  Method(Matrix* x, double beta, int kind, const rmg_level_spec* levels, uint64_t n_levels,
         const rmg_solver_config& solver);
  SolveResult solve_rhs(const double* rhs_dev, double* w_dev);
  // rebuild the beta-dependent parts for a new regularization (same hierarchy)
  void set_beta(double beta);
  void precondition(const double* r_dev, double* z_dev);
  int64_t n_levels() const { return static_cast<int64_t>(coarse_.size()) + 1; }
  int64_t coarse_size() const { return coarse_.empty() ? 0 : coarse_[0]->mat->f(); }
  Matrix& level_matrix(size_t k) const { return k == 0 ? *fine_ : *coarse_[k - 1]->mat; }
  double level_beta(size_t k) const { return k == 0 ? beta_ : coarse_[k - 1]->beta; }
  // the level's smoothing weight: Richardson omega_k (krylov.cpp:539-546), or the
  // damped-Jacobi weight for pcg_vcycle
  double omega(size_t k) const {
    if (vc_kind()) return k < vc_.size() ? vc_[k]->w : 0.0;
    return k < omega_.size() ? omega_[k] : 0.0;
  }
  const std::vector<int64_t>& labels(size_t k) const;
  Matrix* fine() const { return fine_; }
  int kind() const { return kind_; }
  // pcg_vcycle and its additive-fine-level variant share the hierarchy, smoothers and cycle
  bool vc_kind() const { return kind_ == RMG_METHOD_PCG_VCYCLE || kind_ == RMG_METHOD_PCG_VCYCLE_ADDITIVE; }
  // pcg_vcycle_additive: the finest level enters additively, and so does every level
  // whose spec says so (rmg_level_spec.additive)
  bool vc_additive(size_t k) const {
    return kind_ == RMG_METHOD_PCG_VCYCLE_ADDITIVE && (k == 0 || (k < specs_.size() && specs_[k].spec.additive != 0));
  }
  rmg_solver_config solver;
  double time_operator(size_t level, uint64_t reps, bool flush, double* k1_ms, double* k2_ms);
  void set_profiling(bool on);
  const OpProfile& profile(size_t level) const { return *prof_.at(level); }
  const DenseInner* dense(size_t level) const { return level < dense_.size() ? dense_[level].get() : nullptr; }

 private:
  uint64_t precond(size_t k, const double* r, double* z);
  uint64_t run_fcg(size_t k, const double* rhs, bool record, SolveResult* out);
  uint64_t run_cg(size_t k, const double* rhs, const double* inv_diag, bool record, SolveResult* out);
  OpProfile* prof(size_t k) { return profiling_ ? prof_[k].get() : nullptr; }
  void collect_profiles();
  bool profiling_ = false;
  std::vector<std::unique_ptr<OpProfile>> prof_;
  Context* ctx_;
  Matrix* fine_;
  double beta_;
  int kind_;
  std::vector<LevelSpecHost> specs_;
  std::vector<std::unique_ptr<CoarseLevelDev>> coarse_;
  std::vector<double> omega_, lambda_;
  std::vector<std::unique_ptr<KrylovWork>> work_;  // per level 0..L-1
  std::vector<std::unique_ptr<DenseInner>> dense_;  // per level (nullptr: host-sequenced path)
  void build_dense_levels(const std::vector<double>& ainv_host);
  uint64_t run_dense(size_t k, const double* rhs);
  uint64_t run_fgmres(const double* rhs, SolveResult* out);
  void jacobi_diag();
  std::vector<double> level_gram(Matrix& m, double beta);
  // pcg_vcycle: per smoothed level k < L, D_k^-1 and the
  // damped-Jacobi weight 1 / lambda_max(D_k^-1 A_k); scratch x1, y, e
  struct VcLevel {
    DBuf<double> dinv, x1, y, e;
    double w = 0.0;
  };
  std::vector<std::unique_ptr<VcLevel>> vc_;
  void build_vcycle();
  // pcg_vcycle's iteration as a CUDA graph inside a device-side while loop (a
  // conditional node whose condition a kernel sets from the solver's done flag):
  // one graph launch per solve, no host round trip per iteration
  struct GraphLoop {
    cudaGraph_t g = nullptr;
    cudaGraphExec_t exec = nullptr;
    uint64_t launches_per_iter = 0;
    DBuf<unsigned long long> passes;  // loop guard (reset before each launch)
    ~GraphLoop() {
      if (exec) cudaGraphExecDestroy(exec);
      if (g) cudaGraphDestroy(g);
    }
  };
  std::unique_ptr<GraphLoop> vc_graph_;
  std::unique_ptr<GraphLoop> fcg_graph_;  // the outer FCG loop when no inner level needs the host
  std::unique_ptr<GraphLoop> cg_graph_[2];  // level-0 cg, jacobi_cg
  std::unique_ptr<GraphLoop> bw_graph_;     // batched pcg_vcycle (k columns)
  int bw_graph_k_ = 0;
  // set_beta retires a loop graph instead of destroying it: the previous one is destroyed
  // there (between solves) and one executable graph stays alive while the next is
  // instantiated inside the following solve -- with none alive, capture + instantiate of the
  // next took 23 ms instead of 0.3 ms in one solve out of three to ten
  // (profiles/r2_bench_graph_retire.log)
  std::unique_ptr<GraphLoop> bw_graph_retired_, vc_graph_retired_;
  void block_iteration(int k);
  bool build_block_graph(int k);
  void set_beta_impl(double beta);
  void fcg_iteration(size_t k);
  bool build_fcg_graph();
  void pcg_vcycle_iteration();
  bool build_vcycle_graph();
  void vcycle(size_t k, const double* r, double* z, const int32_t* done);
  uint64_t run_pcg_vcycle(const double* rhs, SolveResult* out);
  // batched pcg_vcycle: k right-hand sides in lock step over the block operator
  struct BlockLevel {
    DBuf<double> x1, y, e, rc, ec;
  };
  std::vector<std::unique_ptr<BlockLevel>> bl_;
  struct BlockWork {
    int k = 0;
    DBuf<double> x, r, z, p, ap, rhs_cm, partial, dots, hist;
    DBuf<BlockScalars> sc;
  } bw_;
  void bvcycle(size_t lv, const double* r, double* z, int k);
  // z = M r for k columns: the V-cycle, Jacobi (z = D^-1 r) or identity (cg)
  void bprecond(const double* r, double* z, int k);
  // solve_block -> bvcycle: where an additive finest level leaves the partials of <r, z>
  double* brz_partial_ = nullptr;
  double* brz_out_ = nullptr;
  int brz_g_ = 0;
  bool brz_done_ = false;
  // pcg_vcycle: dense G_k = X_k^T X_k per level k >= 1 where n_k^2 doubles are
  // fewer bytes than an X_k sweep pair; nullptr: sweep X_k
  struct DenseGram {
    DBuf<double> G, scratch;  // + split-K partials of the block GEMM
    int64_t n = 0, ld = 0;
  };
  std::vector<std::unique_ptr<DenseGram>> dg_;
  bool dg_built_ = false;
  void build_dense_grams();
  const DenseGram* dgram(size_t k) const { return k < dg_.size() ? dg_[k].get() : nullptr; }
  // G = X^T X of a level on the device (bit-identical to coarse_gram's sums)
  void device_gram(Matrix& m, double* G, int64_t ld);
  // X_c = X P of a sparse level on the device (bit-identical to coarsen)
  HostCsr coarsen_level(Matrix& m, const Aggregation& agg);

 public:
  // pcg_vcycle over single-GPU CSR levels: solve_batch runs the k columns in lock step
  bool block_capable() const;
  // b_cm: column-major n_samples x k (device), w_cm: column-major F x k (device)
  std::vector<SolveResult> solve_block(const double* b_cm, double* w_cm, int k);

 private:
  std::vector<int64_t> sketch_clustering(Matrix& m, const rmg_level_spec& cs, int64_t* nc);
  DBuf<double> gm_basis_, gm_z_, gm_h_, gm_part_;  // FGMRES: basis, preconditioned basis, Hessenberg column
  DenseKrylovArgs dense_args(size_t k, const double* rhs);
  void tune_dense_partials(size_t k);
  DBuf<double> ainv_, rc_last_, ec_last_;
  DBuf<char> pad_;  // RMG_DENSE_PAD diagnostics
  std::vector<DBuf<char>> pads_;
  DBuf<double> inv_diag_;
  std::vector<std::vector<int64_t>> labels_;
};

}  // namespace rmg
