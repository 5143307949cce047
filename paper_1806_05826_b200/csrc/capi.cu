// extern "C" boundary of ridgemg_b200 (include/ridgemg_b200.h).  Each entry
// point translates C++ exceptions into the status codes of the header and
// keeps the message in a thread-local buffer (rmg_last_error).
#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <new>
#include <string>
#include <thread>

#include "ridgemg_b200.h"
#include "ingest.hpp"
#include "runtime.cuh"

struct rmg_context {
  rmg::Context c;
  explicit rmg_context(int dev) : c(dev) {}
};
struct rmg_matrix {
  rmg::Matrix m;
  rmg_matrix(rmg::Context* ctx, rmg::HostCsr h, bool detect, rmg::Comm* comm = nullptr,
             const rmg::DenseInput* din = nullptr)
      : m(ctx, std::move(h), detect, comm, din) {}
  rmg_matrix(rmg::Context* ctx, int64_t n, int64_t f, const rmg::DenseInput& din) : m(ctx, n, f, din) {}
  rmg_matrix(rmg::Context* ctx, rmg::HostCsr local, int64_t n_global, int64_t row0, bool detect, rmg::Comm* comm)
      : m(ctx, std::move(local), n_global, row0, detect, comm) {}
  rmg_matrix(rmg::Context* ctx, int64_t n_global, int64_t row0, int64_t n_local, int64_t f,
             const rmg::DenseInput& din, rmg::Comm* comm)
      : m(ctx, n_global, row0, n_local, f, din, comm) {}
};
struct rmg_host_csr {
  rmg::HostCsr h;
};
struct rmg_comm {
  rmg::Comm c;
  rmg_comm(int nranks, int rank, const ncclUniqueId& id, int device) : c(nranks, rank, id, device) {}
  rmg_comm(int nranks, int rank, rmg_host_allreduce_fn fn, void* user) : c(nranks, rank, fn, user) {}
};
struct rmg_method {
  rmg::Method m;
  rmg::DBuf<double> b, rhs, w;  // staging for host-pointer calls
  rmg::DBuf<double> bb, wb;     // ... and for batched calls (kept: no allocation per call)
  template <class... A>
  explicit rmg_method(A&&... a) : m(std::forward<A>(a)...) {}
};

namespace {

thread_local std::string g_err;

template <class F>
int guard(F&& f) {
  try {
    f();
    return RMG_OK;
  } catch (const std::invalid_argument& e) {
    g_err = e.what();
    return RMG_ERR_INVALID_ARGUMENT;
  } catch (const rmg::CudaError& e) {
    g_err = e.what();
    return RMG_ERR_CUDA;
  } catch (const std::runtime_error& e) {
    g_err = e.what();
    return RMG_ERR_RUNTIME;
  } catch (const std::bad_alloc&) {
    g_err = "out of host memory";
    return RMG_ERR_INTERNAL;
  } catch (const std::exception& e) {
    g_err = e.what();
    return RMG_ERR_INTERNAL;
  } catch (...) {
    g_err = "unknown error";
    return RMG_ERR_INTERNAL;
  }
}

std::unique_lock<std::recursive_mutex> hold(rmg::Context* c) { return std::unique_lock<std::recursive_mutex>(c->mu); }

void need(const void* p, const char* what) {
  if (p == nullptr) throw rmg::InvalidArgument(std::string(what) + " must not be NULL");
}

// Device view of a caller vector: either the pointer itself or a staged copy.
const double* stage_in(rmg::Context& c, const double* p, size_t n, int32_t on_device, rmg::DBuf<double>& buf) {
  if (on_device) return p;
  if (buf.size() < std::max<size_t>(n, 1)) buf.alloc(std::max<size_t>(n, 1));
  if (n) RMG_CK(cudaMemcpyAsync(buf.get(), p, n * 8, cudaMemcpyHostToDevice, c.stream));
  return buf.get();
}
double* stage_out(size_t n, int32_t on_device, double* p, rmg::DBuf<double>& buf) {
  if (on_device) return p;
  if (buf.size() < std::max<size_t>(n, 1)) buf.alloc(std::max<size_t>(n, 1));
  return buf.get();
}
void finish_out(rmg::Context& c, const double* dev, double* host, size_t n, int32_t on_device) {
  if (!on_device && n) RMG_CK(cudaMemcpyAsync(host, dev, n * 8, cudaMemcpyDeviceToHost, c.stream));
  c.sync();
}

void fill_report(const rmg::SolveResult& r, uint64_t launches, rmg_solve_report* out) {
  if (!out) return;
  out->iterations = r.iterations;
  out->converged = r.converged ? 1 : 0;
  out->wall_time_s = r.wall;
  out->final_relative_residual = r.final_rel;
  out->kernel_launches = launches;
  if (out->residual_history)
    std::memcpy(out->residual_history, r.hist.data(), std::min<size_t>(out->residual_capacity, r.hist.size()) * 8);
  if (out->inner_iterations) {
    const size_t n = std::min<size_t>(out->inner_capacity, r.inner.size());
    for (size_t i = 0; i < n; ++i) out->inner_iterations[i] = r.inner[i];
  }
}

}  // namespace

extern "C" {

const char* rmg_last_error(void) { return g_err.c_str(); }

int rmg_version(int32_t* major, int32_t* minor) {
  return guard([&] {
    need(major, "major");
    need(minor, "minor");
    *major = 0;
    *minor = 1;
  });
}

int rmg_context_create(int32_t device, rmg_context** out) {
  return guard([&] {
    need(out, "out");
    *out = new rmg_context(device);
  });
}

int rmg_context_destroy(rmg_context* ctx) {
  return guard([&] { delete ctx; });
}

int rmg_context_set_stream(rmg_context* ctx, void* stream) {
  return guard([&] {
    need(ctx, "ctx");
    const auto lk_ = hold(&ctx->c);
    RMG_CK(cudaStreamSynchronize(ctx->c.stream));
    if (ctx->c.own_stream) cudaStreamDestroy(ctx->c.stream);
    ctx->c.own_stream = false;
    ctx->c.stream = static_cast<cudaStream_t>(stream);
  });
}

int rmg_context_synchronize(rmg_context* ctx) {
  return guard([&] {
    need(ctx, "ctx");
    const auto lk_ = hold(&ctx->c);
    ctx->c.sync();
  });
}

int rmg_matrix_create_csr(rmg_context* ctx, uint64_t n, uint64_t f, const uint64_t* rp, const uint64_t* ci,
                          const double* values, int32_t detect_pattern, rmg_matrix** out) {
  return guard([&] {
    need(ctx, "ctx");
    const auto lk_ = hold(&ctx->c);
    need(out, "out");
    need(rp, "row_offsets");
    rmg::HostCsr h;
    h.n = static_cast<int64_t>(n);
    h.f = static_cast<int64_t>(f);
    h.ptr.assign(rp, rp + n + 1);
    const uint64_t nnz = rp[n];
    if (nnz) need(ci, "column_indices");
    h.idx.assign(ci, ci + nnz);
    if (values) h.val.assign(values, values + nnz);
    RMG_CK(cudaSetDevice(ctx->c.device));
    *out = new rmg_matrix(&ctx->c, std::move(h), detect_pattern != 0);
  });
}

namespace {
// Host CSR view of a dense row-major array (setup: clustering, coarsening);
// exact zeros are not stored, fp32 values widen exactly.
rmg::HostCsr dense_to_csr(uint64_t n, uint64_t f, const void* data, uint64_t ld, int32_t fp32) {
  if (ld < f) throw rmg::InvalidArgument("dense X: leading dimension below the feature count");
  auto at = [&](uint64_t i, uint64_t j) {
    return fp32 ? static_cast<double>(static_cast<const float*>(data)[i * ld + j])
                : static_cast<const double*>(data)[i * ld + j];
  };
  rmg::HostCsr h;
  h.n = static_cast<int64_t>(n);
  h.f = static_cast<int64_t>(f);
  h.ptr.assign(n + 1, 0);
  const uint64_t T = std::max(1u, std::min(64u, std::thread::hardware_concurrency()));
  auto par = [&](auto fn) {  // contiguous row ranges per thread
    std::vector<std::thread> pool;
    for (uint64_t t = 0; t < T; ++t)
      pool.emplace_back([&, t] { fn(n * t / T, n * (t + 1) / T); });
    for (auto& th : pool) th.join();
  };
  par([&](uint64_t lo, uint64_t hi) {
    for (uint64_t i = lo; i < hi; ++i) {
      int64_t c = 0;
      for (uint64_t j = 0; j < f; ++j) c += at(i, j) != 0.0;
      h.ptr[i + 1] = c;
    }
  });
  for (uint64_t i = 0; i < n; ++i) h.ptr[i + 1] += h.ptr[i];
  h.idx.resize(h.ptr[n]);
  h.val.resize(h.ptr[n]);
  par([&](uint64_t lo, uint64_t hi) {
    for (uint64_t i = lo; i < hi; ++i) {
      int64_t q = h.ptr[i];
      for (uint64_t j = 0; j < f; ++j) {
        const double v = at(i, j);
        if (v != 0.0) {
          h.idx[q] = static_cast<int64_t>(j);
          h.val[q++] = v;
        }
      }
    }
  });
  return h;
}
}  // namespace

int rmg_matrix_create_dense(rmg_context* ctx, uint64_t n, uint64_t f, const void* data, uint64_t ld, int32_t fp32,
                            rmg_matrix** out) {
  return guard([&] {
    need(ctx, "ctx");
    const auto lk_ = hold(&ctx->c);
    need(out, "out");
    if (n != 0 && f != 0) need(data, "data");
    rmg::DenseInput din;
    din.data = data;
    din.fp32 = fp32 != 0;
    din.ld = static_cast<int64_t>(ld);
    RMG_CK(cudaSetDevice(ctx->c.device));
    if (std::getenv("RMG_DENSE_HOST_SETUP") != nullptr)  // diagnostics: setup from a host CSR view
      *out = new rmg_matrix(&ctx->c, dense_to_csr(n, f, data, ld, fp32), false, nullptr, &din);
    else  // no host CSR, hierarchy setup on the device
      *out = new rmg_matrix(&ctx->c, static_cast<int64_t>(n), static_cast<int64_t>(f), din);
  });
}

int rmg_matrix_create_dense_sharded(rmg_context* ctx, rmg_comm* comm, uint64_t n, uint64_t f, const void* data,
                                    uint64_t ld, int32_t fp32, rmg_matrix** out) {
  return guard([&] {
    need(ctx, "ctx");
    const auto lk_ = hold(&ctx->c);
    need(comm, "comm");
    need(out, "out");
    if (n != 0 && f != 0) need(data, "data");
    rmg::DenseInput din;
    din.data = data;
    din.fp32 = fp32 != 0;
    din.ld = static_cast<int64_t>(ld);
    RMG_CK(cudaSetDevice(ctx->c.device));
    *out = new rmg_matrix(&ctx->c, dense_to_csr(n, f, data, ld, fp32), false, &comm->c, &din);
  });
}

int rmg_comm_unique_id(uint8_t* id_out) {
  return guard([&] {
    need(id_out, "id_out");
    static_assert(sizeof(ncclUniqueId) == RMG_UNIQUE_ID_BYTES, "ncclUniqueId size");
    ncclUniqueId id;
    const ncclResult_t e = ncclGetUniqueId(&id);
    if (e != ncclSuccess) throw rmg::CudaError(std::string("ncclGetUniqueId: ") + ncclGetErrorString(e));
    std::memcpy(id_out, &id, sizeof(id));
  });
}

int rmg_comm_create(rmg_context* ctx, int32_t nranks, int32_t rank, const uint8_t* id, rmg_comm** out) {
  return guard([&] {
    need(ctx, "ctx");
    const auto lk_ = hold(&ctx->c);
    need(id, "id");
    need(out, "out");
    ncclUniqueId uid;
    std::memcpy(&uid, id, sizeof(uid));
    *out = new rmg_comm(nranks, rank, uid, ctx->c.device);
  });
}

int rmg_comm_create_host(rmg_context* ctx, int32_t nranks, int32_t rank, rmg_host_allreduce_fn fn, void* user,
                         rmg_comm** out) {
  return guard([&] {
    need(ctx, "ctx");
    need(out, "out");
    *out = new rmg_comm(nranks, rank, fn, user);
  });
}

int rmg_comm_destroy(rmg_comm* comm) {
  return guard([&] { delete comm; });
}

int rmg_matrix_create_csr_rows(rmg_context* ctx, rmg_comm* comm, uint64_t n, uint64_t row0, uint64_t n_local,
                               uint64_t f, const uint64_t* rp, const uint64_t* ci, const double* values,
                               int32_t detect_pattern, rmg_matrix** out) {
  return guard([&] {
    need(ctx, "ctx");
    const auto lk_ = hold(&ctx->c);
    need(comm, "comm");
    need(out, "out");
    need(rp, "row_offsets");
    if (rp[0] != 0) throw rmg::InvalidArgument("rmg_matrix_create_csr_rows: row offsets must be rebased to 0");
    rmg::HostCsr h;
    h.n = static_cast<int64_t>(n_local);
    h.f = static_cast<int64_t>(f);
    h.ptr.assign(rp, rp + n_local + 1);
    const uint64_t nnz = rp[n_local];
    if (nnz) need(ci, "column_indices");
    h.idx.assign(ci, ci + nnz);
    if (values) h.val.assign(values, values + nnz);
    RMG_CK(cudaSetDevice(ctx->c.device));
    *out = new rmg_matrix(&ctx->c, std::move(h), static_cast<int64_t>(n), static_cast<int64_t>(row0),
                          detect_pattern != 0, &comm->c);
  });
}

int rmg_matrix_create_dense_rows(rmg_context* ctx, rmg_comm* comm, uint64_t n, uint64_t row0, uint64_t n_local,
                                 uint64_t f, const void* data, uint64_t ld, int32_t fp32, rmg_matrix** out) {
  return guard([&] {
    need(ctx, "ctx");
    const auto lk_ = hold(&ctx->c);
    need(comm, "comm");
    need(out, "out");
    if (n_local != 0 && f != 0) need(data, "data");
    rmg::DenseInput din;
    din.data = data;
    din.fp32 = fp32 != 0;
    din.ld = static_cast<int64_t>(ld);
    RMG_CK(cudaSetDevice(ctx->c.device));
    *out = new rmg_matrix(&ctx->c, static_cast<int64_t>(n), static_cast<int64_t>(row0), static_cast<int64_t>(n_local),
                          static_cast<int64_t>(f), din, &comm->c);
  });
}

int rmg_matrix_create_csr_sharded(rmg_context* ctx, rmg_comm* comm, uint64_t n, uint64_t f, const uint64_t* rp,
                                  const uint64_t* ci, const double* values, int32_t detect_pattern, rmg_matrix** out) {
  return guard([&] {
    need(ctx, "ctx");
    const auto lk_ = hold(&ctx->c);
    need(comm, "comm");
    need(out, "out");
    need(rp, "row_offsets");
    rmg::HostCsr h;
    h.n = static_cast<int64_t>(n);
    h.f = static_cast<int64_t>(f);
    h.ptr.assign(rp, rp + n + 1);
    const uint64_t nnz = rp[n];
    if (nnz) need(ci, "column_indices");
    h.idx.assign(ci, ci + nnz);
    if (values) h.val.assign(values, values + nnz);
    RMG_CK(cudaSetDevice(ctx->c.device));
    *out = new rmg_matrix(&ctx->c, std::move(h), detect_pattern != 0, &comm->c);
  });
}

int rmg_matrix_shard(const rmg_matrix* m, uint64_t* row0, uint64_t* row1, int32_t* nranks, int32_t* rank) {
  return guard([&] {
    need(m, "matrix");
    if (row0) *row0 = static_cast<uint64_t>(m->m.row0);
    if (row1) *row1 = static_cast<uint64_t>(m->m.row1);
    if (nranks) *nranks = m->m.comm ? m->m.comm->nranks : 1;
    if (rank) *rank = m->m.comm ? m->m.comm->rank : 0;
  });
}

int rmg_shard_rows(const uint64_t* rp, uint64_t n, int32_t nranks, uint64_t* bounds_out) {
  return guard([&] {
    need(rp, "row_offsets");
    need(bounds_out, "bounds_out");
    const std::vector<int64_t> p(rp, rp + n + 1);
    const std::vector<int64_t> b = rmg::partition_rows(p, nranks);
    for (size_t i = 0; i < b.size(); ++i) bounds_out[i] = static_cast<uint64_t>(b[i]);
  });
}

int rmg_matrix_destroy(rmg_matrix* m) {
  return guard([&] {
    if (m == nullptr) return;
    const auto lk_ = hold(m->m.ctx);
    delete m;
  });
}

int rmg_matrix_shape(const rmg_matrix* m, uint64_t* n, uint64_t* f, uint64_t* nnz, int32_t* is_pattern) {
  return guard([&] {
    need(m, "matrix");
    if (n) *n = m->m.n();
    if (f) *f = m->m.f();
    if (nnz) *nnz = m->m.nnz();
    if (is_pattern) *is_pattern = m->m.pattern ? 1 : 0;
  });
}

int rmg_matrix_is_dense(const rmg_matrix* m, int32_t* dense, int32_t* fp32) {
  return guard([&] {
    need(m, "matrix");
    if (dense) *dense = m->m.dense ? 1 : 0;
    if (fp32) *fp32 = m->m.dense ? m->m.dense->view.fp32 : 0;
  });
}

int rmg_matrix_hot_layout(const rmg_matrix* m, uint64_t* hot_features, uint64_t* sample_blocks,
                          uint64_t* block_samples) {
  return guard([&] {
    need(m, "matrix");
    const bool on = m->m.hot != nullptr;
    if (hot_features) *hot_features = on ? static_cast<uint64_t>(m->m.hot->view.H) : 0;
    if (sample_blocks) *sample_blocks = on ? static_cast<uint64_t>(m->m.hot->view.nblk) : 0;
    if (block_samples) *block_samples = on ? static_cast<uint64_t>(m->m.hot->view.B) : 0;
  });
}

int rmg_spmv(rmg_matrix* m, const double* v, double* y, int32_t on_device) {
  return guard([&] {
    need(m, "matrix");
    const auto lk_ = hold(m->m.ctx);
    rmg::Context& c = *m->m.ctx;
    RMG_CK(cudaSetDevice(c.device));
    rmg::DBuf<double> bi, bo;
    const double* dv = stage_in(c, v, m->m.f(), on_device, bi);
    double* dy = stage_out(m->m.n(), on_device, y, bo);
    m->m.spmv(dv, dy);
    finish_out(c, dy, y, m->m.n(), on_device);
  });
}

int rmg_spmv_transpose(rmg_matrix* m, const double* u, double* y, int32_t on_device) {
  return guard([&] {
    need(m, "matrix");
    const auto lk_ = hold(m->m.ctx);
    rmg::Context& c = *m->m.ctx;
    RMG_CK(cudaSetDevice(c.device));
    rmg::DBuf<double> bi, bo;
    const double* du = stage_in(c, u, m->m.n(), on_device, bi);
    double* dy = stage_out(m->m.f(), on_device, y, bo);
    m->m.spmv_t(du, dy);
    finish_out(c, dy, y, m->m.f(), on_device);
  });
}

int rmg_ridge_apply(rmg_matrix* m, double beta, const double* w, double* out, int32_t on_device) {
  return guard([&] {
    need(m, "matrix");
    const auto lk_ = hold(m->m.ctx);
    if (beta < 0.0) throw rmg::InvalidArgument("RidgeOperator: beta must be nonnegative, got " + std::to_string(beta));
    rmg::Context& c = *m->m.ctx;
    RMG_CK(cudaSetDevice(c.device));
    rmg::DBuf<double> bi, bo;
    const double* dw = stage_in(c, w, m->m.f(), on_device, bi);
    double* dout = stage_out(m->m.f(), on_device, out, bo);
    rmg::XtArgs a;
    a.v = dw;
    a.out = dout;
    a.beta = beta;
    m->m.apply(dw, rmg::Epi::Axpby, a);
    finish_out(c, dout, out, m->m.f(), on_device);
  });
}

int rmg_ridge_apply_block(rmg_matrix* m, double beta, const double* v, double* out, uint64_t k, int32_t on_device) {
  return guard([&] {
    need(m, "matrix");
    const auto lk_ = hold(m->m.ctx);
    rmg::Context& c = *m->m.ctx;
    RMG_CK(cudaSetDevice(c.device));
    const size_t cnt = static_cast<size_t>(m->m.f()) * k;
    rmg::DBuf<double> bi, bo;
    const double* dv = stage_in(c, v, cnt, on_device, bi);
    double* dout = stage_out(cnt, on_device, out, bo);
    m->m.apply_block(dv, dout, beta, static_cast<int>(k));
    finish_out(c, dout, out, cnt, on_device);
  });
}

int rmg_gram_diagonal(rmg_matrix* m, double beta, double* out, int32_t on_device) {
  return guard([&] {
    need(m, "matrix");
    const auto lk_ = hold(m->m.ctx);
    rmg::Context& c = *m->m.ctx;
    RMG_CK(cudaSetDevice(c.device));
    rmg::DBuf<double> bo;
    double* d = stage_out(m->m.f(), on_device, out, bo);
    m->m.gram_diagonal(beta, d);
    finish_out(c, d, out, m->m.f(), on_device);
  });
}

int rmg_lambda_max(rmg_matrix* m, double tol, uint64_t max_iters, uint64_t seed, double* value, uint64_t* iterations,
                   int32_t* converged) {
  return guard([&] {
    need(m, "matrix");
    const auto lk_ = hold(m->m.ctx);
    need(value, "value");
    RMG_CK(cudaSetDevice(m->m.ctx->device));
    uint64_t it = 0;
    bool cv = false;
    *value = m->m.lambda_max(tol, max_iters, seed, &it, &cv);
    if (iterations) *iterations = it;
    if (converged) *converged = cv ? 1 : 0;
  });
}

int rmg_rng_normals(uint64_t seed, uint64_t n, double* out) {
  return guard([&] {
    need(out, "out");
    rmg::CounterRng rng(seed);
    for (uint64_t i = 0; i < n; ++i) out[i] = rng.next_normal();
  });
}

int rmg_generate_rhs(rmg_matrix* m, uint64_t seed, double* b_out, double* rhs_out) {
  return guard([&] {
    need(m, "matrix");
    const auto lk_ = hold(m->m.ctx);
    need(b_out, "b_out");
    rmg::CounterRng rng(seed);
    const int64_t n = m->m.n();
    for (int64_t i = 0; i < n; ++i) b_out[i] = rng.next_normal();
    if (rhs_out) {
      rmg::Context& c = *m->m.ctx;
      RMG_CK(cudaSetDevice(c.device));
      rmg::DBuf<double> bi, bo;
      const double* db = stage_in(c, b_out, n, 0, bi);
      double* dr = stage_out(m->m.f(), 0, rhs_out, bo);
      m->m.spmv_t(db, dr);
      finish_out(c, dr, rhs_out, m->m.f(), 0);
    }
  });
}

int rmg_synth_dense_clustered(uint64_t n, uint64_t f, uint64_t groups, double noise, uint64_t seed,
                              rmg_host_csr** out, uint64_t* nnz) {
  return guard([&] {
    need(out, "out");
    auto* h = new rmg_host_csr{rmg::synth_dense_clustered(static_cast<int64_t>(n), static_cast<int64_t>(f),
                                                          static_cast<int64_t>(groups), noise, seed)};
    *out = h;
    if (nnz) *nnz = h->h.nnz();
  });
}

int rmg_synth_sparse_zipf(uint64_t n, uint64_t f, double mean_nnz, double zipf_s, int32_t abs_normal_values,
                          uint64_t seed, rmg_host_csr** out, uint64_t* nnz) {
  return guard([&] {
    need(out, "out");
    auto* h = new rmg_host_csr{rmg::synth_sparse_zipf(static_cast<int64_t>(n), static_cast<int64_t>(f), mean_nnz,
                                                      zipf_s, abs_normal_values != 0, seed)};
    *out = h;
    if (nnz) *nnz = h->h.nnz();
  });
}

int rmg_synth_sparse_zipf_rows(uint64_t n, uint64_t f, double mean_nnz, double zipf_s, int32_t abs_normal_values,
                               uint64_t seed, rmg_host_csr** out, uint64_t* nnz) {
  return guard([&] {
    need(out, "out");
    auto* h = new rmg_host_csr{rmg::synth_sparse_zipf_rows(static_cast<int64_t>(n), static_cast<int64_t>(f),
                                                           mean_nnz, zipf_s, abs_normal_values != 0, seed)};
    *out = h;
    if (nnz) *nnz = h->h.nnz();
  });
}

int rmg_synth_sparse_zipf_row_range(uint64_t n, uint64_t f, double mean_nnz, double zipf_s,
                                    int32_t abs_normal_values, uint64_t seed, uint64_t row0, uint64_t row1,
                                    rmg_host_csr** out, uint64_t* nnz) {
  return guard([&] {
    need(out, "out");
    auto* h = new rmg_host_csr{rmg::synth_sparse_zipf_rows(static_cast<int64_t>(n), static_cast<int64_t>(f), mean_nnz,
                                                           zipf_s, abs_normal_values != 0, seed,
                                                           static_cast<int64_t>(row0), static_cast<int64_t>(row1))};
    *out = h;
    if (nnz) *nnz = h->h.nnz();
  });
}

int rmg_read_matrix_market(const char* path, rmg_host_csr** out, uint64_t* nnz) {
  return guard([&] {
    need(path, "path");
    need(out, "out");
    auto* h = new rmg_host_csr{rmg::read_matrix_market(path)};
    *out = h;
    if (nnz) *nnz = h->h.nnz();
  });
}

int rmg_host_csr_create(uint64_t n, uint64_t f, const uint64_t* rp, const uint64_t* ci, const double* v,
                        rmg_host_csr** out) {
  return guard([&] {
    need(rp, "row_offsets");
    need(out, "out");
    rmg::HostCsr h;
    h.n = static_cast<int64_t>(n);
    h.f = static_cast<int64_t>(f);
    h.ptr.assign(rp, rp + n + 1);
    if (rp[n]) need(ci, "column_indices");
    h.idx.assign(ci, ci + rp[n]);
    if (v) h.val.assign(v, v + rp[n]);
    rmg::validate_csr(h);
    *out = new rmg_host_csr{std::move(h)};
  });
}

int rmg_host_csr_shape(const rmg_host_csr* h, uint64_t* n, uint64_t* f, uint64_t* nnz, int32_t* has_values) {
  return guard([&] {
    need(h, "host csr");
    if (n) *n = static_cast<uint64_t>(h->h.n);
    if (f) *f = static_cast<uint64_t>(h->h.f);
    if (nnz) *nnz = static_cast<uint64_t>(h->h.nnz());
    if (has_values) *has_values = h->h.val.empty() ? 0 : 1;
  });
}

int rmg_host_csr_sha256(const rmg_host_csr* h, char* sha_hex) {
  return guard([&] {
    need(h, "host csr");
    need(sha_hex, "sha_hex");
    const std::string d = rmg::csr_sha256(h->h);
    std::memcpy(sha_hex, d.c_str(), d.size() + 1);
  });
}

int rmg_host_csr_save(const rmg_host_csr* h, const char* path) {
  return guard([&] {
    need(h, "host csr");
    need(path, "path");
    rmg::save_csr(h->h, path);
  });
}

int rmg_host_csr_load(const char* path, int32_t verify, rmg_host_csr** out, uint64_t* nnz, char* sha_hex) {
  return guard([&] {
    need(path, "path");
    need(out, "out");
    std::string d;
    auto* h = new rmg_host_csr{rmg::load_csr(path, verify != 0, &d)};
    *out = h;
    if (nnz) *nnz = h->h.nnz();
    if (sha_hex) std::memcpy(sha_hex, d.c_str(), d.size() + 1);
  });
}

int rmg_matrix_create_from_host(rmg_context* ctx, const rmg_host_csr* h, int32_t detect_pattern, rmg_matrix** out) {
  return guard([&] {
    need(ctx, "ctx");
    const auto lk_ = hold(&ctx->c);
    need(h, "host csr");
    need(out, "out");
    RMG_CK(cudaSetDevice(ctx->c.device));
    *out = new rmg_matrix(&ctx->c, h->h, detect_pattern != 0);
  });
}

int rmg_host_csr_export(const rmg_host_csr* h, uint64_t* rp, uint64_t* ci, double* v) {
  return guard([&] {
    need(h, "host csr");
    if (rp)
      for (int64_t i = 0; i <= h->h.n; ++i) rp[i] = static_cast<uint64_t>(h->h.ptr[i]);
    if (ci)
      for (int64_t k = 0; k < h->h.nnz(); ++k) ci[k] = static_cast<uint64_t>(h->h.idx[k]);
    if (v) {
      if (h->h.val.empty())
        std::fill(v, v + h->h.nnz(), 1.0);
      else
        std::memcpy(v, h->h.val.data(), h->h.val.size() * 8);
    }
  });
}

int rmg_host_csr_destroy(rmg_host_csr* h) {
  return guard([&] { delete h; });
}

int rmg_method_prepare(rmg_matrix* m, double beta, int32_t kind, const rmg_level_spec* levels, uint64_t n_levels,
                       const rmg_solver_config* solver, rmg_method** out) {
  return guard([&] {
    need(m, "matrix");
    const auto lk_ = hold(m->m.ctx);
    need(out, "out");
    rmg_solver_config cfg{1e-6, 1000, 20};
    if (solver) cfg = *solver;
    RMG_CK(cudaSetDevice(m->m.ctx->device));
    *out = new rmg_method(&m->m, beta, kind, levels, n_levels, cfg);
  });
}

int rmg_method_set_beta(rmg_method* pm, double beta) {
  return guard([&] {
    need(pm, "method");
    const auto lk_ = hold(pm->m.fine()->ctx);
    pm->m.set_beta(beta);
  });
}

int rmg_method_destroy(rmg_method* pm) {
  return guard([&] {
    if (pm == nullptr) return;
    const auto lk_ = hold(pm->m.fine()->ctx);
    delete pm;
  });
}

int rmg_method_solve_rhs(rmg_method* pm, const double* rhs, double* w_out, rmg_solve_report* report, int32_t on_device) {
  return guard([&] {
    need(pm, "method");
    const auto lk_ = hold(pm->m.fine()->ctx);
    need(rhs, "rhs");
    need(w_out, "w_out");
    rmg::Matrix& x = *pm->m.fine();
    rmg::Context& c = *x.ctx;
    RMG_CK(cudaSetDevice(c.device));
    const uint64_t l0 = c.launches;
    const double* drhs = stage_in(c, rhs, x.f(), on_device, pm->rhs);
    double* dw = stage_out(x.f(), on_device, w_out, pm->w);
    const rmg::SolveResult r = pm->m.solve_rhs(drhs, dw);
    finish_out(c, dw, w_out, x.f(), on_device);
    fill_report(r, c.launches - l0, report);
  });
}

int rmg_method_solve(rmg_method* pm, const double* b, double* w_out, rmg_solve_report* report, int32_t on_device) {
  return guard([&] {
    need(pm, "method");
    const auto lk_ = hold(pm->m.fine()->ctx);
    need(b, "b");
    need(w_out, "w_out");
    rmg::Matrix& x = *pm->m.fine();
    rmg::Context& c = *x.ctx;
    RMG_CK(cudaSetDevice(c.device));
    const uint64_t l0 = c.launches;
    const double* db = stage_in(c, b, x.n(), on_device, pm->b);
    if (pm->rhs.size() < static_cast<size_t>(std::max<int64_t>(1, x.f()))) pm->rhs.alloc(std::max<int64_t>(1, x.f()));
    x.spmv_t(db, pm->rhs.get());  // krylov.cpp:655, outside the solver timer
    double* dw = stage_out(x.f(), on_device, w_out, pm->w);
    const rmg::SolveResult r = pm->m.solve_rhs(pm->rhs.get(), dw);
    finish_out(c, dw, w_out, x.f(), on_device);
    fill_report(r, c.launches - l0, report);
  });
}

int rmg_method_solve_batch(rmg_method* pm, const double* b, double* w_out, uint64_t k, rmg_solve_report* reports,
                           int32_t on_device) {
  return guard([&] {
    need(pm, "method");
    need(b, "b");
    need(w_out, "w_out");
    const auto lk_ = hold(pm->m.fine()->ctx);
    rmg::Matrix& x = *pm->m.fine();
    const int64_t n = x.n(), f = x.f();
    if (k > 1 && k <= 64 && pm->m.block_capable() && std::getenv("RMG_BATCH_SEQ") == nullptr) {
      // pcg_vcycle: the k columns in lock step over the block operator
      rmg::Context& c = *x.ctx;
      RMG_CK(cudaSetDevice(c.device));
      const uint64_t l0 = c.launches;
      const double* db = stage_in(c, b, static_cast<size_t>(n) * k, on_device, pm->bb);
      double* dw = stage_out(static_cast<size_t>(f) * k, on_device, w_out, pm->wb);
      const std::vector<rmg::SolveResult> rs = pm->m.solve_block(db, dw, static_cast<int>(k));
      finish_out(c, dw, w_out, static_cast<size_t>(f) * k, on_device);
      for (uint64_t q = 0; q < k; ++q) fill_report(rs[q], (c.launches - l0) / k, reports ? reports + q : nullptr);
      return;
    }
    // column q of the column-major blocks b (n x k) and w (f x k) is one solve
    for (uint64_t q = 0; q < k; ++q) {
      const int rc = rmg_method_solve(pm, b + q * n, w_out + q * f, reports ? reports + q : nullptr, on_device);
      if (rc != RMG_OK) throw rmg::RuntimeError("rmg_method_solve_batch: right-hand side " + std::to_string(q) +
                                                ": " + g_err);
    }
  });
}

int rmg_method_precondition(rmg_method* pm, const double* r, double* z, int32_t on_device) {
  return guard([&] {
    need(pm, "method");
    const auto lk_ = hold(pm->m.fine()->ctx);
    rmg::Matrix& x = *pm->m.fine();
    rmg::Context& c = *x.ctx;
    RMG_CK(cudaSetDevice(c.device));
    const double* dr = stage_in(c, r, x.f(), on_device, pm->rhs);
    double* dz = stage_out(x.f(), on_device, z, pm->w);
    pm->m.precondition(dr, dz);
    finish_out(c, dz, z, x.f(), on_device);
  });
}

int rmg_method_info(const rmg_method* pm, uint64_t* n_levels, uint64_t* coarse_size) {
  return guard([&] {
    need(pm, "method");
    if (n_levels) *n_levels = pm->m.n_levels();
    if (coarse_size) *coarse_size = pm->m.coarse_size();
  });
}

int rmg_method_level(const rmg_method* pm, uint64_t level, uint64_t* n_features, uint64_t* nnz, double* beta,
                     double* omega) {
  return guard([&] {
    need(pm, "method");
    const auto lk_ = hold(pm->m.fine()->ctx);
    if (level >= static_cast<uint64_t>(pm->m.n_levels())) throw rmg::InvalidArgument("level index out of range");
    const rmg::Matrix& mk = pm->m.level_matrix(level);
    if (n_features) *n_features = mk.f();
    if (nnz) *nnz = mk.nnz();
    if (beta) *beta = pm->m.level_beta(level);
    if (omega) *omega = pm->m.omega(level);
  });
}

int rmg_method_level_labels(const rmg_method* pm, uint64_t level, int64_t* labels_out) {
  return guard([&] {
    need(pm, "method");
    const auto lk_ = hold(pm->m.fine()->ctx);
    need(labels_out, "labels_out");
    const auto& l = pm->m.labels(level);
    std::memcpy(labels_out, l.data(), l.size() * sizeof(int64_t));
  });
}

int rmg_method_level_matrix(const rmg_method* pm, uint64_t level, uint64_t* rp, uint64_t* ci, double* v) {
  return guard([&] {
    need(pm, "method");
    const auto lk_ = hold(pm->m.fine()->ctx);
    if (level >= static_cast<uint64_t>(pm->m.n_levels())) throw rmg::InvalidArgument("level index out of range");
    rmg::Matrix& mk = pm->m.level_matrix(level);
    if (mk.device_setup()) {  // device-resident dense level: every stored entry, row-major (nnz = N x F)
      const rmg::DenseDev& d = mk.dense->view;
      std::vector<double> buf(static_cast<size_t>(d.rows) * d.ld);
      if (d.fp32) {
        std::vector<float> fb(buf.size());
        if (!fb.empty()) RMG_CK(cudaMemcpy(fb.data(), d.data, fb.size() * 4, cudaMemcpyDeviceToHost));
        for (size_t q = 0; q < fb.size(); ++q) buf[q] = fb[q];
      } else if (!buf.empty()) {
        RMG_CK(cudaMemcpy(buf.data(), d.data, buf.size() * 8, cudaMemcpyDeviceToHost));
      }
      for (int64_t i = 0; i < d.rows; ++i) {
        if (rp) rp[i] = static_cast<uint64_t>(i * d.cols);
        for (int64_t j = 0; j < d.cols; ++j) {
          if (ci) ci[i * d.cols + j] = static_cast<uint64_t>(j);
          if (v) v[i * d.cols + j] = buf[i * d.ld + j];
        }
      }
      if (rp) rp[d.rows] = static_cast<uint64_t>(d.rows * d.cols);
      return;
    }
    const rmg::HostCsr& h = mk.host_csr();
    if (rp)
      for (int64_t i = 0; i <= h.n; ++i) rp[i] = static_cast<uint64_t>(h.ptr[i]);
    if (ci)
      for (int64_t k = 0; k < h.nnz(); ++k) ci[k] = static_cast<uint64_t>(h.idx[k]);
    if (v) std::memcpy(v, h.val.data(), h.val.size() * 8);
  });
}

int rmg_solve_system(rmg_matrix* m, double beta, int32_t kind, const rmg_level_spec* levels, uint64_t n_levels,
                     const rmg_solver_config* solver, const double* b, double* w_out, rmg_solve_report* report,
                     uint64_t* coarse_size) {
  rmg_method* pm = nullptr;
  int rc = rmg_method_prepare(m, beta, kind, levels, n_levels, solver, &pm);
  if (rc != RMG_OK) return rc;
  rc = rmg_method_solve(pm, b, w_out, report, 0);
  if (rc == RMG_OK && coarse_size) *coarse_size = pm->m.coarse_size();
  const std::string keep = g_err;
  rmg_method_destroy(pm);
  g_err = keep;
  return rc;
}

int rmg_method_time_operator(rmg_method* pm, uint64_t level, uint64_t reps, int32_t flush_l2, double* ms_per_apply,
                             double* ms_k1, double* ms_k2) {
  return guard([&] {
    need(pm, "method");
    const auto lk_ = hold(pm->m.fine()->ctx);
    double k1 = 0.0, k2 = 0.0;
    RMG_CK(cudaSetDevice(pm->m.fine()->ctx->device));
    const double t = pm->m.time_operator(level, reps, flush_l2 != 0, &k1, &k2);
    if (ms_per_apply) *ms_per_apply = t;
    if (ms_k1) *ms_k1 = k1;
    if (ms_k2) *ms_k2 = k2;
  });
}

// Diagnostics (not part of the public header): phase timestamps of the
// persistent inner solver of `level` (needs RMG_DENSE_TIMING at prepare time).
int rmg_debug_dense_timing(rmg_method* pm, uint64_t level, unsigned long long* out256) {
  return guard([&] {
    need(pm, "method");
    const auto lk_ = hold(pm->m.fine()->ctx);
    const rmg::DenseInner* d = pm->m.dense(level);
    if (d == nullptr || d->timing.get() == nullptr) throw rmg::InvalidArgument("no dense timing buffer");
    RMG_CK(cudaMemcpy(out256, d->timing.get(), 512 * sizeof(unsigned long long), cudaMemcpyDeviceToHost));
  });
}

int rmg_method_set_profiling(rmg_method* pm, int32_t on) {
  return guard([&] {
    need(pm, "method");
    const auto lk_ = hold(pm->m.fine()->ctx);
    pm->m.set_profiling(on != 0);
  });
}

int rmg_method_profile(const rmg_method* pm, uint64_t level, uint64_t* applications, double* ms_k1, double* ms_k2) {
  return guard([&] {
    need(pm, "method");
    const auto lk_ = hold(pm->m.fine()->ctx);
    if (level >= static_cast<uint64_t>(pm->m.n_levels())) throw rmg::InvalidArgument("level index out of range");
    const rmg::OpProfile& p = pm->m.profile(level);
    if (applications) *applications = p.count;
    if (ms_k1) *ms_k1 = p.ms_k1;
    if (ms_k2) *ms_k2 = p.ms_k2;
  });
}

}  // extern "C"
