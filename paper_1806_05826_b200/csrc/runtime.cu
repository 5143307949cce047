// Host orchestration of the ridgemg_b200 solve path.  See runtime.cuh.
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <numeric>
#include <thread>

#include "runtime.cuh"
#include "dense_gram.cuh"
#include "spmm_tma.cuh"
#include "fgmres.cuh"
#include "dense_setup.hpp"
#include "kmeans_gpu.hpp"

namespace rmg {

namespace {
// graph while-loops (pcg_vcycle, outer FCG): continue while the solver is not done
// (a guard counter bounds every device-side loop at `limit` passes: if a done flag
// were never raised the host loop takes over instead of the GPU spinning forever)
__global__ void k_set_while(cudaGraphConditionalHandle h, const int32_t* done, unsigned long long* passes,
                            unsigned long long limit) {
  const unsigned long long c = ++*passes;
  cudaGraphSetConditional(h, (*done || c >= limit) ? 0u : 1u);
}
// batched solves: continue while any column runs
__global__ void k_set_while_any(cudaGraphConditionalHandle h, const BlockScalars* sc, int k,
                                unsigned long long* passes, unsigned long long limit) {
  unsigned run = 0;
  for (int c = 0; c < k; ++c) run |= sc[c].done ? 0u : 1u;
  const unsigned long long c = ++*passes;
  cudaGraphSetConditional(h, (run != 0u && c < limit) ? 1u : 0u);
}
}  // namespace

// A graph holding one while node whose body is `body()` (captured on the
// context's private capture stream, with ctx->stream pointing at it meanwhile)
// followed by the kernel that re-evaluates the condition from `done`.
bool capture_while_graph(Context* ctx, const int32_t* done, const std::function<void()>& body, cudaGraph_t* g_out,
                         cudaGraphExec_t* exec_out, uint64_t* launches_out, unsigned long long* passes,
                         unsigned long long limit, const BlockScalars* block_sc = nullptr, int block_k = 0) {
  cudaGraph_t g = nullptr;
  if (cudaGraphCreate(&g, 0) != cudaSuccess) return false;
  auto fail = [&] {
    cudaGetLastError();
    if (g) cudaGraphDestroy(g);
    return false;
  };
  cudaGraphConditionalHandle h;
  if (cudaGraphConditionalHandleCreate(&h, g, 1, cudaGraphCondAssignDefault) != cudaSuccess) return fail();
  cudaGraphNodeParams cp = {};
  cp.type = cudaGraphNodeTypeConditional;
  cp.conditional.handle = h;
  cp.conditional.type = cudaGraphCondTypeWhile;
  cp.conditional.size = 1;
  cudaGraphNode_t node;
  if (cudaGraphAddNode(&node, g, nullptr, 0, &cp) != cudaSuccess) return fail();
  cudaGraph_t bodyg = cp.conditional.phGraph_out[0];
  if (ctx->capture_stream == nullptr &&
      cudaStreamCreateWithFlags(&ctx->capture_stream, cudaStreamNonBlocking) != cudaSuccess)
    return fail();
  const cudaStream_t orig = ctx->stream;
  if (cudaStreamBeginCaptureToGraph(ctx->capture_stream, bodyg, nullptr, nullptr, 0, cudaStreamCaptureModeRelaxed) !=
      cudaSuccess)
    return fail();
  ctx->stream = ctx->capture_stream;
  const uint64_t l0 = ctx->launches;
  bool ok = true;
  try {
    body();
    if (block_sc != nullptr)
      k_set_while_any<<<1, 1, 0, ctx->stream>>>(h, block_sc, block_k, passes, limit);
    else
      k_set_while<<<1, 1, 0, ctx->stream>>>(h, done, passes, limit);
  } catch (...) {
    ok = false;
  }
  ctx->stream = orig;
  cudaGraph_t captured = nullptr;
  const cudaError_t ec = cudaStreamEndCapture(ctx->capture_stream, &captured);
  if (!ok || ec != cudaSuccess || cudaGetLastError() != cudaSuccess) return fail();
  *launches_out = ctx->launches - l0 + 1;
  ctx->launches = l0;
  if (cudaGraphInstantiate(exec_out, g, 0) != cudaSuccess) return fail();
  *g_out = g;
  return true;
}

// ------------------------------------------------------------------ Context
Context::Context(int dev) : device(dev) {
  int n = 0;
  RMG_CK(cudaGetDeviceCount(&n));
  if (dev < 0 || dev >= n) throw InvalidArgument("rmg_context_create: device " + std::to_string(dev) + " not present");
  RMG_CK(cudaSetDevice(dev));
  RMG_CK(cudaStreamCreateWithFlags(&stream, cudaStreamNonBlocking));
  own_stream = true;
  RMG_CK(cudaMallocHost(&pinned_sc, 2 * sizeof(KrylovScalars)));
}

void Context::read2(const KrylovScalars* a, KrylovScalars* ha, const KrylovScalars* b, KrylovScalars* hb) {
  RMG_CK(cudaMemcpyAsync(pinned_sc, a, sizeof(KrylovScalars), cudaMemcpyDeviceToHost, stream));
  RMG_CK(cudaMemcpyAsync(pinned_sc + 1, b, sizeof(KrylovScalars), cudaMemcpyDeviceToHost, stream));
  RMG_CK(cudaStreamSynchronize(stream));
  *ha = pinned_sc[0];
  *hb = pinned_sc[1];
}

Context::~Context() {
  if (pinned_sc) cudaFreeHost(pinned_sc);
  if (capture_stream) cudaStreamDestroy(capture_stream);
  if (own_stream && stream) cudaStreamDestroy(stream);
}

void Context::sync() { RMG_CK(cudaStreamSynchronize(stream)); }

KrylovScalars Context::read(const KrylovScalars* dev) {
  RMG_CK(cudaMemcpyAsync(pinned_sc, dev, sizeof(KrylovScalars), cudaMemcpyDeviceToHost, stream));
  RMG_CK(cudaStreamSynchronize(stream));
  return *pinned_sc;
}

// ------------------------------------------------------------------ sparse upload
namespace {

int lanes_for(double avg) {
  if (avg <= 6.0) return 4;
  if (avg <= 24.0) return 8;
  if (avg <= 96.0) return 16;
  return 32;
}

std::vector<int32_t> narrow(const std::vector<int64_t>& v, const char* what) {
  std::vector<int32_t> o(v.size());
  const size_t T = v.size() < (size_t{1} << 22) ? 1 : std::max(1u, std::min(32u, std::thread::hardware_concurrency()));
  std::vector<char> bad(T, 0);
  auto body = [&](size_t t) {
    for (size_t i = v.size() * t / T; i < v.size() * (t + 1) / T; ++i) {
      if (v[i] < 0 || v[i] > INT32_MAX) {
        bad[t] = 1;
        return;
      }
      o[i] = static_cast<int32_t>(v[i]);
    }
  };
  std::vector<std::thread> pool;
  for (size_t t = 1; t < T; ++t) pool.emplace_back(body, t);
  body(0);
  for (auto& th : pool) th.join();
  for (char b : bad)
    if (b) throw InvalidArgument(std::string(what) + " exceeds the int32 device index range");
  return o;
}

}  // namespace

void DeviceSparse::upload(const HostCsr& h, bool pattern, cudaStream_t s, bool narrow16, bool relabel) {
  const auto p32 = narrow(h.ptr, "row offsets");
  ptr.upload(p32.data(), p32.size(), s);
  // Relabel: label = rank of the column by descending nonzero count (ties by
  // column).  Each row keeps its original element order, so every row sum
  // adds the same terms in the same order as without relabeling.
  std::vector<int32_t> label;
  if (relabel) {
    std::vector<int64_t> cnt(h.f, 0);
    for (int64_t c : h.idx) ++cnt[c];
    std::vector<int32_t> inv(h.f);
    std::iota(inv.begin(), inv.end(), 0);
    std::stable_sort(inv.begin(), inv.end(), [&](int32_t a, int32_t b) { return cnt[a] > cnt[b]; });
    label.resize(h.f);
    for (int64_t j = 0; j < h.f; ++j) label[inv[j]] = static_cast<int32_t>(j);
    col_inv.upload(inv.data(), inv.size(), s);
    vperm.alloc(std::max<int64_t>(1, h.f));
  }
  auto col = [&](size_t k) -> int64_t { return relabel ? label[h.idx[k]] : h.idx[k]; };
  if (narrow16) {  // uint16 column indices (half the index stream)
    std::vector<uint16_t> i16(h.idx.size());
    for (size_t k = 0; k < h.idx.size(); ++k) i16[k] = static_cast<uint16_t>(col(k));
    idx16.upload(i16.data(), i16.size(), s);
  } else {
    std::vector<int32_t> i32(h.idx.size());
    for (size_t k = 0; k < h.idx.size(); ++k) {
      const int64_t c = col(k);
      if (c < 0 || c > INT32_MAX) throw InvalidArgument("column indices exceed the int32 device index range");
      i32[k] = static_cast<int32_t>(c);
    }
    idx.upload(i32.data(), i32.size(), s);
  }
  if (!pattern) val.upload(h.val.data(), h.val.size(), s);
  RMG_CK(cudaStreamSynchronize(s));
  view.rows = h.n;
  view.cols = h.f;
  view.nnz = h.nnz();
  view.ptr = ptr.get();
  view.idx = narrow16 ? nullptr : idx.get();
  view.idx16 = narrow16 ? idx16.get() : nullptr;
  view.val = pattern ? nullptr : val.get();
  view.width = lanes_for(h.n ? static_cast<double>(h.nnz()) / static_cast<double>(h.n) : 1.0);
  view.col_inv = relabel ? col_inv.get() : nullptr;
  view.vperm = relabel ? vperm.get() : nullptr;
}

void DeviceSparse::upload_sell(const HostCsr& h, bool pattern, cudaStream_t s, bool narrow16, bool relabel) {
  const int64_t n = h.n, f = h.f;
  // popularity rank of every column (descending count, ties by column)
  std::vector<int64_t> cnt(f, 0);
  for (int64_t c : h.idx) ++cnt[c];
  std::vector<int32_t> inv(f);
  std::iota(inv.begin(), inv.end(), 0);
  std::stable_sort(inv.begin(), inv.end(), [&](int32_t a, int32_t b) { return cnt[a] > cnt[b]; });
  std::vector<int32_t> rank(f);
  for (int64_t j = 0; j < f; ++j) rank[inv[j]] = static_cast<int32_t>(j);
  // rows: length-descending inside 1024-row windows (32 slices per window)
  constexpr int64_t kWin = 1024;
  std::vector<int32_t> order(n);
  std::iota(order.begin(), order.end(), 0);
  auto len = [&](int64_t r) { return h.ptr[r + 1] - h.ptr[r]; };
  for (int64_t w0 = 0; w0 < n; w0 += kWin)
    std::stable_sort(order.begin() + w0, order.begin() + std::min(n, w0 + kWin),
                     [&](int32_t a, int32_t b) { return len(a) > len(b); });
  const int64_t ns = (n + 31) / 32;
  std::vector<int64_t> off(ns + 1, 0);
  for (int64_t sl = 0; sl < ns; ++sl) off[sl + 1] = off[sl] + 32 * len(order[sl * 32]);
  if (off[ns] > INT32_MAX) throw InvalidArgument("SELL layout exceeds the int32 device index range");
  std::vector<int32_t> srow(ns * 32, -1), slen(ns * 32, 0), i32;
  std::vector<uint16_t> i16;
  std::vector<double> vals;
  if (narrow16)
    i16.assign(off[ns], 0);
  else
    i32.assign(off[ns], 0);
  if (!pattern) vals.assign(off[ns], 0.0);
  const int64_t T = std::max<int64_t>(1, std::min<int64_t>(64, std::thread::hardware_concurrency()));
  std::vector<std::thread> pool;
  for (int64_t t = 0; t < T; ++t) {
    pool.emplace_back([&, t] {
      std::vector<std::pair<int32_t, int64_t>> el;
      for (int64_t sl = t; sl < ns; sl += T) {
        for (int lane = 0; lane < 32; ++lane) {
          const int64_t q = sl * 32 + lane;
          if (q >= n) break;
          const int64_t r = order[q];
          srow[q] = static_cast<int32_t>(r);
          slen[q] = static_cast<int32_t>(len(r));
          el.clear();
          for (int64_t k = h.ptr[r]; k < h.ptr[r + 1]; ++k) el.emplace_back(rank[h.idx[k]], k);
          std::sort(el.begin(), el.end());
          for (size_t j = 0; j < el.size(); ++j) {
            const int64_t d = off[sl] + static_cast<int64_t>(j) * 32 + lane;
            const int64_t c = h.idx[el[j].second];
            const int64_t lab = relabel ? rank[c] : c;
            if (narrow16)
              i16[d] = static_cast<uint16_t>(lab);
            else
              i32[d] = static_cast<int32_t>(lab);
            if (!pattern) vals[d] = h.val[el[j].second];
          }
        }
      }
    });
  }
  for (auto& th : pool) th.join();
  std::vector<int32_t> off32(off.begin(), off.end());
  sell_off.upload(off32.data(), off32.size(), s);
  sell_row.upload(srow.data(), srow.size(), s);
  sell_len.upload(slen.data(), slen.size(), s);
  if (narrow16)
    idx16.upload(i16.data(), i16.size(), s);
  else
    idx.upload(i32.data(), i32.size(), s);
  if (!pattern) val.upload(vals.data(), vals.size(), s);
  if (relabel) {
    col_inv.upload(inv.data(), inv.size(), s);
    vperm.alloc(std::max<int64_t>(1, f));
  }
  RMG_CK(cudaStreamSynchronize(s));
  view = SparseDev{};
  view.rows = n;
  view.cols = f;
  view.nnz = h.nnz();
  view.idx = narrow16 ? nullptr : idx.get();
  view.idx16 = narrow16 ? idx16.get() : nullptr;
  view.val = pattern ? nullptr : val.get();
  view.col_inv = relabel ? col_inv.get() : nullptr;
  view.vperm = relabel ? vperm.get() : nullptr;
  view.sell_off = sell_off.get();
  view.sell_row = sell_row.get();
  view.sell_len = sell_len.get();
  view.n_slices = ns;
}

// Work items over the rows of the X^T CSR,
// by length class: short rows (<= 8 per lane of a W-lane group), medium rows
// (one warp, <= 2048), long rows (fixed CTA segments).  Each CTA item holds
// about C nonzeros, so no lane group owns a row much longer than its peers'.
void DeviceSchedule::build(const HostCsr& xt, cudaStream_t s, int64_t features, const std::vector<char>* skip) {
  const int64_t V = xt.n, nnz = xt.nnz();
  // ~12 items per SM: the first schedule (4 per SM) ran 0.61 waves at 29 % occupancy
  const int64_t C = std::max<int64_t>(512, std::min<int64_t>(16384, nnz / (148 * 12)));
  // lane width from the median row length among rows that are not long
  std::vector<int64_t> lens;
  lens.reserve(V);
  for (int64_t j = 0; j < V; ++j) {
    const int64_t len = xt.ptr[j + 1] - xt.ptr[j];
    if (len > 0 && len <= 2048 && !(skip && (*skip)[j])) lens.push_back(len);
  }
  int width = 8;
  if (!lens.empty()) {
    std::nth_element(lens.begin(), lens.begin() + lens.size() / 2, lens.end());
    width = lanes_for(static_cast<double>(lens[lens.size() / 2]));
  }
  const int64_t short_max = 8LL * width, medium_max = 2048;
  const int64_t seg = std::max<int64_t>(C, 4096);
  std::vector<int32_t> perm_short, perm_medium;
  std::vector<int4> it;
  std::vector<int32_t> lcol, lfirst, lnseg, lslot;
  int slot = 0, segs = 0;
  for (int64_t j = 0; j < V; ++j) {
    if (skip && (*skip)[j]) continue;
    const int64_t len = xt.ptr[j + 1] - xt.ptr[j];
    if (len <= short_max) {
      perm_short.push_back(static_cast<int32_t>(j));
    } else if (len <= medium_max) {
      perm_medium.push_back(static_cast<int32_t>(j));
    } else {
      const int id = static_cast<int>(lcol.size());
      const int nseg = static_cast<int>((len + seg - 1) / seg);
      lcol.push_back(static_cast<int32_t>(j));
      lfirst.push_back(segs);
      lnseg.push_back(nseg);
      lslot.push_back(slot++);
      for (int q = 0; q < nseg; ++q) {
        const int64_t b = xt.ptr[j] + q * seg, e = std::min<int64_t>(xt.ptr[j + 1], b + seg);
        it.push_back(make_int4(id, (int)b, (int)e, segs++));
      }
    }
  }
  std::vector<int32_t> prm(perm_short);
  prm.insert(prm.end(), perm_medium.begin(), perm_medium.end());
  auto pack = [&](int64_t q0, int64_t q1, int kind, int64_t max_rows) {
    int64_t start = q0, acc = 0;
    for (int64_t q = q0; q < q1; ++q) {
      const int64_t len = xt.ptr[prm[q] + 1] - xt.ptr[prm[q]];
      if ((acc + len > C || q - start >= max_rows) && q > start) {
        it.push_back(make_int4((int)start, (int)q, kind, slot++));
        start = q;
        acc = 0;
      }
      acc += std::max<int64_t>(len, 1);
    }
    if (q1 > start) it.push_back(make_int4((int)start, (int)q1, kind, slot++));
  };
  pack(0, static_cast<int64_t>(perm_short.size()), -1, 4096);
  pack(static_cast<int64_t>(perm_short.size()), static_cast<int64_t>(prm.size()), -2, 4096);
  perm.upload(prm.data(), prm.size(), s);
  items.upload(it.data(), it.size(), s);
  long_col.upload(lcol.data(), lcol.size(), s);
  long_first.upload(lfirst.data(), lfirst.size(), s);
  long_nseg.upload(lnseg.data(), lnseg.size(), s);
  long_slot.upload(lslot.data(), lslot.size(), s);
  seg_partial.alloc(std::max(1, segs));
  slots.alloc(std::max(1, slot) * 2);
  col_ticket.alloc(std::max<size_t>(1, lcol.size()));
  grid_ticket.alloc(1);
  RMG_CK(cudaMemsetAsync(col_ticket.get(), 0, col_ticket.size() * sizeof(unsigned), s));
  RMG_CK(cudaMemsetAsync(grid_ticket.get(), 0, sizeof(unsigned), s));
  RMG_CK(cudaStreamSynchronize(s));
  view.items = items.get();
  view.n_items = static_cast<int>(it.size());
  view.long_col = long_col.get();
  view.long_first_seg = long_first.get();
  view.long_nseg = long_nseg.get();
  view.long_slot = long_slot.get();
  view.n_long = static_cast<int>(lcol.size());
  view.n_segs = segs;
  view.n_slots = slot;
  view.seg_partial = seg_partial.get();
  view.col_ticket = col_ticket.get();
  view.slots = slots.get();
  view.grid_ticket = grid_ticket.get();
  view.width = width;
  view.perm = perm.get();
  view.features = features;
}

// ------------------------------------------------------------------ profiling
OpProfile::~OpProfile() {
  for (cudaEvent_t e : pool) cudaEventDestroy(e);
}
void OpProfile::mark(cudaStream_t s) {
  if (used == pool.size()) {
    cudaEvent_t e;
    RMG_CK(cudaEventCreate(&e));
    pool.push_back(e);
  }
  RMG_CK(cudaEventRecord(pool[used++], s));
}
void OpProfile::collect() {
  for (size_t i = 0; i + 3 <= used; i += 3) {
    float a = 0.f, b = 0.f;
    RMG_CK(cudaEventElapsedTime(&a, pool[i], pool[i + 1]));
    RMG_CK(cudaEventElapsedTime(&b, pool[i + 1], pool[i + 2]));
    ms_k1 += a;
    ms_k2 += b;
    ++count;
  }
  used = 0;
}
void OpProfile::reset() {
  used = 0;
  count = 0;
  ms_k1 = ms_k2 = 0.0;
}

// ------------------------------------------------------------------ Matrix
// ------------------------------------------------------------------ multi-GPU
Comm::Comm(int nr, int r, const ncclUniqueId& id, int device) : nranks(nr), rank(r) {
  if (nr < 1 || r < 0 || r >= nr) throw InvalidArgument("rmg_comm_create: rank outside [0, nranks)");
  RMG_CK(cudaSetDevice(device));
  const ncclResult_t e = ncclCommInitRank(&comm, nr, id, r);
  if (e != ncclSuccess) throw CudaError(std::string("ncclCommInitRank: ") + ncclGetErrorString(e));
}

Comm::Comm(int nr, int r, HostAllreduceFn fn, void* user) : nranks(nr), rank(r), host_fn(fn), host_user(user) {
  if (nr < 1 || r < 0 || r >= nr) throw InvalidArgument("rmg_comm_create: rank outside [0, nranks)");
  if (fn == nullptr) throw InvalidArgument("rmg_comm_create_host: null all-reduce function");
}

Comm::~Comm() {
  if (comm) ncclCommDestroy(comm);
  if (pinned) cudaFreeHost(pinned);
}

void Comm::allreduce(const double* send, double* recv, int64_t count, cudaStream_t s) {
  if (count <= 0) return;
  if (host_fn == nullptr) {
    const ncclResult_t e =
        ncclAllReduce(send, recv, static_cast<size_t>(count), ncclDouble, ncclSum, comm, s);
    if (e != ncclSuccess) throw CudaError(std::string("ncclAllReduce: ") + ncclGetErrorString(e));
    return;
  }
  if (pinned_n < static_cast<size_t>(count)) {
    if (pinned) cudaFreeHost(pinned);
    pinned = nullptr;
    RMG_CK(cudaMallocHost(&pinned, static_cast<size_t>(count) * sizeof(double)));
    pinned_n = static_cast<size_t>(count);
  }
  RMG_CK(cudaMemcpyAsync(pinned, send, static_cast<size_t>(count) * sizeof(double), cudaMemcpyDeviceToHost, s));
  RMG_CK(cudaStreamSynchronize(s));
  if (host_fn(host_user, pinned, static_cast<uint64_t>(count)) != 0)
    throw RuntimeError("host all-reduce callback failed");
  RMG_CK(cudaMemcpyAsync(recv, pinned, static_cast<size_t>(count) * sizeof(double), cudaMemcpyHostToDevice, s));
  RMG_CK(cudaStreamSynchronize(s));  // the pinned buffer is reused by the next call
}

std::vector<int64_t> partition_rows(const std::vector<int64_t>& rp, int nranks) {
  if (nranks < 1) throw InvalidArgument("partition_rows: nranks must be positive");
  const int64_t n = static_cast<int64_t>(rp.size()) - 1, nnz = rp.back();
  std::vector<int64_t> b(nranks + 1, n);
  b[0] = 0;
  for (int r = 1; r < nranks; ++r) {  // first row whose start reaches r/nranks of the nonzeros
    const int64_t target = (nnz * r + nranks - 1) / nranks;
    b[r] = std::lower_bound(rp.begin(), rp.end() - 1, target) - rp.begin();
    b[r] = std::max(b[r], b[r - 1]);
  }
  return b;
}

void Matrix::allreduce_sums(double* sendbuf, double* recvbuf, int64_t count) {
  comm->allreduce(sendbuf, recvbuf, count, ctx->stream);
}

// Hybrid X^T pass.  Sample blocks: a multiple of 2 x 148
// blocks of <= kHotBlockMax samples (two 108 KB t-slices per SM).  Hot features:
// >= 4 nonzeros per block on average (the SMEM gathers then amortize the block
// bookkeeping), most popular first, capped so the [block x hot] partials
// (<= 64 MB) stay L2-resident.  Only when the samples span >= 296 blocks of
// >= 4096 (smaller t-vectors are L2/L1-resident and gain nothing).
void Matrix::build_hot(const HostCsr& ht, int64_t n_samples) {
  const char* env = std::getenv("RMG_XT_HOT");
  const bool want = env != nullptr ? std::string(env) == "1" : n_samples >= 296LL * 4096;
  if (!want || n_samples < 296) return;
  const int64_t F = ht.n;
  const int64_t unit = 296;
  const int64_t nblk = unit * ((n_samples + unit * kHotBlockMax - 1) / (unit * kHotBlockMax));
  const int64_t B = (n_samples + nblk - 1) / nblk;
  std::vector<int32_t> order(F);
  std::iota(order.begin(), order.end(), 0);
  auto cnt = [&](int64_t f) { return ht.ptr[f + 1] - ht.ptr[f]; };
  std::stable_sort(order.begin(), order.end(), [&](int32_t a, int32_t b) { return cnt(a) > cnt(b); });
  // [block x hot] partials budget (RMG_HOT_CAP_MB; default 256 MB: at cfg 5 full scale
  // (1184 sample blocks) 96 MB capped the hot set at 10 k features, K2 3256 -> 3078 us)
  const char* capmb = std::getenv("RMG_HOT_CAP_MB");
  const int64_t cap_bytes = (capmb != nullptr ? std::max(1LL, std::atoll(capmb)) : 256LL) << 20;
  const int64_t cap = std::max<int64_t>(0, cap_bytes / (8 * nblk));
  const char* hm = std::getenv("RMG_HOT_MIN");  // hot: >= this many nonzeros per block (mean)
  const int64_t min_per_block = hm != nullptr ? std::max(1, std::atoi(hm)) : 4;
  int64_t H = 0, hA = 0;
  while (H < F && H < cap && cnt(order[H]) >= min_per_block * nblk) ++H;
  while (hA < H && cnt(order[hA]) >= 64 * nblk) ++hA;
  if (H == 0) return;
  auto hx = std::make_unique<HotXt>();
  std::vector<int32_t> feat(order.begin(), order.begin() + H);
  // (block, hot row) counts, prefix, fill -- threads over hot rows
  std::vector<int64_t> rp(static_cast<size_t>(nblk * H + 1), 0);
  const int64_t T = std::max<int64_t>(1, std::min<int64_t>(64, std::thread::hardware_concurrency()));
  auto par = [&](auto fn) {
    std::vector<std::thread> pool;
    for (int64_t t = 0; t < T; ++t) pool.emplace_back([&, t] {
      for (int64_t h = t; h < H; h += T) fn(h);
    });
    for (auto& th : pool) th.join();
  };
  par([&](int64_t h) {
    for (int64_t k = ht.ptr[feat[h]]; k < ht.ptr[feat[h] + 1]; ++k) ++rp[(ht.idx[k] / B) * H + h + 1];
  });
  // Long rows are read 8 entries (16 bytes) per lane: every (block, long row) segment is
  // padded to a multiple of 8 entries and every block to a multiple of 8 (so the segments
  // start 16-byte aligned); padding entries point at the zero slot ts[B] (value 0).
  std::vector<int32_t> real_cnt(static_cast<size_t>(nblk * H));
  for (int64_t b = 0; b < nblk; ++b) {
    int64_t tot = 0;
    for (int64_t h = 0; h < H; ++h) {
      int64_t& c = rp[b * H + h + 1];
      real_cnt[b * H + h] = static_cast<int32_t>(c);
      if (h < hA) c = (c + 7) / 8 * 8;
      tot += c;
    }
    rp[b * H + H] += (8 - tot % 8) % 8;  // the block's last row takes the block's padding
  }
  for (size_t q = 0; q + 1 < rp.size(); ++q) rp[q + 1] += rp[q];
  const int64_t hnnz = rp.back();
  if (hnnz > INT32_MAX || B >= 65535) return;
  std::vector<uint16_t> i16(hnnz, static_cast<uint16_t>(B));
  std::vector<double> v(pattern ? 0 : hnnz, 0.0);
  par([&](int64_t h) {
    int64_t cur_b = -1, pos = 0;
    for (int64_t k = ht.ptr[feat[h]]; k < ht.ptr[feat[h] + 1]; ++k) {  // samples ascending
      const int64_t b = ht.idx[k] / B;
      if (b != cur_b) {
        cur_b = b;
        pos = rp[b * H + h];
      }
      i16[pos] = static_cast<uint16_t>(ht.idx[k] - b * B);
      if (!pattern) v[pos] = ht.val[k];
      ++pos;
    }
  });
  // Long rows (warp per row: lanes read 32 consecutive entries, two half-warp
  // phases of 16 eight-byte SMEM loads): order each (block, row) segment in rounds
  // of one entry per bank pair (sample index mod 16), so a half-warp's 16 gathers of
  // the t-slice hit 16 distinct bank pairs instead of colliding at random.  The sum
  // order changes (still fixed: deterministic).  RMG_HOT_BANKS=0 keeps sample order.
  if (std::getenv("RMG_HOT_BANKS") == nullptr || std::string(std::getenv("RMG_HOT_BANKS")) != "0") {
    par([&](int64_t h) {
      if (h >= hA) return;
      std::vector<uint16_t> bi[16];
      std::vector<double> bv[16];
      for (int64_t b = 0; b < nblk; ++b) {
        const int64_t q0 = rp[b * H + h], q1 = q0 + real_cnt[b * H + h];  // the real entries; padding follows
        for (int k = 0; k < 16; ++k) {
          bi[k].clear();
          bv[k].clear();
        }
        for (int64_t q = q0; q < q1; ++q) {
          bi[i16[q] & 15].push_back(i16[q]);
          if (!pattern) bv[i16[q] & 15].push_back(v[q]);
        }
        size_t pos[16] = {0};
        int64_t q = q0;
        while (q < q1)
          for (int k = 0; k < 16; ++k)
            if (pos[k] < bi[k].size()) {
              i16[q] = bi[k][pos[k]];
              if (!pattern) v[q] = bv[k][pos[k]];
              ++pos[k];
              ++q;
            }
      }
    });
  }
  // lane l of the long-row warp reads entries 8 l .. 8 l + 7 of each 256-entry group: store the
  // group transposed, so that the lanes' u-th entries are consecutive entries of the order above
  par([&](int64_t h) {
    if (h >= hA) return;
    std::vector<uint16_t> ti;
    std::vector<double> tv;
    for (int64_t b = 0; b < nblk; ++b) {
      const int64_t q0 = rp[b * H + h], q1 = rp[b * H + h + 1];
      for (int64_t g0 = q0; g0 < q1; g0 += 256) {
        const int64_t g = std::min<int64_t>(256, q1 - g0), lanes = g / 8;
        ti.assign(i16.begin() + g0, i16.begin() + g0 + g);
        if (!pattern) tv.assign(v.begin() + g0, v.begin() + g0 + g);
        for (int64_t l = 0; l < lanes; ++l)
          for (int64_t u = 0; u < 8; ++u) {
            i16[g0 + 8 * l + u] = ti[u * lanes + l];
            if (!pattern) v[g0 + 8 * l + u] = tv[u * lanes + l];
          }
      }
    }
  });
  std::vector<int32_t> rp32(rp.begin(), rp.end());
  cudaStream_t s = ctx->stream;
  hx->ptr.upload(rp32.data(), rp32.size(), s);
  hx->idx16.upload(i16.data(), i16.size(), s);
  if (!pattern) hx->val.upload(v.data(), v.size(), s);
  hx->feat.upload(feat.data(), feat.size(), s);
  hx->view.S = static_cast<int>(std::min<int64_t>(8, nblk));
  hx->partial.alloc(static_cast<size_t>(nblk * H));
  hx->red2.alloc(static_cast<size_t>(hx->view.S * H));
  std::vector<char> skip(F, 0);
  for (int64_t h = 0; h < H; ++h) skip[feat[h]] = 1;
  hx->cold.build(ht, s, F, &skip);
  // t (N doubles) beyond ~64 MB no longer stays in the L2 between the cold gathers:
  // split the cold rows by sample chunk of 2 M (16 MB of t) -- RMG_XT_CHUNK=0/1 forces
  {
    const char* ce = std::getenv("RMG_XT_CHUNK");
    const bool chunked = ce != nullptr ? std::string(ce) == "1" : n_samples > 8000000;
    if (chunked) {
      const int64_t S = std::getenv("RMG_XT_CHUNK_ROWS") ? std::atoll(std::getenv("RMG_XT_CHUNK_ROWS")) : 2000000;
      const int64_t C = (n_samples + S - 1) / S;
      std::vector<int32_t> cold;
      for (int64_t f = 0; f < F; ++f)
        if (!skip[f] && ht.ptr[f + 1] > ht.ptr[f]) cold.push_back(static_cast<int32_t>(f));
      hx->n_cold = static_cast<int64_t>(cold.size());
      hx->cold_list.upload(cold.data(), cold.size(), s);
      hx->chunk_part.alloc(static_cast<size_t>(C) * std::max<int64_t>(1, F));
      RMG_CK(cudaMemsetAsync(hx->chunk_part.get(), 0, hx->chunk_part.size() * sizeof(double), s));
      hx->chunk_x.resize(C);
      hx->chunk_sched.resize(C);
      for (int64_t c = 0; c < C; ++c) {
        HostCsr cc;  // rows = features (cold only), samples of chunk c, increasing
        cc.n = F;
        cc.f = ht.f;
        cc.ptr.assign(F + 1, 0);
        for (int64_t f = 0; f < F; ++f) {
          int64_t cnt = 0;
          if (!skip[f]) {
            const int64_t* b = ht.idx.data() + ht.ptr[f];
            const int64_t* e = ht.idx.data() + ht.ptr[f + 1];
            cnt = std::lower_bound(b, e, (c + 1) * S) - std::lower_bound(b, e, c * S);
          }
          cc.ptr[f + 1] = cc.ptr[f] + cnt;
        }
        cc.idx.resize(cc.ptr[F]);
        if (!pattern) cc.val.resize(cc.ptr[F]);
        for (int64_t f = 0; f < F; ++f) {
          if (skip[f]) continue;
          const int64_t* b = ht.idx.data() + ht.ptr[f];
          const int64_t* e = ht.idx.data() + ht.ptr[f + 1];
          const int64_t k0 = std::lower_bound(b, e, c * S) - ht.idx.data();
          const int64_t k1 = std::lower_bound(b, e, (c + 1) * S) - ht.idx.data();
          std::copy(ht.idx.begin() + k0, ht.idx.begin() + k1, cc.idx.begin() + cc.ptr[f]);
          if (!pattern) std::copy(ht.val.begin() + k0, ht.val.begin() + k1, cc.val.begin() + cc.ptr[f]);
        }
        hx->chunk_x[c].upload(cc, pattern, s, false);
        std::vector<char> empty(F, 0);
        for (int64_t f = 0; f < F; ++f) empty[f] = cc.ptr[f + 1] == cc.ptr[f] ? 1 : 0;
        hx->chunk_sched[c].build(cc, s, F, &empty);
      }
    }
  }
  // RMG_XT_COLD_NA=1: the cold features' t gathers bypass L1 (measured slower on the
  // cfg 5 shard, 586 vs 555 us: the L1 still catches some reuse)
  hx->cold.view.stream_t = std::getenv("RMG_XT_COLD_NA") != nullptr ? 1 : 0;
  RMG_CK(cudaStreamSynchronize(s));
  HotXtDev& d = hx->view;
  d.ptr = hx->ptr.get();
  d.idx16 = hx->idx16.get();
  d.val = pattern ? nullptr : hx->val.get();
  d.feat = hx->feat.get();
  d.partial = hx->partial.get();
  d.red2 = hx->red2.get();
  d.H = static_cast<int>(H);
  d.hA = static_cast<int>(hA);
  d.nblk = static_cast<int>(nblk);
  d.B = static_cast<int>(B);
  d.N = n_samples;
  hot = std::move(hx);
  if (part.size() == 0) {  // sums + finishing epilogue, as in the sharded pass
    part.alloc(std::max<int64_t>(1, F));
    fin_grid = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(296, (F + 255) / 256)));
    fin_slots.alloc(static_cast<size_t>(fin_grid) * 2);
    fin_ticket.alloc(1);
    RMG_CK(cudaMemsetAsync(fin_ticket.get(), 0, sizeof(unsigned), s));
  }
}

// K1's chunk-interleaved layout (kernels.cuh, BlockK1v2): rows sorted by (hot chunks,
// cold chunks) inside 1024-row windows, slices of 8 rows, entries in label order.
void Matrix::build_k1v2(const HostCsr& xr, const std::vector<int32_t>& rank, int64_t h1) {
  const int64_t n = xr.n;
  if (n == 0 || h1 <= 0 || h1 >= 65535) return;
  const int64_t nslots = (n + 1023) / 1024 * 1024, ns8 = nslots / 8;
  std::vector<int32_t> hch(n), cch(n);
  for (int64_t r = 0; r < n; ++r) {
    int64_t nh = 0;
    for (int64_t q = xr.ptr[r]; q < xr.ptr[r + 1]; ++q) nh += rank[xr.idx[q]] < h1 ? 1 : 0;
    hch[r] = static_cast<int32_t>((nh + 3) / 4);
    cch[r] = static_cast<int32_t>((xr.ptr[r + 1] - xr.ptr[r] - nh + 3) / 4);
  }
  std::vector<int32_t> srow(nslots, -1);
  std::vector<int32_t> order;
  for (int64_t w0 = 0; w0 < n; w0 += 1024) {
    const int64_t w1 = std::min(n, w0 + 1024);
    order.resize(w1 - w0);
    std::iota(order.begin(), order.end(), static_cast<int32_t>(w0));
    std::stable_sort(order.begin(), order.end(), [&](int32_t a, int32_t b) {
      return hch[a] != hch[b] ? hch[a] > hch[b] : cch[a] > cch[b];
    });
    std::copy(order.begin(), order.end(), srow.begin() + w0);
  }
  std::vector<int32_t> off(ns8 + 1, 0), nhot(ns8, 0);
  int64_t run = 0;
  for (int64_t sl = 0; sl < ns8; ++sl) {
    int32_t wh = 0, wc = 0;
    for (int i = 0; i < 8; ++i) {
      const int32_t r = srow[sl * 8 + i];
      if (r < 0) continue;
      wh = std::max(wh, hch[r]);
      wc = std::max(wc, cch[r]);
    }
    off[sl] = static_cast<int32_t>(run);
    nhot[sl] = wh;
    run += wh + wc;
    if (run * 96 > INT32_MAX) return;  // keep the round-2 passes
  }
  off[ns8] = static_cast<int32_t>(run);
  const size_t rec_ints = pattern ? 32 : 96;
  std::vector<int32_t> rec(std::max<size_t>(1, static_cast<size_t>(run) * rec_ints), 0);
  for (int64_t sl = 0; sl < ns8; ++sl)  // padding labels: H1 in hot records, -1 in cold ones
    for (int64_t j = off[sl]; j < off[sl + 1]; ++j)
      std::fill_n(rec.begin() + j * rec_ints, 32, j < off[sl] + nhot[sl] ? static_cast<int32_t>(h1) : -1);
  std::vector<std::pair<int32_t, int64_t>> row;
  for (int64_t sl = 0; sl < ns8; ++sl)
    for (int i = 0; i < 8; ++i) {
      const int32_t r = srow[sl * 8 + i];
      if (r < 0) continue;
      row.clear();
      for (int64_t q = xr.ptr[r]; q < xr.ptr[r + 1]; ++q) row.emplace_back(rank[xr.idx[q]], q);
      std::sort(row.begin(), row.end());  // label order = descending popularity
      int64_t eh = 0, ec = 0;
      for (const auto& pq : row) {
        const bool is_hot = pq.first < h1;
        int64_t& e = is_hot ? eh : ec;
        const size_t j = static_cast<size_t>(off[sl]) + (is_hot ? 0 : nhot[sl]) + e / 4;
        int32_t* rp = rec.data() + j * rec_ints;
        rp[i * 4 + e % 4] = pq.first;
        if (!pattern) std::memcpy(rp + 32 + 2 * (i * 4 + e % 4), &xr.val[pq.second], sizeof(double));
        ++e;
      }
    }
  cudaStream_t s = ctx->stream;
  bk_off.upload(off.data(), off.size(), s);
  bk_nhot.upload(nhot.data(), std::max<size_t>(1, nhot.size()), s);
  bk_srow.upload(srow.data(), srow.size(), s);
  bk_rec.upload(rec.data(), rec.size(), s);
  RMG_CK(cudaStreamSynchronize(s));
  bk1v2.H1 = static_cast<int>(h1);
  bk1v2.n_slices8 = ns8;
  bk1v2.off = bk_off.get();
  bk1v2.nhot = bk_nhot.get();
  bk1v2.srow = bk_srow.get();
  bk1v2.rec = bk_rec.get();
  bk1v2.pattern = pattern;
}

// Hot features of the block X^T pass (kernels.cuh, BlockHot): per sample block the hot
// features' entries, cut into segments of <= 64 (most popular feature first, then
// ascending samples), sorted by length, 8 to a slice, as records; every segment has a
// 16-double partial, and fptr / fidx list each feature's partials in (block, segment)
// order for the fold.
void Matrix::build_block_hot(const HostCsr& ht, const std::vector<int32_t>& feat, int64_t R, int64_t nblk) {
  constexpr int64_t kSeg = 64;
  const int64_t H = static_cast<int64_t>(feat.size());
  const size_t rec_ints = pattern ? 32 : 96;
  std::vector<int64_t> cur(H);  // next entry of each hot feature (the blocks are walked in order)
  for (int64_t h = 0; h < H; ++h) cur[h] = ht.ptr[feat[h]];
  struct Seg { int32_t h; int64_t q0; int32_t len; };
  std::vector<Seg> segs;
  std::vector<int32_t> order;
  std::vector<int32_t> boff(nblk + 1, 0), off(1, 0), rec;
  std::vector<std::vector<int32_t>> flist(H);
  int64_t n_slices = 0, n_rec = 0;
  for (int64_t b = 0; b < nblk; ++b) {
    const int64_t lim = (b + 1) * R;
    segs.clear();
    for (int64_t h = 0; h < H; ++h) {
      const int64_t q0 = cur[h], qe = ht.ptr[feat[h] + 1];
      int64_t q = q0;
      while (q < qe && ht.idx[q] < lim) ++q;
      cur[h] = q;
      for (int64_t a = q0; a < q; a += kSeg)
        segs.push_back(Seg{static_cast<int32_t>(h), a, static_cast<int32_t>(std::min(kSeg, q - a))});
    }
    order.resize(segs.size());
    std::iota(order.begin(), order.end(), 0);
    std::stable_sort(order.begin(), order.end(), [&](int32_t x, int32_t y) { return segs[x].len > segs[y].len; });
    std::vector<int32_t> slot_of(segs.size());
    for (size_t p = 0; p < order.size(); ++p) slot_of[order[p]] = static_cast<int32_t>(n_slices * 8 + p);
    for (size_t sg = 0; sg < segs.size(); ++sg) flist[segs[sg].h].push_back(slot_of[sg]);
    boff[b] = static_cast<int32_t>(n_slices);
    const int64_t bs = (static_cast<int64_t>(segs.size()) + 7) / 8;
    for (int64_t sl = 0; sl < bs; ++sl) {
      const int64_t first = sl * 8;
      const int64_t w = (segs[order[first]].len + 3) / 4;  // sorted: the slice's first segment is its longest
      rec.resize(static_cast<size_t>(n_rec + w) * rec_ints, 0);
      for (int64_t j = 0; j < w; ++j) std::fill_n(rec.begin() + (n_rec + j) * rec_ints, 32, static_cast<int32_t>(R));
      for (int i = 0; i < 8 && first + i < static_cast<int64_t>(segs.size()); ++i) {
        const Seg& sg = segs[order[first + i]];
        for (int32_t e = 0; e < sg.len; ++e) {
          int32_t* rp = rec.data() + static_cast<size_t>(n_rec + e / 4) * rec_ints;
          rp[i * 4 + e % 4] = static_cast<int32_t>(ht.idx[sg.q0 + e] - b * R);
          if (!pattern) std::memcpy(rp + 32 + 2 * (i * 4 + e % 4), &ht.val[sg.q0 + e], sizeof(double));
        }
      }
      n_rec += w;
      if (n_rec * 96 > INT32_MAX) return;  // keep the gather pass for everything
      off.push_back(static_cast<int32_t>(n_rec));
    }
    n_slices += bs;
  }
  boff[nblk] = static_cast<int32_t>(n_slices);
  std::vector<int32_t> fptr(H + 1, 0), fidx;
  for (int64_t h = 0; h < H; ++h) {
    fidx.insert(fidx.end(), flist[h].begin(), flist[h].end());
    fptr[h + 1] = static_cast<int32_t>(fidx.size());
  }
  cudaStream_t s = ctx->stream;
  bh_boff.upload(boff.data(), boff.size(), s);
  bh_off.upload(off.data(), off.size(), s);
  bh_rec.upload(rec.data(), std::max<size_t>(1, rec.size()), s);
  bh_feat.upload(feat.data(), feat.size(), s);
  bh_fptr.upload(fptr.data(), fptr.size(), s);
  bh_fidx.upload(fidx.data(), std::max<size_t>(1, fidx.size()), s);
  bh_part.alloc(std::max<size_t>(1, static_cast<size_t>(n_slices) * 8 * 16));
  RMG_CK(cudaMemsetAsync(bh_part.get(), 0, bh_part.size() * sizeof(double), s));
  RMG_CK(cudaStreamSynchronize(s));
  bhot.H = static_cast<int>(H);
  bhot.R = static_cast<int>(R);
  bhot.nblk = static_cast<int>(nblk);
  bhot.boff = bh_boff.get();
  bhot.off = bh_off.get();
  bhot.rec = bh_rec.get();
  bhot.feat = bh_feat.get();
  bhot.fptr = bh_fptr.get();
  bhot.fidx = bh_fidx.get();
  bhot.part = bh_part.get();
  bhot.pattern = pattern;
}

// Block operator schedule: rows of X^T with <= 512 nonzeros
// are one unit each (a half-warp, elements in order); longer rows are split
// into items of 512 whose partials are finished in item order.
void Matrix::build_block_schedule(const HostCsr& xr, const HostCsr& ht) {
  // A half-warp walks <= kItem elements; longer rows are split into items with a finishing
  // pass.  Measured on cfg 3 (cold rows reach ~1500 entries per chunk): 512 -> 1120 us per apply
  // (the items ran last: a tail), 2048 and above -> 1030 us (no row is split).  RMG_BLOCK_ITEM
  // overrides (diagnostics).
  const int64_t kItem = std::getenv("RMG_BLOCK_ITEM") ? std::max<int64_t>(16, std::atoll(std::getenv("RMG_BLOCK_ITEM"))) : 2048;
  // sample chunks: T's chunk slice (rows x 16 columns x 8 B) <= 64 MB stays in L2
  // between K1 writing and the X^T pass reading it; chunks are whole 1024-row
  // SELL windows (RMG_BLOCK_CHUNK_ROWS overrides the row count)
  const int64_t n = ht.f, F = ht.n;
  int64_t rmax = (int64_t{64} << 20) / (16 * 8);
  if (const char* e = std::getenv("RMG_BLOCK_CHUNK_ROWS")) rmax = std::max<int64_t>(1, std::atoll(e));
  const int64_t nch0 = std::max<int64_t>(1, (n + rmax - 1) / rmax);
  int64_t rows = ((n + nch0 - 1) / nch0 + 1023) / 1024 * 1024;
  rows = std::max<int64_t>(rows, 1024);
  const int nch = static_cast<int>(std::max<int64_t>(1, (n + rows - 1) / rows));
  bchunk_rows = rows;
  // per X^T row j and chunk boundary c: the first entry with sample >= c * rows
  std::vector<int32_t> bounds(static_cast<size_t>(nch + 1) * F);
  for (int64_t j = 0; j < F; ++j) {
    int64_t q = ht.ptr[j];
    for (int c = 0; c <= nch; ++c) {
      const int64_t lim = std::min<int64_t>(n, static_cast<int64_t>(c) * rows);
      while (q < ht.ptr[j + 1] && ht.idx[q] < lim) ++q;
      bounds[static_cast<size_t>(c) * F + j] = static_cast<int32_t>(c == nch ? ht.ptr[j + 1] : q);
    }
  }
  cudaStream_t s = ctx->stream;
  bbounds.upload(bounds.data(), bounds.size(), s);
  const bool tma = tma_spmm_enabled();
  // K1's hot labels: the H1 most popular columns (the relabeled SELL's
  // labels 0 .. H1-1) from shared memory, the rest in a second SELL layout
  bhot1 = BlockHotK1{};
  bk1v2 = BlockK1v2{};
  {
    const char* e1 = std::getenv("RMG_BLOCK_HOTK1");  // rows of V kept in shared memory (0: off)
    const int64_t h1 = std::min<int64_t>(xr.f, e1 != nullptr ? std::max<int64_t>(0, std::atoll(e1)) : 1400);
    const char* e2 = std::getenv("RMG_BLOCK_K1V2");  // "0": the round-2 split K1 (kernels.cu)
    const bool v2 = e2 == nullptr || std::atoi(e2) != 0;
    std::vector<int32_t> rank;
    if (!tma && h1 > 0 && x.view.col_inv != nullptr && h1 <= 1600) {
      std::vector<int64_t> cnt(xr.f, 0);  // the SELL's popularity ranks (same sort as upload_sell)
      for (int64_t c : xr.idx) ++cnt[c];
      std::vector<int32_t> inv(xr.f);
      rank.resize(xr.f);
      std::iota(inv.begin(), inv.end(), 0);
      std::stable_sort(inv.begin(), inv.end(), [&](int32_t a, int32_t b) { return cnt[a] > cnt[b]; });
      for (int64_t j = 0; j < xr.f; ++j) rank[inv[j]] = static_cast<int32_t>(j);
      if (v2) build_k1v2(xr, rank, h1);
    }
    if (!rank.empty() && bk1v2.H1 == 0) {
      std::vector<int32_t> hptr(xr.n + 1, 0);
      std::vector<uint16_t> hlab;
      std::vector<double> hval;
      HostCsr cold;
      cold.n = xr.n;
      cold.f = xr.f;
      cold.ptr.assign(xr.n + 1, 0);
      std::vector<std::pair<int32_t, int64_t>> row;
      for (int64_t r = 0; r < xr.n; ++r) {
        row.clear();
        for (int64_t q = xr.ptr[r]; q < xr.ptr[r + 1]; ++q) {
          if (rank[xr.idx[q]] < h1) {
            row.emplace_back(rank[xr.idx[q]], q);
          } else {
            cold.idx.push_back(xr.idx[q]);
            cold.val.push_back(xr.val.empty() ? 1.0 : xr.val[q]);
          }
        }
        std::sort(row.begin(), row.end());  // popularity order, as the SELL rows
        for (const auto& pq : row) {
          hlab.push_back(static_cast<uint16_t>(pq.first));
          if (!pattern) hval.push_back(xr.val[pq.second]);
        }
        hptr[r + 1] = static_cast<int32_t>(hlab.size());
        cold.ptr[r + 1] = static_cast<int64_t>(cold.idx.size());
      }
      if (hlab.size() < static_cast<size_t>(INT32_MAX)) {
        bh1_ptr.upload(hptr.data(), hptr.size(), s);
        bh1_lab.upload(hlab.data(), hlab.size(), s);
        if (!pattern) bh1_val.upload(hval.data(), hval.size(), s);
        bh1_cold.upload_sell(cold, pattern, s, cold.f <= 65536, false);
        RMG_CK(cudaStreamSynchronize(s));
        bhot1.H1 = static_cast<int>(h1);
        bhot1.ptr = bh1_ptr.get();
        bhot1.lab = bh1_lab.get();
        bhot1.val = pattern ? nullptr : bh1_val.get();
        bhot1.cold = bh1_cold.view;
      }
    }
  }
  // hot features: >= hot_min entries per sample block of R rows on
  // average, most popular first; they leave the chunked gather pass
  std::vector<char> is_hot(F, 0);
  bhot = BlockHot{};
  {
    const char* e = std::getenv("RMG_BLOCK_HOTXT");  // "0": off; a number: the per-block minimum
    const double hot_min = e != nullptr ? std::atof(e) : 4.0;  // measured: 4 (2.11 ms) < 8 < 2 < off (2.27 ms)
    // rows per sample block: <= 1536 (192 KB of T rows in shared memory), chosen so that
    // the blocks fill whole waves of one CTA per SM
    int sms = 148;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, ctx->device);
    const int64_t waves = std::max<int64_t>(1, ((n + 1535) / 1536 + sms - 1) / sms);
    int64_t R = ((n + sms * waves - 1) / (sms * waves) + 7) / 8 * 8;
    R = std::min<int64_t>(1536, std::max<int64_t>(512, R));
    if (const char* er = std::getenv("RMG_BLOCK_HOTXT_ROWS")) R = std::min<int64_t>(1536, std::max<int64_t>(8, std::atoll(er)));
    const int64_t nblk = (n + R - 1) / R;
    std::vector<int32_t> feat;
    if (!tma && hot_min > 0.0 && nblk >= 2) {
      std::vector<int64_t> order(F);
      std::iota(order.begin(), order.end(), int64_t{0});
      auto cnt = [&](int64_t j) { return ht.ptr[j + 1] - ht.ptr[j]; };
      std::stable_sort(order.begin(), order.end(), [&](int64_t a, int64_t b) { return cnt(a) > cnt(b); });
      for (int64_t j : order) {
        if (static_cast<double>(cnt(j)) < hot_min * static_cast<double>(nblk) || feat.size() >= 4096) break;
        feat.push_back(static_cast<int32_t>(j));
      }
    }
    const int64_t H = static_cast<int64_t>(feat.size());
    if (H > 0) build_block_hot(ht, feat, R, nblk);
    if (bhot.H > 0)
      for (int32_t j : feat) is_hot[j] = 1;
  }
  if (tma) {  // X's row CSR for the TMA K1 (column order: the reference's summation order per row)
    const std::vector<int32_t> i32 = narrow(xr.idx, "column indices");
    bx_idx.upload(i32.data(), i32.size(), s);
    if (!pattern) bx_val.upload(xr.val.data(), xr.val.size(), s);
    RMG_CK(cudaStreamSynchronize(s));
  }
  bchunk_bufs.clear();
  bchunk_bufs.resize(nch);
  bviews.assign(nch, BlockXtSchedule{});
  int max_segs = 1;
  for (int c = 0; c < nch; ++c) {
    std::vector<int32_t> sh;
    std::vector<int4> it, mu;
    int segs = 0;
    for (int64_t r = 0; r < F; ++r) {
      if (is_hot[r]) continue;  // summed by the hot pass
      const int64_t a = bounds[static_cast<size_t>(c) * F + r], e = bounds[static_cast<size_t>(c + 1) * F + r];
      if (e - a <= kItem) {
        sh.push_back(static_cast<int32_t>(r));
      } else {
        const int first = segs;
        for (int64_t b = a; b < e; b += kItem)
          it.push_back(make_int4(static_cast<int>(r), static_cast<int>(b), static_cast<int>(std::min(e, b + kItem)),
                                 segs++));
        mu.push_back(make_int4(static_cast<int>(r), first, segs - first, 0));
      }
    }
    max_segs = std::max(max_segs, segs);
    // longest first: the two half-warps of a warp get rows of similar length
    std::stable_sort(sh.begin(), sh.end(), [&](int32_t a, int32_t b) {
      const size_t oa = static_cast<size_t>(c) * F, ob = static_cast<size_t>(c + 1) * F;
      return bounds[ob + a] - bounds[oa + a] > bounds[ob + b] - bounds[oa + b];
    });
    BlockChunkBufs& cb = bchunk_bufs[c];
    cb.sh.upload(sh.data(), sh.size(), s);
    cb.it.upload(it.data(), it.size(), s);
    cb.mu.upload(mu.data(), mu.size(), s);
    const int64_t r0 = static_cast<int64_t>(c) * rows, r1 = std::min(n, r0 + rows);
    std::vector<int4> u1, u2;  // TMA units: longest first (round-robin warps stay balanced)
    for (int64_t r = tma ? r0 : r1; r < r1; ++r)
      u1.push_back(make_int4(static_cast<int>(r), static_cast<int>(xr.ptr[r]), static_cast<int>(xr.ptr[r + 1]), -1));
    std::stable_sort(u1.begin(), u1.end(), [](const int4& a, const int4& b) { return a.z - a.y > b.z - b.y; });
    for (int32_t r : sh) {
      if (!tma) break;
      u2.push_back(make_int4(r, bounds[static_cast<size_t>(c) * F + r], bounds[static_cast<size_t>(c + 1) * F + r], -1));
    }
    std::vector<int4> itl(tma ? it : std::vector<int4>{});
    std::stable_sort(itl.begin(), itl.end(), [](const int4& a, const int4& b) { return a.z - a.y > b.z - b.y; });
    u2.insert(u2.begin(), itl.begin(), itl.end());
    cb.u1.upload(u1.data(), u1.size(), s);
    cb.u2.upload(u2.data(), u2.size(), s);
    BlockXtSchedule& v = bviews[c];
    v.short_rows = cb.sh.get();
    v.n_short = static_cast<int>(sh.size());
    v.items = cb.it.get();
    v.n_items = static_cast<int>(it.size());
    v.multi = cb.mu.get();
    v.n_multi = static_cast<int>(mu.size());
    v.e_begin = bbounds.get() + static_cast<size_t>(c) * F;
    v.e_end = bbounds.get() + static_cast<size_t>(c + 1) * F;
    if (tma) {
      v.tk1 = TmaSpmm{cb.u1.get(), static_cast<int>(u1.size()), bx_idx.get(), pattern ? nullptr : bx_val.get()};
      v.tk2 = TmaSpmm{cb.u2.get(), static_cast<int>(u2.size()), xt.view.idx, pattern ? nullptr : xt.view.val};
    }
    v.slice0 = r0 / 32;
    v.n_slices = (r1 + 31) / 32 - r0 / 32;
    RMG_CK(cudaStreamSynchronize(s));  // host vectors above go out of scope
  }
  bseg.alloc(static_cast<size_t>(max_segs) * 16);
  for (auto& v : bviews) v.seg = bseg.get();
}

// Dense X, k right-hand sides: the operator is the dense contraction
// (X^T X) V + beta V.  G = X^T X (F <= 1024: <= 8 MB, beta-free, kept for the matrix's
// lifetime, so a beta sweep and every later block apply reuse it) is formed once on the
// FP64 tensor cores (syrk_dense_dmma), and each apply is one DMMA skinny GEMM.
void Matrix::ensure_block_gram() {
  if (bgram.size() > 0) return;
  const int64_t nf = f();
  bgram_ld = (nf + 1) / 2 * 2;
  bgram.alloc(static_cast<size_t>(std::max<int64_t>(1, nf)) * bgram_ld);
  bgram_scratch.alloc(static_cast<size_t>(std::max<int64_t>(1, gram_gemm_scratch(nf))));
  RMG_CK(cudaMemsetAsync(bgram.get(), 0, bgram.size() * sizeof(double), ctx->stream));
  const DenseDev& d = dense->view;
  syrk_dense_dmma(ctx->stream, d.data, d.fp32, d.ld, d.rows, d.cols, bgram.get(), bgram_ld);
}

// First block call on a CSR matrix: build the block layouts from the host CSR.  Not
// inside a graph capture (it allocates and synchronizes): solve_block calls it first.
void Matrix::ensure_block_schedule() {
  if (block_built || dense) return;
  if (comm != nullptr) throw InvalidArgument("block operator: single-GPU matrices only");
  ensure_operator();  // the block layouts follow the K1 layout's column relabeling
  const HostCsr ht = transpose(host);
  build_block_schedule(host, ht);
  block_built = true;
}

void Matrix::apply_block(const double* v, double* out, double beta, int k, bool sync) {
  if (comm != nullptr) throw InvalidArgument("block operator: single-GPU matrices only");
  if (k <= 0 || k > 64) throw InvalidArgument("block operator: k must be in [1, 64]");
  if (beta < 0.0) throw InvalidArgument("RidgeOperator: beta must be nonnegative");
  if (dense) {
    ensure_block_gram();
    launch_gram_gemm(bgram.get(), bgram_ld, v, beta, out, f(), k, bgram_scratch.get(), ctx->stream);
    if (sync) ctx->sync();
    return;
  }
  ensure_block_schedule();
  const size_t nt = static_cast<size_t>(std::max<int64_t>(1, n())) * k, nv = static_cast<size_t>(std::max<int64_t>(1, f())) * k;
  if (bt.size() < nt) bt.alloc(nt);
  if (x.view.col_inv != nullptr && bvp.size() < nv) bvp.alloc(nv);
  launch_ridge_block(x.view, xt.view, bviews.data(), static_cast<int>(bviews.size()), bhot, bhot1, bk1v2, v, out, beta, k,
                     bt.get(),
                     bvp.get(), ctx->stream);
  if (sync) ctx->sync();
}

void Matrix::xt_block_cm(const double* b_cm, double* out, int k) {
  if (comm != nullptr) throw InvalidArgument("block operator: single-GPU matrices only");
  if (k <= 0 || k > 64) throw InvalidArgument("block operator: k must be in [1, 64]");
  const size_t nt = static_cast<size_t>(std::max<int64_t>(1, n())) * k;
  if (dense) {  // X^T B in one sweep of X per 16 columns, on the FP64 tensor cores
    const DenseDev& d = dense->view;
    const size_t need = static_cast<size_t>(std::max<int64_t>(1, xtb_scratch(d.rows, d.cols)));
    if (bt.size() < need) bt.alloc(need);
    launch_xtb_dmma(ctx->stream, d.data, d.fp32, d.ld, d.rows, d.cols, b_cm, k, out, bt.get());
    return;
  }
  ensure_block_schedule();
  if (bt.size() < nt) bt.alloc(nt);
  launch_bcol2row(b_cm, bt.get(), n(), k, ctx->stream);
  launch_ridge_block(x.view, xt.view, bviews.data(), static_cast<int>(bviews.size()), bhot, bhot1, bk1v2, nullptr, out,
                     0.0, k, bt.get(), nullptr, ctx->stream, true);
}

// Dense X kept on the device: rows padded to ld = F rounded up to 4 elements
// (16 B aligned rows), the fused single-sweep operator's scratch.
void Matrix::init_dense(DBuf<char>&& data, int fp32, int64_t ld, int64_t rows) {
  if (host.f > kDenseMaxCols) throw InvalidArgument("dense X: more than 1024 features (use CSR)");
  pattern = false;
  auto d = std::make_unique<DenseStore>();
  d->data = std::move(data);
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, ctx->device);
  d->view.n_cta = sms;
  d->partial.alloc(static_cast<size_t>(std::max<int64_t>(1, host.f)) * sms);
  d->view.fin_grid = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(sms, (host.f + 7) / 8)));
  d->fin_slots.alloc(static_cast<size_t>(d->view.fin_grid) * 2);
  d->fin_ticket.alloc(1);
  RMG_CK(cudaMemsetAsync(d->fin_ticket.get(), 0, sizeof(unsigned), ctx->stream));
  RMG_CK(cudaStreamSynchronize(ctx->stream));
  d->view.data = d->data.get();
  d->view.fp32 = fp32;
  d->view.ld = ld;
  d->view.rows = rows;
  d->view.cols = host.f;
  d->view.partial = d->partial.get();
  d->view.fin_slots = d->fin_slots.get();
  d->view.fin_ticket = d->fin_ticket.get();
  dense = std::move(d);
  t.alloc(std::max<int64_t>(1, rows));
  gram_sc.alloc(1);
}

void Matrix::init_dense_from_host(const void* data, int fp32, int64_t ld_in, int64_t rows) {
  if (host.f > kDenseMaxCols) throw InvalidArgument("dense X: more than 1024 features (use CSR)");
  const size_t esz = fp32 ? 4 : 8;
  const int64_t ld = (host.f + 3) / 4 * 4;
  DBuf<char> dev(std::max<size_t>(1, static_cast<size_t>(rows) * ld * esz));
  // staged through a pinned buffer in row blocks (16 B aligned padded rows)
  const int64_t block = std::max<int64_t>(1, (64ll << 20) / std::max<int64_t>(1, ld * esz));
  char* stage = nullptr;
  RMG_CK(cudaMallocHost(&stage, static_cast<size_t>(std::min(block, std::max<int64_t>(rows, 1))) * ld * esz));
  try {
    for (int64_t r0 = 0; r0 < rows; r0 += block) {
      const int64_t nr = std::min(block, rows - r0);
      RMG_CK(cudaStreamSynchronize(ctx->stream));  // the staging buffer is free again
      std::memset(stage, 0, static_cast<size_t>(nr) * ld * esz);
      for (int64_t i = 0; i < nr; ++i)
        std::memcpy(stage + static_cast<size_t>(i) * ld * esz,
                    static_cast<const char*>(data) + static_cast<size_t>(r0 + i) * ld_in * esz,
                    static_cast<size_t>(host.f) * esz);
      RMG_CK(cudaMemcpyAsync(dev.get() + static_cast<size_t>(r0) * ld * esz, stage, static_cast<size_t>(nr) * ld * esz,
                             cudaMemcpyHostToDevice, ctx->stream));
    }
    RMG_CK(cudaStreamSynchronize(ctx->stream));
  } catch (...) {
    cudaFreeHost(stage);
    throw;
  }
  cudaFreeHost(stage);
  init_dense(std::move(dev), fp32, ld, rows);
}

// Dense X without a host CSR: setup runs on the device.
Matrix::Matrix(Context* c, int64_t n, int64_t f, const DenseInput& din) : ctx(c) {
  host.n = n;
  host.f = f;
  host_ok = false;
  if (din.ld < f) throw InvalidArgument("dense X: leading dimension below the feature count");
  RMG_CK(cudaSetDevice(ctx->device));
  row0 = 0;
  row1 = n;
  init_dense_from_host(din.data, din.fp32, din.ld, n);
}

Matrix::Matrix(Context* c, int64_t n, int64_t f, DBuf<char>&& data, int fp32, int64_t ld) : ctx(c) {
  host.n = n;
  host.f = f;
  host_ok = false;
  RMG_CK(cudaSetDevice(ctx->device));
  row0 = 0;
  row1 = n;
  init_dense(std::move(data), fp32, ld, n);
}

Matrix::Matrix(Context* c, int64_t n_glob, int64_t r0, int64_t n_local, int64_t f, const DenseInput& din, Comm* cm)
    : ctx(c), comm(cm) {
  if (comm == nullptr) throw InvalidArgument("rmg_matrix_create_dense_rows: needs a communicator");
  if (r0 < 0 || n_local < 0 || r0 + n_local > n_glob)
    throw InvalidArgument("rmg_matrix_create_dense_rows: rows [row0, row0 + n_local) outside [0, n_samples)");
  if (din.ld < f) throw InvalidArgument("dense X: leading dimension below the feature count");
  host.n = n_local;
  host.f = f;
  host_ok = false;
  n_global = n_glob;
  rows_only = true;
  row0 = r0;
  row1 = r0 + n_local;
  RMG_CK(cudaSetDevice(ctx->device));
  alloc_comm_buffers();
  init_dense_from_host(din.data, din.fp32, din.ld, n_local);
}

Matrix::Matrix(Context* c, int64_t n_glob, int64_t r0, int64_t n_local, int64_t f, DBuf<char>&& data, int fp32,
               int64_t ld, Comm* cm)
    : ctx(c), comm(cm) {
  host.n = n_local;
  host.f = f;
  host_ok = false;
  n_global = n_glob;
  rows_only = true;
  row0 = r0;
  row1 = r0 + n_local;
  RMG_CK(cudaSetDevice(ctx->device));
  alloc_comm_buffers();
  init_dense(std::move(data), fp32, ld, n_local);
}

// The canonical CSR of a device-resident dense X (exact zeros not stored, as
// dense_to_csr), built on first use by host-only setup (leader-follower).
const HostCsr& Matrix::host_csr() {
  if (host_ok) return host;
  const DenseDev& v = dense->view;
  const size_t esz = v.fp32 ? 4 : 8;
  std::vector<char> buf(static_cast<size_t>(v.rows) * v.ld * esz);
  if (!buf.empty())
    RMG_CK(cudaMemcpyAsync(buf.data(), v.data, buf.size(), cudaMemcpyDeviceToHost, ctx->stream));
  RMG_CK(cudaStreamSynchronize(ctx->stream));
  HostCsr h;
  h.n = v.rows;
  h.f = v.cols;
  h.ptr.assign(h.n + 1, 0);
  for (int64_t i = 0; i < h.n; ++i) {
    for (int64_t j = 0; j < h.f; ++j) {
      const double x = v.fp32 ? static_cast<double>(reinterpret_cast<const float*>(buf.data())[i * v.ld + j])
                              : reinterpret_cast<const double*>(buf.data())[i * v.ld + j];
      if (x != 0.0) {
        h.idx.push_back(j);
        h.val.push_back(x);
      }
    }
    h.ptr[i + 1] = h.nnz();
  }
  host = std::move(h);
  host_ok = true;
  return host;
}

Matrix::Matrix(Context* c, HostCsr h, bool detect_pattern, Comm* cm, const DenseInput* din, bool defer_operator)
    : ctx(c), host(std::move(h)), comm(cm) {
  defer_op = defer_operator && cm == nullptr && din == nullptr;  // the deferred build reads `host` = the local rows
  const auto tv = std::chrono::steady_clock::now();
  validate_csr(host);
  pattern = host.val.empty();
  if (!pattern && detect_pattern)
    pattern = std::all_of(host.val.begin(), host.val.end(), [](double v) { return v == 1.0; });
  if (host.val.empty()) host.val.assign(host.nnz(), 1.0);
  if (std::getenv("RMG_SETUP_LOG") != nullptr && host.nnz() > (1 << 24))
    std::fprintf(stderr, "[rmg setup]   upload %-10s %8.3f s\n", "validate",
                 std::chrono::duration<double>(std::chrono::steady_clock::now() - tv).count());
  RMG_CK(cudaSetDevice(ctx->device));
  row0 = 0;
  row1 = host.n;
  HostCsr shard;
  if (comm != nullptr) {  // this rank's nnz-balanced row block (rows rebased to 0)
    const std::vector<int64_t> b = partition_rows(host.ptr, comm->nranks);
    row0 = b[comm->rank];
    row1 = b[comm->rank + 1];
    shard.n = row1 - row0;
    shard.f = host.f;
    shard.ptr.resize(shard.n + 1);
    for (int64_t i = 0; i <= shard.n; ++i) shard.ptr[i] = host.ptr[row0 + i] - host.ptr[row0];
    shard.idx.assign(host.idx.begin() + host.ptr[row0], host.idx.begin() + host.ptr[row1]);
    shard.val.assign(host.val.begin() + host.ptr[row0], host.val.begin() + host.ptr[row1]);
  }
  const HostCsr& local = comm != nullptr ? shard : host;
  if (din != nullptr) {  // dense X: one row-major device copy, fused single-sweep operator
    if (din->ld < host.f) throw InvalidArgument("dense X: leading dimension below the feature count");
    if (comm != nullptr) alloc_comm_buffers();
    const char* src = static_cast<const char*>(din->data) + static_cast<size_t>(row0) * din->ld * (din->fp32 ? 4 : 8);
    init_dense_from_host(src, din->fp32, din->ld, local.n);
    return;
  }
  init_sparse(local);
}

Matrix::Matrix(Context* c, HostCsr local, int64_t n_glob, int64_t r0, bool detect_pattern, Comm* cm,
               bool defer_operator)
    : ctx(c), host(std::move(local)), comm(cm) {
  defer_op = defer_operator;
  validate_csr(host);
  if (comm == nullptr) throw InvalidArgument("rmg_matrix_create_csr_rows: needs a communicator");
  if (r0 < 0 || n_glob < 0 || r0 + host.n > n_glob)
    throw InvalidArgument("rmg_matrix_create_csr_rows: rows [row0, row0 + n_local) outside [0, n_samples)");
  n_global = n_glob;
  rows_only = true;
  row0 = r0;
  row1 = r0 + host.n;
  pattern = host.val.empty();
  if (!pattern && detect_pattern)
    pattern = std::all_of(host.val.begin(), host.val.end(), [](double v) { return v == 1.0; });
  if (host.val.empty()) host.val.assign(host.nnz(), 1.0);
  RMG_CK(cudaSetDevice(ctx->device));
  init_sparse(host);
}

void Matrix::alloc_comm_buffers() {
  part.alloc(std::max<int64_t>(1, host.f));
  red.alloc(std::max<int64_t>(1, std::max(host.f, n())));
  fin_grid = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(296, (host.f + 255) / 256)));
  fin_slots.alloc(static_cast<size_t>(fin_grid) * 2);
  fin_ticket.alloc(1);
  RMG_CK(cudaMemsetAsync(fin_ticket.get(), 0, sizeof(unsigned), ctx->stream));
}

// the device copies of this rank's rows (the whole matrix when unsharded)
void Matrix::init_sparse(const HostCsr& local) {
  // the device index range is int32: checked on the rows this device holds
  if (local.n > INT32_MAX || local.f > INT32_MAX || local.nnz() > INT32_MAX)
    throw InvalidArgument("FeatureMatrix: dimensions exceed the single-device int32 index range");
  if (comm != nullptr) alloc_comm_buffers();
  // Column relabeling pays once v (F doubles) outgrows L1 (measured on the
  // cfg 5 shard, profiles/r1_operator.md); RMG_RELABEL=0/1 overrides.
  const bool slog = std::getenv("RMG_SETUP_LOG") != nullptr && local.nnz() > (1 << 24);
  auto tp = std::chrono::steady_clock::now();
  auto lap = [&](const char* what) {  // RMG_SETUP_LOG: where a large level's upload goes
    if (!slog) return;
    RMG_CK(cudaStreamSynchronize(ctx->stream));
    const auto now = std::chrono::steady_clock::now();
    std::fprintf(stderr, "[rmg setup]   upload %-10s %8.3f s\n", what, std::chrono::duration<double>(now - tp).count());
    tp = now;
  };
  if (!defer_op) {
    upload_k1(local);
    lap("K1 layout");
  }
  const HostCsr ht = transpose(local);
  lap("transpose");
  xt.upload(ht, pattern, ctx->stream, false);
  lap("X^T copy");
  sched.build(ht, ctx->stream, local.f);
  lap("X^T sched");
  if (!defer_op) {
    build_hot(ht, local.n);
    lap("hot blocks");
  }
  op_ready = !defer_op;
  // the block operator's layouts (K1 records, hot X^T blocks, chunk schedules) are built
  // on the first block call (ensure_block_schedule): most matrices never see one
  t.alloc(std::max<int64_t>(1, local.n));
  gram_sc.alloc(1);
}

void Matrix::upload_k1(const HostCsr& local) {
  // Column relabeling pays once v (F doubles) outgrows L1 (measured on the
  // cfg 5 shard, profiles/r1_operator.md); RMG_RELABEL=0/1 overrides.
  const char* rl = std::getenv("RMG_RELABEL");
  const bool relabel = rl != nullptr ? std::string(rl) == "1" : local.f * 8 > 192 * 1024;
  const char* k1 = std::getenv("RMG_K1");  // "csr": the row-CSR K1 (diagnostics)
  if (k1 != nullptr && std::string(k1) == "csr")
    x.upload(local, pattern, ctx->stream, local.f <= 65536, relabel);
  else
    x.upload_sell(local, pattern, ctx->stream, local.f <= 65536, relabel);
}

// the layouts a deferred level skipped at construction (K1, hot X^T blocks), on its first application
void Matrix::ensure_operator() {
  if (op_ready) return;
  cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
  RMG_CK(cudaStreamIsCapturing(ctx->stream, &cap));
  if (cap != cudaStreamCaptureStatusNone)
    throw RuntimeError("Matrix::ensure_operator: a deferred level was first applied inside a graph capture");
  upload_k1(host);
  build_hot(transpose(host), host.n);
  op_ready = true;
}

namespace {
// X^T pass of one operator application: fused epilogue, or (sharded) partial
// sums + all-reduce of the F-vector + epilogue pass.
void xt_pass(Matrix& m, const double* t, Epi epi, const XtArgs& args) {
  XtArgs a = args;
  a.t = t;
  if (m.comm == nullptr && !m.hot) {
    launch_xt(m.xt.view, m.sched.view, epi, a, m.ctx->stream);
    return;
  }
  XtArgs pa = a;
  pa.out = m.part.get();
  if (m.hot) {  // hybrid: cold rows (segmented) + hot rows (sample-blocked), sums only
    static const bool serial = std::getenv("RMG_XT_SERIAL") != nullptr;
    HotXt& h = *m.hot;
    cudaStream_t cs = m.ctx->stream;
    if (!serial && h.side == nullptr) {
      RMG_CK(cudaStreamCreateWithFlags(&h.side, cudaStreamNonBlocking));
      RMG_CK(cudaEventCreateWithFlags(&h.fork, cudaEventDisableTiming));
      RMG_CK(cudaEventCreateWithFlags(&h.join, cudaEventDisableTiming));
    }
    if (!serial) {  // fork: the cold pass on the side stream
      RMG_CK(cudaEventRecord(h.fork, m.ctx->stream));
      RMG_CK(cudaStreamWaitEvent(h.side, h.fork, 0));
      cs = h.side;
    }
    if (h.chunk_x.empty()) {
      launch_xt(m.xt.view, h.cold.view, Epi::Plain, pa, cs);
    } else {  // sample-chunked cold pass: partials per chunk, combined in chunk order
      const int64_t F = m.f();
      for (size_t c = 0; c < h.chunk_x.size(); ++c) {
        XtArgs ca = pa;
        ca.out = h.chunk_part.get() + c * F;
        launch_xt(h.chunk_x[c].view, h.chunk_sched[c].view, Epi::Plain, ca, cs);
      }
      const KrylovScalars* csc = (epi == Epi::Fcg || epi == Epi::Cg) ? a.sc : nullptr;
      launch_chunk_combine(h.chunk_part.get(), static_cast<int>(h.chunk_x.size()), F, h.cold_list.get(), h.n_cold,
                           m.part.get(), a.done, csc, cs);
    }
    const KrylovScalars* sc = (epi == Epi::Fcg || epi == Epi::Cg) ? a.sc : nullptr;
    launch_xt_hot(h.view, t, a.done, sc, m.part.get(), m.ctx->stream);
    if (!serial) {  // join before the epilogue reads both parts
      RMG_CK(cudaEventRecord(h.join, h.side));
      RMG_CK(cudaStreamWaitEvent(m.ctx->stream, h.join, 0));
    }
    m.ctx->launches += 3;
  } else {
    launch_xt(m.xt.view, m.sched.view, Epi::Plain, pa, m.ctx->stream);
  }
  const double* sums = m.part.get();
  if (m.comm != nullptr) {
    m.allreduce_sums(m.part.get(), m.red.get(), m.f());
    sums = m.red.get();
  }
  launch_xt_epilogue(sums, m.f(), epi, a, m.fin_slots.get(), m.fin_ticket.get(), m.fin_grid, m.ctx->stream);
  m.ctx->launches += 1;
}
}  // namespace

// Dense X: fused X^T (X v) sweep; sharded: plain sums, all-reduce, epilogue.
static void dense_apply(Matrix& m, const double* v, int stride, const KrylovScalars* sc, Epi epi,
                        const XtArgs& args) {
  if (m.comm == nullptr) {
    launch_dense_ata(m.dense->view, v, stride, sc, epi, args, m.ctx->stream);
  } else {
    XtArgs pa = args;
    pa.out = m.part.get();
    launch_dense_ata(m.dense->view, v, stride, sc, Epi::Plain, pa, m.ctx->stream);
    m.allreduce_sums(m.part.get(), m.red.get(), m.f());
    launch_xt_epilogue(m.red.get(), m.f(), epi, args, m.fin_slots.get(), m.fin_ticket.get(), m.fin_grid,
                       m.ctx->stream);
  }
  m.ctx->launches += 2;
}

void Matrix::apply(const double* v, Epi epi, const XtArgs& args, OpProfile* prof) {
  if (dense) {
    if (prof) prof->mark(ctx->stream);
    dense_apply(*this, v, 0, nullptr, epi, args);
    if (prof) {
      prof->mark(ctx->stream);
      prof->mark(ctx->stream);
    }
    return;
  }
  ensure_operator();
  if (prof) prof->mark(ctx->stream);
  launch_spmv_rows(x.view, v, t.get(), args.done, ctx->stream);
  if (prof) prof->mark(ctx->stream);
  xt_pass(*this, t.get(), epi, args);
  if (prof) prof->mark(ctx->stream);
  ctx->launches += 2;
}

void Matrix::apply_ring(const double* v_ring, int stride, const KrylovScalars* sc, Epi epi, const XtArgs& args,
                        OpProfile* prof) {
  if (dense) {
    if (prof) prof->mark(ctx->stream);
    dense_apply(*this, v_ring, stride, sc, epi, args);
    if (prof) {
      prof->mark(ctx->stream);
      prof->mark(ctx->stream);
    }
    return;
  }
  ensure_operator();
  if (prof) prof->mark(ctx->stream);
  launch_spmv_rows_ring(x.view, v_ring, stride, sc, t.get(), ctx->stream);
  if (prof) prof->mark(ctx->stream);
  xt_pass(*this, t.get(), epi, args);
  if (prof) prof->mark(ctx->stream);
  ctx->launches += 2;
}

void Matrix::spmv(const double* v, double* y) {
  if (!dense) ensure_operator();
  auto rows = [&](double* yy) {
    if (dense)
      launch_dense_spmv(dense->view, v, yy, ctx->stream);
    else
      launch_spmv_rows(x.view, v, yy, nullptr, ctx->stream);
  };
  if (comm == nullptr) {
    rows(y);
  } else {  // own rows into a zeroed N-vector, then sum over ranks
    RMG_CK(cudaMemsetAsync(y, 0, static_cast<size_t>(n()) * sizeof(double), ctx->stream));
    rows(y + row0);
    allreduce_sums(y, y, n());
  }
  ctx->launches += 1;
}

// gram_diagonal (ridge.cpp:30-37); sharded: local sums, all-reduce, + beta
void Matrix::gram_diagonal(double beta, double* out) {
  if (comm == nullptr) {
    if (dense)
      launch_dense_diag(dense->view, beta, out, ctx->stream);
    else
      launch_diag_gram(xt.view, sched.view, beta, out, ctx->stream);
    return;
  }
  if (dense)
    launch_dense_diag(dense->view, 0.0, part.get(), ctx->stream);
  else
    launch_diag_gram(xt.view, sched.view, 0.0, part.get(), ctx->stream);
  allreduce_sums(part.get(), red.get(), f());
  std::vector<double> h(f());
  if (!h.empty()) RMG_CK(cudaMemcpyAsync(h.data(), red.get(), h.size() * 8, cudaMemcpyDeviceToHost, ctx->stream));
  ctx->sync();
  for (double& d : h) d = beta + d;
  if (!h.empty()) RMG_CK(cudaMemcpyAsync(out, h.data(), h.size() * 8, cudaMemcpyHostToDevice, ctx->stream));
  ctx->sync();
}

void Matrix::spmv_t(const double* u, double* y) {
  XtArgs a;
  a.out = y;
  if (dense) {
    if (comm == nullptr) {
      launch_dense_xt(dense->view, u, Epi::Plain, a, ctx->stream);
    } else {
      XtArgs pa = a;
      pa.out = part.get();
      launch_dense_xt(dense->view, u + row0, Epi::Plain, pa, ctx->stream);
      allreduce_sums(part.get(), red.get(), f());
      RMG_CK(cudaMemcpyAsync(y, red.get(), static_cast<size_t>(f()) * 8, cudaMemcpyDeviceToDevice, ctx->stream));
    }
    ctx->launches += 2;
    return;
  }
  xt_pass(*this, u + row0, Epi::Plain, a);  // sharded: this rank's samples of u
  ctx->launches += 1;
}

// estimate_lambda_max (krylov.cpp:62-92) with the Gram operator on the device
double Matrix::lambda_max(double tol, uint64_t max_iters, uint64_t seed, uint64_t* iters, bool* conv) {
  const int64_t nf = f();
  std::vector<double> v(nf);
  CounterRng rng(seed);
  for (auto& e : v) e = rng.next_normal();
  double nv = 0.0;
  for (double e : v) nv += e * e;
  nv = std::sqrt(nv);
  if (nv == 0.0) nv = 1.0;
  for (auto& e : v) e /= nv;
  DBuf<double> dv, dw(std::max<int64_t>(1, nf));
  dv.upload(v.data(), v.size(), ctx->stream);
  double prev = 0.0, lam = 0.0;
  *conv = false;
  *iters = 0;
  for (uint64_t it = 0; it < max_iters; ++it) {
    XtArgs a;
    a.v = dv.get();
    a.out = dw.get();
    a.sc = gram_sc.get();
    apply(dv.get(), Epi::Gram, a);
    lam = ctx->read(gram_sc.get()).lambda;
    *iters = it + 1;
    if (lam == 0.0) {
      *conv = true;
      return lam;
    }
    launch_scale_by_lambda(dw.get(), dv.get(), nf, gram_sc.get(), ctx->stream);
    ctx->launches += 1;
    if (it > 0 && std::abs(lam - prev) <= tol * lam) {
      *conv = true;
      return lam;
    }
    prev = lam;
  }
  return lam;
}

// ------------------------------------------------------------------ Krylov workspace
KrylovWork::KrylovWork(int64_t n_, int keep_, uint64_t max_iters_, double tol, cudaStream_t s) : n(n_), keep(keep_) {
  if (keep > kMaxKeep) throw InvalidArgument("truncation above the supported maximum of " + std::to_string(kMaxKeep));
  const size_t m = std::max<int64_t>(1, n);
  b.alloc(m);
  x.alloc(m);
  r.alloc(m);
  z.alloc(m);
  z1.alloc(m);
  p_ring.alloc(m * (keep + 1));
  ap_ring.alloc(m * (keep + 1));
  vw.grid = vec_grid(n);
  slots.alloc(static_cast<size_t>(vw.grid) * 32);
  ticket.alloc(1);
  RMG_CK(cudaMemsetAsync(ticket.get(), 0, sizeof(unsigned), s));
  vw.slots = slots.get();
  vw.ticket = ticket.get();
  sc.alloc(1);
  set_params(tol, max_iters_, keep, s);
}

void KrylovWork::set_params(double tol, uint64_t max_iters_, int keep_m, cudaStream_t s) {
  max_iters = max_iters_;
  hist.alloc(max_iters + 1);
  inner_hist.alloc(max_iters + 1);
  KrylovScalars h;
  std::memset(&h, 0, sizeof(h));
  h.tol = tol;
  h.max_iters = static_cast<int32_t>(std::min<uint64_t>(max_iters, INT32_MAX));
  h.keep = keep_m;
  h.done = 1;
  RMG_CK(cudaMemcpyAsync(sc.get(), &h, sizeof(h), cudaMemcpyHostToDevice, s));
  RMG_CK(cudaStreamSynchronize(s));
}

// ------------------------------------------------------------------ Method
namespace {

std::vector<int64_t> run_clustering(const HostCsr& cur, const LevelSpecHost& ls, int64_t* nc, cudaStream_t stream) {
  const rmg_level_spec& s = ls.spec;
  if (s.clustering_kind == RMG_CLUSTER_IMPORTED) {
    if (static_cast<int64_t>(ls.labels.size()) != cur.f)
      throw InvalidArgument("imported labels: expected one label per feature of the level");
    *nc = static_cast<int64_t>(s.n_clusters);
    return ls.labels;
  }
  const HostCsr src = s.normalize_columns ? normalized_columns(cur) : cur;
  const HostCsr cols = transpose(src);
  const unsigned threads = std::max(1u, std::thread::hardware_concurrency());
  Clustering c;
  switch (s.clustering_kind) {
    case RMG_CLUSTER_LEADER_TOLERANCE: c = leader_follower(cols, s.tolerance); break;
    case RMG_CLUSTER_LEADER_TARGET: c = leader_follower_target(cols, static_cast<int64_t>(s.target_size)); break;
    case RMG_CLUSTER_KMEANS: {
      const int64_t k = static_cast<int64_t>(s.target_size);
      if (std::getenv("RMG_KMEANS_HOST") == nullptr && k >= 1 && k <= cols.n &&
          kmeans_gpu_supported(src.n, src.f, k, src.nnz()))
        c = kmeans_gpu(stream, cols, src, k, s.kmeans_max_iters, s.seed);  // bit-identical labels
      else
        c = kmeans(cols, k, s.kmeans_max_iters, s.seed, threads);
      break;
    }
    default: throw InvalidArgument("unknown clustering kind " + std::to_string(s.clustering_kind));
  }
  *nc = c.n_clusters;
  return c.labels;
}

}  // namespace

Method::Method(Matrix* x, double beta, int kind, const rmg_level_spec* levels, uint64_t n_levels,
               const rmg_solver_config& sol)
    : solver(sol), ctx_(x->ctx), fine_(x), beta_(beta), kind_(kind) {
  if (beta < 0.0) throw InvalidArgument("RidgeOperator: beta must be nonnegative, got " + std::to_string(beta));
  if (kind < RMG_METHOD_CG || kind > RMG_METHOD_PCG_VCYCLE_ADDITIVE)
    throw InvalidArgument("unknown method kind " + std::to_string(kind));
  if (solver.max_iters > static_cast<uint64_t>(INT32_MAX)) throw InvalidArgument("max_iters too large");
  const int keep0 = static_cast<int>(std::max<uint64_t>(solver.truncation, 1));
  RMG_CK(cudaSetDevice(ctx_->device));
  cudaStream_t s = ctx_->stream;

  if (kind == RMG_METHOD_CG || kind == RMG_METHOD_JACOBI_CG) {
    work_.push_back(std::make_unique<KrylovWork>(x->f(), 1, solver.max_iters, solver.tol, s));
    if (kind == RMG_METHOD_JACOBI_CG) jacobi_diag();  // krylov.cpp:623-626, 41-47
    return;
  }

  if (n_levels == 0 || levels == nullptr)
    throw InvalidArgument(kind != RMG_METHOD_FCG_MULTILEVEL ? "two-level method requires one level spec"
                                                            : "multilevel method requires level specs");
  const bool multi = kind == RMG_METHOD_FCG_MULTILEVEL || kind == RMG_METHOD_PCG_VCYCLE ||
                     kind == RMG_METHOD_PCG_VCYCLE_ADDITIVE;
  const uint64_t L = multi ? n_levels : 1;
  if (L > RMG_MAX_LEVELS) throw InvalidArgument("too many levels");
  for (uint64_t k = 0; k < L; ++k) {
    LevelSpecHost ls;
    ls.spec = levels[k];
    if (ls.spec.clustering_kind == RMG_CLUSTER_IMPORTED) {
      if (ls.spec.labels == nullptr) throw InvalidArgument("imported clustering without labels");
      const int64_t f = k == 0 ? x->f() : -1;  // sizes of deeper levels are checked when reached
      (void)f;
    }
    ls.spec.labels = nullptr;
    specs_.push_back(ls);
  }
  if (kind != RMG_METHOD_FCG_MULTILEVEL) specs_[0].spec.coarse_kind = RMG_COARSE_DIRECT_CHOLESKY;  // krylov.cpp:632-634
  if (kind == RMG_METHOD_PCG_VCYCLE || kind == RMG_METHOD_PCG_VCYCLE_ADDITIVE)  // intermediate levels are visited by the recursive cycle
    for (uint64_t k = 0; k < L; ++k)
      specs_[k].spec.coarse_kind = k + 1 == L ? RMG_COARSE_DIRECT_CHOLESKY : RMG_COARSE_INNER_FCG;
  // krylov.cpp:495-505
  for (uint64_t k = 0; k + 1 < L; ++k)
    if (specs_[k].spec.coarse_kind == RMG_COARSE_DIRECT_CHOLESKY)
      throw InvalidArgument("build_hierarchy: only the last level may use direct_cholesky");
  if (specs_[L - 1].spec.coarse_kind != RMG_COARSE_DIRECT_CHOLESKY)
    throw InvalidArgument("build_hierarchy: the coarsest level must use direct_cholesky");

  // levels (krylov.cpp:512-530)
  const bool slog = std::getenv("RMG_SETUP_LOG") != nullptr;  // setup phase timings on stderr
  auto tnow = [] { return std::chrono::steady_clock::now(); };
  auto tlog = [&](const char* what, uint64_t k, std::chrono::steady_clock::time_point t0) {
    if (slog)
      std::fprintf(stderr, "[rmg setup] level %llu %-12s %8.3f s\n", static_cast<unsigned long long>(k), what,
                   std::chrono::duration<double>(tnow() - t0).count());
  };
  // V-cycle kinds: a coarse level that enters additively or keeps a dense Gram matrix never
  // applies X_k, so its K1 layout and hot X^T blocks wait for a first application
  // (Matrix::ensure_operator; build_vcycle applies the levels that smooth); RMG_EAGER_LEVELS=1
  // builds them all at once as before
  const bool defer_coarse = (kind == RMG_METHOD_PCG_VCYCLE || kind == RMG_METHOD_PCG_VCYCLE_ADDITIVE) &&
                            std::getenv("RMG_EAGER_LEVELS") == nullptr;
  double beta_run = beta;
  for (uint64_t k = 0; k < L; ++k) {
    auto t0 = tnow();
    Matrix& curm = level_matrix(k);
    const int64_t cur_f = curm.f();
    // dense X without a host CSR: k-means, X_c = X P and the Gram matrices on
    // the device, bit-identical to the host restatement
    const bool dev = curm.device_setup();
    if (levels[k].clustering_kind == RMG_CLUSTER_IMPORTED)
      specs_[k].labels.assign(levels[k].labels, levels[k].labels + cur_f);
    const double next_beta = specs_[k].spec.has_beta_override ? specs_[k].spec.beta_override : beta_run;
    int64_t nc = 0;
    std::vector<int64_t> lab;
    const rmg_level_spec& cs = specs_[k].spec;
    const bool dense_rows = curm.rows_only && curm.dense != nullptr;  // per-rank dense rows
    if (dev && cs.clustering_kind == RMG_CLUSTER_KMEANS) {
      const int64_t k_c = static_cast<int64_t>(cs.target_size);
      if (k_c < 1 || k_c > cur_f) throw InvalidArgument("kmeans: k outside [1, F]");
      const int64_t ldx = (cur_f + 1) / 2 * 2;
      DBuf<double> xc(static_cast<size_t>(std::max<int64_t>(1, curm.n())) * ldx);
      dense_columns_f64(s, curm.dense->view, cs.normalize_columns != 0, xc.get(), ldx);
      Clustering c = kmeans_dense_gpu(s, xc.get(), curm.n(), cur_f, ldx, k_c, cs.kmeans_max_iters, cs.seed);
      nc = c.n_clusters;
      lab = std::move(c.labels);
    } else if (cs.clustering_kind == RMG_CLUSTER_KMEANS_SKETCH) {
      lab = sketch_clustering(curm, cs, &nc);
    } else if ((dev || curm.rows_only) && cs.clustering_kind == RMG_CLUSTER_IMPORTED) {
      if (static_cast<int64_t>(specs_[k].labels.size()) != cur_f)
        throw InvalidArgument("imported labels: expected one label per feature of the level");
      nc = static_cast<int64_t>(cs.n_clusters);
      if (nc < 1 || nc > cur_f) throw InvalidArgument("imported labels: n_clusters outside [1, F]");
      for (int64_t v : specs_[k].labels)
        if (v < 0 || v >= nc) throw InvalidArgument("imported labels: label outside [0, n_clusters)");
      lab = specs_[k].labels;
    } else if (curm.rows_only) {  // every rank holds only its rows: no exact column clustering
      throw InvalidArgument(
          "build_hierarchy: a row-sharded matrix (rmg_matrix_create_csr_rows / _dense_rows) needs kmeans_sketch or imported "
          "labels; exact k-means / leader-follower need every row of a column on one device");
    } else {
      lab = run_clustering(curm.host_csr(), specs_[k], &nc, s);
    }
    tlog("clustering", k, t0);
    t0 = tnow();
    if (nc >= cur_f)
      throw InvalidArgument("build_hierarchy: level " + std::to_string(k + 1) + " has " + std::to_string(nc) +
                            " clusters, not smaller than its fine level (" + std::to_string(cur_f) + " features)");
    auto lvl = std::make_unique<CoarseLevelDev>();
    lvl->agg = make_aggregation(lab, nc);
    if (dev) {
      const int64_t ldc = (nc + 3) / 4 * 4;
      DBuf<char> xcd(std::max<size_t>(1, static_cast<size_t>(curm.n()) * ldc * sizeof(double)));
      coarsen_dense_gpu(s, curm.dense->view, lvl->agg, reinterpret_cast<double*>(xcd.get()), ldc);
      lvl->mat = std::make_unique<Matrix>(ctx_, curm.n(), nc, std::move(xcd), 0, ldc);
    } else if (dense_rows) {  // X_k = X P on this rank's rows, on the device
      const int64_t ldc = (nc + 3) / 4 * 4, nl = curm.n_local();
      DBuf<char> xcd(std::max<size_t>(1, static_cast<size_t>(nl) * ldc * sizeof(double)));
      coarsen_dense_gpu(s, curm.dense->view, lvl->agg, reinterpret_cast<double*>(xcd.get()), ldc);
      lvl->mat = std::make_unique<Matrix>(ctx_, curm.n_global, curm.row0, nl, nc, std::move(xcd), 0, ldc, curm.comm);
    } else if (curm.rows_only) {  // X_k = X P is row-local: every rank coarsens its own rows
      lvl->mat = std::make_unique<Matrix>(ctx_, coarsen_level(curm, lvl->agg), curm.n_global, curm.row0, true,
                                          curm.comm, defer_coarse);
    } else {
      lvl->mat = std::make_unique<Matrix>(ctx_, coarsen_level(curm, lvl->agg), true, nullptr, nullptr, defer_coarse);
    }
    lvl->beta = next_beta;
    lvl->label.upload(lvl->agg.label.data(), lvl->agg.label.size(), s);
    lvl->weight.upload(lvl->agg.weight.data(), lvl->agg.weight.size(), s);
    lvl->mptr.upload(lvl->agg.mptr.data(), lvl->agg.mptr.size(), s);
    lvl->members.upload(lvl->agg.members.data(), lvl->agg.members.size(), s);
    {
      HostCsr pt;  // P^T: row s lists the members of cluster s in increasing order
      pt.n = nc;
      pt.f = cur_f;
      pt.ptr.assign(lvl->agg.mptr.begin(), lvl->agg.mptr.end());
      pt.idx.assign(lvl->agg.members.begin(), lvl->agg.members.end());
      pt.val.resize(pt.idx.size());
      for (size_t q = 0; q < pt.idx.size(); ++q) pt.val[q] = lvl->agg.weight[pt.idx[q]];
      lvl->pt.upload(pt, false, s);
      lvl->pt_sched.build(pt, s, nc);
    }
    labels_.push_back(std::move(lab));
    coarse_.push_back(std::move(lvl));
    beta_run = next_beta;
    tlog("coarsen", k, t0);
  }
  const int64_t fc_last = coarse_.back()->mat->f();
  if (fc_last > 4096)  // kDirectSolveCap, krylov.hpp:170
    throw InvalidArgument("build_hierarchy: coarsest level has " + std::to_string(fc_last) +
                          " features, above the direct-solve cap 4096");
  // omega_k = 2 / (beta_k + lambda_max(X_k^T X_k)) (krylov.cpp:539-546)
  for (uint64_t k = 0; k < L; ++k) {
    if (specs_[k].spec.has_omega_override) {
      if (!(specs_[k].spec.omega_override > 0.0))
        throw InvalidArgument("TwoLevelPreconditioner: omega must be positive");
      omega_.push_back(specs_[k].spec.omega_override);
      lambda_.push_back(0.0);
      continue;
    }
    if (k >= 1 && !level_matrix(k).op_ready) {  // V-cycle kinds take their weights in build_vcycle
      lambda_.push_back(0.0);
      omega_.push_back(0.0);
      continue;
    }
    uint64_t its;
    bool cv;
    const auto t0 = tnow();
    const double lmax = level_matrix(k).lambda_max(1e-4, 200, 0x5eed + k, &its, &cv);
    lambda_.push_back(lmax);  // beta-independent: reused by set_beta
    omega_.push_back(2.0 / (level_beta(k) + lmax));
    tlog("lambda_max", k, t0);
  }
  // coarsest dense solve (krylov.cpp:349-376), through A_c^{-1}
  {
    auto t0 = tnow();
    const std::vector<double> ac = level_gram(*coarse_.back()->mat, coarse_.back()->beta);
    const std::vector<double> inv =
        spd_inverse(ac, fc_last, "level " + std::to_string(L - 1) + " -> " + std::to_string(L));
    ainv_.upload(inv.data(), inv.size(), s);
    rc_last_.alloc(std::max<int64_t>(1, fc_last));
    ec_last_.alloc(std::max<int64_t>(1, fc_last));
    // workspaces: level 0 = outer FCG, level k >= 1 = inner solve configured by spec k-1
    work_.push_back(std::make_unique<KrylovWork>(x->f(), keep0, solver.max_iters, solver.tol, s));
    if (const char* pad = std::getenv("RMG_DENSE_PAD"))  // diagnostics: shift the inner buffers
      pad_.alloc(static_cast<size_t>(std::atoll(pad)));
    if (const char* pad = std::getenv("RMG_PAD_W")) {
      pads_.emplace_back();
      pads_.back().alloc(static_cast<size_t>(std::atoll(pad)));
    }
    for (uint64_t k = 1; k < L; ++k) {
      const rmg_level_spec& sp = specs_[k - 1].spec;
      const int keep = static_cast<int>(std::max<uint64_t>(sp.coarse_truncation, 1));
      work_.push_back(
          std::make_unique<KrylovWork>(level_matrix(k).f(), keep, sp.coarse_max_iters, sp.coarse_tol, s));
    }
    tlog("coarsest_inv", L, t0);
    t0 = tnow();
    build_dense_levels(inv);
    tlog("dense_levels", L, t0);
    if (vc_kind()) {
      t0 = tnow();
      build_vcycle();
      tlog("vcycle", L, t0);
    }
    t0 = tnow();
    for (size_t k = 1; k < dense_.size(); ++k)
      if (dense_[k]) tune_dense_partials(k);
    tlog("tune", L, t0);
  }
  ctx_->sync();
}

// RMG_CLUSTER_KMEANS_SKETCH: the reference's k-means
// (kmeans_dense_gpu, bit-identical arithmetic) on S = G^T X, G an N x d sign
// matrix, the columns of X unit-normalised first when asked.
std::vector<int64_t> Method::sketch_clustering(Matrix& m, const rmg_level_spec& cs, int64_t* nc) {
  if (m.comm != nullptr && m.dense != nullptr && !m.rows_only)
    throw InvalidArgument("kmeans_sketch: replicated-setup sharded dense matrices unsupported");
  const int64_t f = m.f(), n = m.n();
  const int64_t k = static_cast<int64_t>(cs.target_size);
  if (k < 1 || k > f) throw InvalidArgument("kmeans: k outside [1, F]");
  const int d = cs.sketch_dim == 0 ? 32 : static_cast<int>(std::min<uint64_t>(cs.sketch_dim, 1u << 30));
  if (d < 1 || d > 32) throw InvalidArgument("kmeans_sketch: sketch dimension outside [1, 32]");
  cudaStream_t s = ctx_->stream;
  const int64_t ldS = (f + 1) / 2 * 2;
  DBuf<double> S(static_cast<size_t>(d) * ldS);
  RMG_CK(cudaMemsetAsync(S.get(), 0, S.size() * sizeof(double), s));
  if (m.dense && m.rows_only) {  // this rank's rows; columns scaled by the all-reduced norms
    const int64_t ldx = (f + 1) / 2 * 2, nl = m.n_local();
    DBuf<double> xc(static_cast<size_t>(std::max<int64_t>(1, nl)) * ldx);
    dense_columns_f64(s, m.dense->view, false, xc.get(), ldx);
    sketch_dense_gpu(s, xc.get(), nl, f, ldx, d, cs.seed, S.get(), ldS, m.row0);
    m.allreduce_sums(S.get(), S.get(), static_cast<int64_t>(d) * ldS);
    if (cs.normalize_columns) {  // G^T (X D^-1) = (G^T X) D^-1, D = the global column norms
      DBuf<double> nrm(std::max<int64_t>(1, f));
      m.gram_diagonal(0.0, nrm.get());
      std::vector<double> v(f), hs(static_cast<size_t>(d) * ldS);
      if (f) RMG_CK(cudaMemcpyAsync(v.data(), nrm.get(), f * 8, cudaMemcpyDeviceToHost, s));
      RMG_CK(cudaMemcpyAsync(hs.data(), S.get(), hs.size() * 8, cudaMemcpyDeviceToHost, s));
      ctx_->sync();
      for (int c = 0; c < d; ++c)
        for (int64_t j = 0; j < f; ++j)
          if (v[j] > 0.0) hs[c * ldS + j] /= std::sqrt(v[j]);
      S.upload(hs.data(), hs.size(), s);
    }
  } else if (m.dense) {
    const int64_t ldx = (f + 1) / 2 * 2;
    DBuf<double> xc(static_cast<size_t>(std::max<int64_t>(1, n)) * ldx);
    dense_columns_f64(s, m.dense->view, cs.normalize_columns != 0, xc.get(), ldx);
    sketch_dense_gpu(s, xc.get(), n, f, ldx, d, cs.seed, S.get(), ldS);
  } else {
    DBuf<double> nrm;
    if (cs.normalize_columns) {  // normalized_columns (host_setup.cpp:79-90): sum of squares per column
      // in row order = gram_diagonal(0) (ridge.cpp:30-37, same order); sharded: summed over ranks
      nrm.alloc(std::max<int64_t>(1, f));
      m.gram_diagonal(0.0, nrm.get());
      std::vector<double> v(f);
      if (f) RMG_CK(cudaMemcpyAsync(v.data(), nrm.get(), f * 8, cudaMemcpyDeviceToHost, s));
      ctx_->sync();
      for (double& e : v) e = std::sqrt(e);
      nrm.upload(v.data(), v.size(), s);
    }
    // S over this device's rows (global row numbers seed the signs); sharded: summed over ranks
    sketch_sparse_gpu(s, m.xt.view, nrm.get(), d, cs.seed, S.get(), ldS, m.row0);
    if (m.comm != nullptr) m.allreduce_sums(S.get(), S.get(), static_cast<int64_t>(d) * ldS);
  }
  Clustering c = kmeans_dense_gpu(s, S.get(), d, f, ldS, k, cs.kmeans_max_iters, cs.seed);
  *nc = c.n_clusters;
  return std::move(c.labels);
}

// X_k^T X_k + beta I (coarse_gram, krylov.cpp:350-365): on the device for a
// device-resident dense level (the beta-free sums cached: adding beta to the
// diagonal after the sums is what coarse_gram does, so a beta sweep reuses them)
std::vector<double> Method::level_gram(Matrix& m, double beta) {
  const int64_t n = m.f();
  if (m.gram_cache.empty()) {
    if (m.dense != nullptr && m.rows_only) {  // this rank's rows, summed over the ranks
      std::vector<double> g = gram_dense_gpu(ctx_->stream, m.dense->view);
      DBuf<double> d;
      d.upload(g.data(), g.size(), ctx_->stream);
      if (!g.empty()) {
        m.allreduce_sums(d.get(), d.get(), static_cast<int64_t>(g.size()));
        RMG_CK(cudaMemcpyAsync(g.data(), d.get(), g.size() * 8, cudaMemcpyDeviceToHost, ctx_->stream));
      }
      ctx_->sync();
      m.gram_cache = std::move(g);
    } else if (m.device_setup()) {
      m.gram_cache = gram_dense_gpu(ctx_->stream, m.dense->view);
    } else if ((m.comm != nullptr && !m.rows_only) || m.dense != nullptr ||
               (std::getenv("RMG_HOST_GRAM") != nullptr && m.comm == nullptr)) {
      return coarse_gram(m.host_csr(), beta);
    } else {  // sparse level: the same sums on the device (dense_gram.cu), bit-identical;
              // row-sharded: every rank's rows, then summed over the ranks
      DBuf<double> g(static_cast<size_t>(std::max<int64_t>(1, n)) * std::max<int64_t>(1, n));
      device_gram(m, g.get(), n);
      if (m.comm != nullptr) m.allreduce_sums(g.get(), g.get(), n * n);
      m.gram_cache.resize(static_cast<size_t>(n) * n);
      if (n) RMG_CK(cudaMemcpyAsync(m.gram_cache.data(), g.get(), m.gram_cache.size() * 8, cudaMemcpyDeviceToHost,
                                    ctx_->stream));
      ctx_->sync();
    }
  }
  std::vector<double> a = m.gram_cache;
  for (int64_t i = 0; i < n; ++i) a[i * n + i] += beta;  // after the sums, as coarse_gram does
  return a;
}

// G = X^T X of a sparse level on the device: X's row CSR is staged for the
// assembly (the resident K1 copy is SELL-32, possibly relabeled) and X^T is the
// resident feature CSR.  Dense levels: gram_dense_gpu (dense_setup.cu).
void Method::device_gram(Matrix& m, double* G, int64_t ld) {
  cudaStream_t s = ctx_->stream;
  const int64_t n = m.f();
  if (m.dense != nullptr) {
    if (m.gram_cache.empty()) {
      if (m.rows_only) {
        (void)level_gram(m, 0.0);  // fills the all-reduced cache
      } else {
        m.gram_cache = gram_dense_gpu(s, m.dense->view);
      }
    }
    for (int64_t i = 0; i < n; ++i)
      RMG_CK(cudaMemcpyAsync(G + i * ld, m.gram_cache.data() + i * n, n * 8, cudaMemcpyHostToDevice, s));
    ctx_->sync();
    return;
  }
  if (m.comm != nullptr && !m.rows_only)
    throw InvalidArgument("device Gram: replicated-setup sharded matrices keep the host Gram");
  const HostCsr& h = m.host_csr();
  DBuf<int32_t> xp, xi;
  DBuf<double> xv;
  {
    const std::vector<int32_t> p32 = narrow(h.ptr, "row offsets"), i32 = narrow(h.idx, "column indices");
    xp.upload(p32.data(), p32.size(), s);
    xi.upload(i32.data(), i32.size(), s);
    if (!m.pattern) xv.upload(h.val.data(), h.val.size(), s);
    sparse_gram_gpu(s, xp.get(), xi.get(), m.pattern ? nullptr : xv.get(), m.xt.view.ptr, m.xt.view.idx,
                    m.pattern ? nullptr : m.xt.view.val, n, G, ld);
    ctx_->sync();  // the staged CSR is released on return
  }
}

// X_c = X P of a sparse level (coarsening.cpp:112-148) on the device, bit-identical
// to the host restatement `coarsen` (RMG_HOST_COARSEN=1 keeps the host loop).
HostCsr Method::coarsen_level(Matrix& m, const Aggregation& agg) {
  const HostCsr& h = m.host_csr();
  if (std::getenv("RMG_HOST_COARSEN") != nullptr || (m.comm != nullptr && !m.rows_only) || h.nnz() == 0)
    return coarsen(h, agg);
  if (agg.n_fine != h.f) throw InvalidArgument("coarsen: prolongation does not match the matrix features");
  cudaStream_t s = ctx_->stream;
  const int64_t n = h.n, nnz = h.nnz();
  DBuf<int32_t> xp, xi, lab, cnt, ci;
  DBuf<double> xv, wt, cv;
  const bool slog = std::getenv("RMG_SETUP_LOG") != nullptr;
  auto tl = std::chrono::steady_clock::now();
  auto lap = [&](const char* what) {
    if (!slog) return;
    ctx_->sync();
    const auto now = std::chrono::steady_clock::now();
    std::fprintf(stderr, "[rmg setup]   coarsen %-9s %8.3f s\n", what, std::chrono::duration<double>(now - tl).count());
    tl = now;
  };
  {
    const std::vector<int32_t> p32 = narrow(h.ptr, "row offsets"), i32 = narrow(h.idx, "column indices");
    xp.upload(p32.data(), p32.size(), s);
    xi.upload(i32.data(), i32.size(), s);
  }
  if (!m.pattern) xv.upload(h.val.data(), h.val.size(), s);
  lab.upload(agg.label.data(), agg.label.size(), s);
  wt.upload(agg.weight.data(), agg.weight.size(), s);
  cnt.alloc(std::max<int64_t>(1, n));
  ci.alloc(std::max<int64_t>(1, nnz));
  cv.alloc(std::max<int64_t>(1, nnz));
  lap("stage");
  auto t1 = std::chrono::steady_clock::now();
  coarsen_rows_gpu(s, xp.get(), xi.get(), m.pattern ? nullptr : xv.get(), n, lab.get(), wt.get(), cnt.get(), ci.get(),
                   cv.get());
  if (slog) {
    ctx_->sync();
    std::fprintf(stderr, "[rmg setup]   coarsen kernel %.3f s\n",
                 std::chrono::duration<double>(std::chrono::steady_clock::now() - t1).count());
  }
  tl = std::chrono::steady_clock::now();
  std::vector<int32_t> hc(n), hi(nnz);
  std::vector<double> hv(nnz);
  RMG_CK(cudaMemcpyAsync(hc.data(), cnt.get(), n * sizeof(int32_t), cudaMemcpyDeviceToHost, s));
  RMG_CK(cudaMemcpyAsync(hi.data(), ci.get(), nnz * sizeof(int32_t), cudaMemcpyDeviceToHost, s));
  RMG_CK(cudaMemcpyAsync(hv.data(), cv.get(), nnz * sizeof(double), cudaMemcpyDeviceToHost, s));
  ctx_->sync();
  lap("D2H");
  HostCsr c;
  c.n = n;
  c.f = agg.n_coarse;
  c.ptr.assign(n + 1, 0);
  for (int64_t r = 0; r < n; ++r) c.ptr[r + 1] = c.ptr[r] + hc[r];
  c.idx.resize(c.ptr[n]);
  c.val.resize(c.ptr[n]);
  // row r's entries were written at its fine offsets: compact (threaded over rows)
  const unsigned T = nnz < (1 << 20) ? 1u : std::max(1u, std::min(32u, std::thread::hardware_concurrency()));
  auto body = [&](unsigned t) {
    for (int64_t r = n * t / T; r < n * (t + 1) / T; ++r)
      for (int64_t q = 0; q < hc[r]; ++q) {
        c.idx[c.ptr[r] + q] = hi[h.ptr[r] + q];
        c.val[c.ptr[r] + q] = hv[h.ptr[r] + q];
      }
  };
  std::vector<std::thread> pool;
  for (unsigned t = 1; t < T; ++t) pool.emplace_back(body, t);
  body(0);
  for (auto& th : pool) th.join();
  lap("compact");
  return c;
}

// pcg_vcycle: dense G_k for the levels where streaming n_k^2 doubles once costs
// fewer bytes than the X_k sweep pair (X_k, then X_k^T) it replaces, and that
// fit comfortably in free HBM (RMG_VC_DENSE=0 keeps the sweeps).
void Method::build_dense_grams() {
  dg_built_ = true;
  dg_.clear();
  dg_.resize(coarse_.size());
  const char* e = std::getenv("RMG_VC_DENSE");
  if (e != nullptr && std::string(e) == "0") return;
  for (size_t k = 1; k < coarse_.size(); ++k) {
    if (vc_additive(k)) continue;  // an additive level never applies its operator
    Matrix& m = level_matrix(k);
    if (m.comm != nullptr && !m.rows_only) continue;
    const int64_t n = m.f();
    const double dense_bytes = 8.0 * static_cast<double>(n) * static_cast<double>(n);
    const double sweep_bytes = m.dense != nullptr ? static_cast<double>(m.n()) * n * 8.0
                                                  : 2.0 * static_cast<double>(m.nnz()) * (m.pattern ? 4.0 : 12.0);
    size_t free_b = 0, total_b = 0;
    RMG_CK(cudaMemGetInfo(&free_b, &total_b));
    if (!(dense_bytes < sweep_bytes) || dense_bytes > 0.4 * static_cast<double>(free_b)) continue;
    if (m.dense == nullptr) {  // assembly cost: k_gram_rows visits sum_r nnz_r^2 entries per 6144-column tile
      const HostCsr& h = m.host_csr();
      double visits = 0.0;
      for (int64_t r = 0; r < h.n; ++r) {
        const double l = static_cast<double>(h.ptr[r + 1] - h.ptr[r]);
        visits += l * l;
      }
      visits *= static_cast<double>((n + 6143) / 6144);
      if (visits > 1e11) continue;  // ~a minute of setup (cfg 5's 50 000-feature level): keep the sweeps
    }
    auto d = std::make_unique<DenseGram>();
    d->n = n;
    d->ld = (n + 1) / 2 * 2;
    d->G.alloc(static_cast<size_t>(std::max<int64_t>(1, n)) * d->ld);
    d->scratch.alloc(static_cast<size_t>(std::max<int64_t>(1, gram_gemm_scratch(n))));
    device_gram(m, d->G.get(), d->ld);
    if (m.comm != nullptr && m.dense == nullptr)  // replicated G_k (dense levels: summed in level_gram)
      m.allreduce_sums(d->G.get(), d->G.get(), n * d->ld);
    dg_[k] = std::move(d);
  }
}

// JacobiPreconditioner (krylov.cpp:41-47): inverse of beta + diag(X^T X)
void Method::jacobi_diag() {
  cudaStream_t s = ctx_->stream;
  DBuf<double> d(std::max<int64_t>(1, fine_->f()));
  fine_->gram_diagonal(beta_, d.get());
  std::vector<double> h(fine_->f());
  if (!h.empty()) RMG_CK(cudaMemcpyAsync(h.data(), d.get(), h.size() * 8, cudaMemcpyDeviceToHost, s));
  ctx_->sync();
  for (double& v : h) {
    if (!(v > 0.0)) throw InvalidArgument("JacobiPreconditioner: diagonal must be positive");
    v = 1.0 / v;
  }
  inv_diag_.upload(h.data(), h.size(), s);
  ctx_->sync();
}

// A new regularization for the same hierarchy (BASELINE cfg 3's beta sweep):
// clustering, P, X_c and lambda_max(X_k^T X_k) do not depend on beta, so only
// the level betas (overrides kept), omega_k = 2 / (beta_k + lambda_k), the
// coarsest inverse and the dense inner levels are rebuilt -- exactly what a
// fresh prepare at this beta computes.
void Method::set_beta(double beta) {
  const int block_k = bw_graph_ && bw_.k == bw_graph_k_ ? bw_graph_k_ : 0;
  const bool had_vc = vc_graph_ != nullptr;
  set_beta_impl(beta);
  // a sweep of solves: the loop graphs for the new beta are part of this step, not of the next solve
  if (block_k > 0 && std::getenv("RMG_NO_GRAPH") == nullptr) build_block_graph(block_k);
  if (had_vc && !vc_graph_ && !profiling_) build_vcycle_graph();
}

void Method::set_beta_impl(double beta) {
  if (beta < 0.0) throw InvalidArgument("RidgeOperator: beta must be nonnegative, got " + std::to_string(beta));
  RMG_CK(cudaSetDevice(ctx_->device));
  fcg_graph_.reset();  // the graphs point at the coarse buffers rebuilt below
  vc_graph_retired_ = std::move(vc_graph_);
  bw_graph_retired_ = std::move(bw_graph_);
  cg_graph_[0].reset();  // beta is a kernel argument of every captured apply
  cg_graph_[1].reset();
  beta_ = beta;
  if (kind_ == RMG_METHOD_CG) return;
  if (kind_ == RMG_METHOD_JACOBI_CG) {
    jacobi_diag();
    return;
  }
  const size_t L = coarse_.size();
  double beta_run = beta;
  for (size_t k = 0; k < L; ++k) {
    const double next = specs_[k].spec.has_beta_override ? specs_[k].spec.beta_override : beta_run;
    coarse_[k]->beta = next;
    beta_run = next;
  }
  for (size_t k = 0; k < L; ++k)
    if (!specs_[k].spec.has_omega_override) omega_[k] = 2.0 / (level_beta(k) + lambda_[k]);
  const int64_t fc_last = coarse_.back()->mat->f();
  const std::vector<double> ac = level_gram(*coarse_.back()->mat, coarse_.back()->beta);
  const std::vector<double> inv = spd_inverse(ac, fc_last, "level " + std::to_string(L - 1) + " -> " + std::to_string(L));
  ainv_.upload(inv.data(), inv.size(), ctx_->stream);
  dense_.clear();
  build_dense_levels(inv);
  for (size_t k = 1; k < dense_.size(); ++k)
    if (dense_[k]) tune_dense_partials(k);
  if (vc_kind()) build_vcycle();
  ctx_->sync();
}

// Dense persistent inner solves (dense_level.cu) for every inner level that
// has at most 4096 unknowns and whose own preconditioner is linear (direct
// coarsest level below it) or absent (inner_cg).
void Method::build_dense_levels(const std::vector<double>& ainv_host) {
  const size_t L = coarse_.size();
  dense_.resize(L + 1);
  if (vc_kind()) return;  // no inner Krylov solves
  if (std::getenv("RMG_DISABLE_DENSE_INNER") != nullptr) return;
  cudaStream_t s = ctx_->stream;
  const unsigned threads = std::max(1u, std::thread::hardware_concurrency());
  for (size_t k = 1; k < L; ++k) {
    const int kind = specs_[k - 1].spec.coarse_kind;
    const bool fcg = kind == RMG_COARSE_INNER_FCG;
    const int64_t n = level_matrix(k).f();
    if (n > 4096 || (fcg && k + 1 != L)) continue;
    auto d = std::make_unique<DenseInner>();
    d->fcg = fcg;
    d->omega = omega_[k];
    const std::vector<double> a = level_gram(level_matrix(k), level_beta(k));  // X_k^T X_k + beta_k I
    auto padk = [&](const char* name) {  // diagnostics: shift one buffer group
      if (const char* e = std::getenv(name)) {
        pads_.emplace_back();
        pads_.back().alloc(static_cast<size_t>(std::atoll(e)));
      }
    };
    d->nc = fcg ? static_cast<int>(coarse_[k]->agg.n_coarse) : 0;
    d->plan = plan_dense_krylov(static_cast<int>(n), d->nc, ctx_->device);
    d->lowrank = fcg && d->nc <= d->plan.max_clusters && std::getenv("RMG_DENSE_FULL_M") == nullptr;
    padk("RMG_PAD_A");
    if (!fcg) {
      d->A.upload(a.data(), a.size(), s);
    } else {  // Q = (I - omega A_k) P A_{k+1}^{-1}
      const Aggregation& agg = coarse_[k]->agg;
      const int64_t nc = agg.n_coarse;
      std::vector<double> g(static_cast<size_t>(n) * nc), q(static_cast<size_t>(n) * nc);
      for (int64_t i = 0; i < n; ++i)
        for (int64_t c = 0; c < nc; ++c) g[i * nc + c] = agg.weight[i] * ainv_host[agg.label[i] * nc + c];
      std::vector<std::thread> pool;
      const int64_t step = (n + threads - 1) / threads;
      for (unsigned t = 0; t < threads; ++t) {
        const int64_t lo = std::min<int64_t>(n, t * step), hi = std::min<int64_t>(n, lo + step);
        pool.emplace_back([&, lo, hi] {
          std::vector<double> acc(nc);
          for (int64_t i = lo; i < hi; ++i) {
            std::fill(acc.begin(), acc.end(), 0.0);
            for (int64_t j = 0; j < n; ++j) {
              const double aij = a[i * n + j];
              if (aij == 0.0) continue;
              const double* gj = &g[j * nc];
              for (int64_t c = 0; c < nc; ++c) acc[c] += aij * gj[c];
            }
            for (int64_t c = 0; c < nc; ++c) q[i * nc + c] = g[i * nc + c] - d->omega * acc[c];
          }
        });
      }
      for (auto& th : pool) th.join();
      if (d->lowrank) {
        // positions in cluster order; A and Q rows follow; segments of (CTA, cluster)
        std::vector<int32_t> perm(n);
        std::iota(perm.begin(), perm.end(), 0);
        std::stable_sort(perm.begin(), perm.end(),
                         [&](int32_t i, int32_t j) { return agg.label[i] < agg.label[j]; });
        std::vector<int32_t> cid(n);
        std::vector<double> wts(n), ap(static_cast<size_t>(n) * n), qp(static_cast<size_t>(n) * nc);
        for (int64_t i = 0; i < n; ++i) {
          cid[i] = static_cast<int32_t>(agg.label[perm[i]]);
          wts[i] = agg.weight[perm[i]];
          const size_t pi = static_cast<size_t>(perm[i]);
          for (int64_t j = 0; j < n; ++j) ap[i * n + j] = a[pi * n + perm[j]];
          std::copy(&q[pi * nc], &q[pi * nc] + nc, &qp[i * nc]);
        }
        const int R = d->plan.rows_per_cta, grid = d->plan.grid;
        std::vector<int32_t> cta_seg0(grid), cseg(nc + 1, -1);
        int32_t segs = 0;
        for (int b = 0; b < grid; ++b) {
          cta_seg0[b] = segs;
          for (int64_t i = static_cast<int64_t>(b) * R; i < std::min<int64_t>(n, (b + 1) * R); ++i) {
            if (i == static_cast<int64_t>(b) * R || cid[i] != cid[i - 1]) {
              if (cseg[cid[i]] < 0) cseg[cid[i]] = segs;
              ++segs;
            }
          }
        }
        cseg[nc] = segs;
        for (int64_t c = nc - 1; c >= 0; --c)  // empty clusters: empty range
          if (cseg[c] < 0) cseg[c] = cseg[c + 1];
        d->n_segments = segs;
        d->lowrank = segs <= d->plan.max_clusters;  // else the dense M fallback below
        if (d->lowrank) {
          d->A.upload(ap.data(), ap.size(), s);
          d->Q.upload(qp.data(), qp.size(), s);
          d->perm.upload(perm.data(), perm.size(), s);
          d->cid.upload(cid.data(), cid.size(), s);
          d->wts.upload(wts.data(), wts.size(), s);
          d->cta_seg0.upload(cta_seg0.data(), cta_seg0.size(), s);
          d->cseg.upload(cseg.data(), cseg.size(), s);
          d->spart.alloc(std::max<int32_t>(1, 3 * segs));
          d->xp.alloc(std::max<int64_t>(1, n));
        }
      }
      if (!d->lowrank) {  // dense M = Q P^T: M[i][j] = Q[i][label_j] w_j
        d->A.upload(a.data(), a.size(), s);
        padk("RMG_PAD_Q");
        std::vector<double> mm(static_cast<size_t>(n) * n);
        for (int64_t i = 0; i < n; ++i)
          for (int64_t j = 0; j < n; ++j) mm[i * n + j] = q[i * nc + agg.label[j]] * agg.weight[j];
        d->Q.upload(mm.data(), mm.size(), s);
      }
    }
    padk("RMG_PAD_P");
    d->pap_ring.alloc(kMaxKeep + 2);
    d->zfull.alloc(std::max<int64_t>(1, n));
    // own 2 MB-granular allocation: the cross-CTA partials are read by every CTA
    // after every grid barrier, so their placement is on the critical path
    d->partials.alloc(std::max<size_t>(static_cast<size_t>(d->plan.grid) * d->plan.partial_stride, 262144));
    d->cg_shared.alloc(4);
    if (std::getenv("RMG_DENSE_TIMING") != nullptr) {
      d->timing.alloc(512);
      RMG_CK(cudaMemsetAsync(d->timing.get(), 0, 512 * sizeof(unsigned long long), s));
    }
    dense_[k] = std::move(d);
  }
}

DenseKrylovArgs Method::dense_args(size_t k, const double* rhs) {
  DenseInner& d = *dense_[k];
  KrylovWork& w = *work_[k];
  DenseKrylovArgs a;
  a.n = static_cast<int>(level_matrix(k).f());
  a.nc = d.nc;
  a.fcg = d.fcg ? 1 : 0;
  a.keep = w.keep;
  a.max_iters = static_cast<int>(std::min<uint64_t>(w.max_iters, INT32_MAX));
  a.tol = specs_[k - 1].spec.coarse_tol;
  a.omega = d.omega;
  a.A = d.A.get();
  a.M = d.Q.get();
  a.b = rhs;
  a.x = w.x.get();
  a.x_out = w.x.get();
  if (d.lowrank) {
    a.lowrank = 1;
    a.n_segments = d.n_segments;
    a.perm = d.perm.get();
    a.cid = d.cid.get();
    a.wts = d.wts.get();
    a.cta_seg0 = d.cta_seg0.get();
    a.cseg = d.cseg.get();
    a.spart = d.spart.get();
    a.x = d.xp.get();
  }
  a.zfull = d.zfull.get();
  a.r = w.r.get();
  a.p_ring = w.p_ring.get();
  a.ap_ring = w.ap_ring.get();
  a.pap_ring = d.pap_ring.get();
  a.partials = d.partials.get();
  a.cg_rz_shared = d.cg_shared.get();
  a.cg_beta_shared = d.cg_shared.get() + 2;
  a.hist = w.hist.get();
  a.sc = w.sc.get();
  a.timing = d.timing.get();
  if (const char* dbg = std::getenv("RMG_DENSE_DBG")) a.dbg = std::atoi(dbg);
  return a;
}

uint64_t Method::run_dense(size_t k, const double* rhs) {
  const DenseKrylovArgs a = dense_args(k, rhs);
  OpProfile* pr = prof(k);  // level-k profile: K1 slot = whole persistent inner solve
  if (pr) pr->mark(ctx_->stream);
  launch_dense_krylov(dense_[k]->plan, a, ctx_->stream);
  if (pr) {
    pr->mark(ctx_->stream);
    pr->mark(ctx_->stream);
  }
  ctx_->launches += 1;
  return 0;
}

// The cross-CTA partials are written and re-read by every CTA after every grid
// barrier; which physical pages they land on moves an inner iteration between
// ~22 and ~29 us on B200 (measured by shifting only this buffer, DESIGN.md
// §4.4).  Physical placement is not controllable, so it is tuned: 8 candidate
// buffers, each timed on a fixed 40-iteration inner solve of a synthetic rhs,
// the fastest kept.  Numerics do not depend on the choice.
void Method::tune_dense_partials(size_t k) {
  if (std::getenv("RMG_DENSE_NO_TUNE") != nullptr) return;
  DenseInner& d = *dense_[k];
  cudaStream_t s = ctx_->stream;
  const int64_t n = level_matrix(k).f();
  const char* tn = std::getenv("RMG_DENSE_TUNE_N");  // candidate buffers (default 8)
  const int kCand = tn != nullptr ? std::max(1, std::min(64, std::atoi(tn))) : 8;
  const size_t count = d.partials.size();
  std::vector<DBuf<double>> cand;
  cand.push_back(std::move(d.partials));
  for (int c = 1; c < kCand; ++c) {
    cand.emplace_back();
    cand.back().alloc(count);
  }
  DBuf<double> b(std::max<int64_t>(1, n));
  launch_fill(b.get(), 1.0, n, s);
  cudaEvent_t e0, e1;
  RMG_CK(cudaEventCreate(&e0));
  RMG_CK(cudaEventCreate(&e1));
  std::vector<float> best_ms(kCand, 1e30f);
  for (int rep = 0; rep < 3; ++rep) {
    for (int c = 0; c < kCand; ++c) {
      d.partials = std::move(cand[c]);
      DenseKrylovArgs a = dense_args(k, b.get());
      a.tol = 0.0;
      a.max_iters = 40;
      a.timing = nullptr;
      RMG_CK(cudaEventRecord(e0, s));
      launch_dense_krylov(d.plan, a, s);
      RMG_CK(cudaEventRecord(e1, s));
      RMG_CK(cudaEventSynchronize(e1));
      float ms = 0.f;
      RMG_CK(cudaEventElapsedTime(&ms, e0, e1));
      best_ms[c] = std::min(best_ms[c], ms);
      cand[c] = std::move(d.partials);
    }
  }
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  const int best = static_cast<int>(std::min_element(best_ms.begin(), best_ms.end()) - best_ms.begin());
  d.partials = std::move(cand[best]);
  d.tuned_ms.assign(best_ms.begin(), best_ms.end());
  d.tuned_pick = best;
  if (std::getenv("RMG_DENSE_TUNE_LOG") != nullptr) {
    std::fprintf(stderr, "[rmg] level %zu partials placement (ms / 40 it):", k);
    for (int c = 0; c < kCand; ++c) std::fprintf(stderr, " %.3f%s", best_ms[c], c == best ? "*" : "");
    std::fprintf(stderr, "\n");
  }
}

const std::vector<int64_t>& Method::labels(size_t k) const {
  if (k >= labels_.size()) throw InvalidArgument("level index out of range");
  return labels_[k];
}

// TwoLevelPreconditioner::apply (krylov.cpp:379-420)
uint64_t Method::precond(size_t k, const double* r, double* z) {
  CoarseLevelDev& c = *coarse_[k];
  const size_t L = coarse_.size();
  const int64_t nc = c.mat->f(), nf = level_matrix(k).f();
  cudaStream_t s = ctx_->stream;
  double* rc = (k + 1 == L) ? rc_last_.get() : work_[k + 1]->b.get();
  {  // r_c = P^T r as a segmented CSR pass (coarsening.cpp:43-55)
    XtArgs ra;
    ra.t = r;
    ra.out = rc;
    launch_xt(c.pt.view, c.pt_sched.view, Epi::Plain, ra, s);
  }
  const double* ec;
  uint64_t inner = 0;
  if (k + 1 == L) {
    launch_dense_gemv(ainv_.get(), rc, ec_last_.get(), nc, nullptr, s);
    ec = ec_last_.get();
    ctx_->launches += 2;
  } else {
    ctx_->launches += 1;
    if (dense_[k + 1])
      inner = run_dense(k + 1, rc);
    else
      inner = specs_[k].spec.coarse_kind == RMG_COARSE_INNER_FCG ? run_fcg(k + 1, rc, false, nullptr)
                                                                  : run_cg(k + 1, rc, nullptr, false, nullptr);
    ec = work_[k + 1]->x.get();
  }
  double* z1 = work_[k]->z1.get();
  launch_prolong(c.label.get(), c.weight.get(), ec, z1, nf, nullptr, s);
  ctx_->launches += 1;
  XtArgs a;
  a.v = z1;
  a.r = r;
  a.out = z;
  a.beta = level_beta(k);
  a.omega = omega_[k];
  level_matrix(k).apply(z1, Epi::Rich, a, prof(k));
  return inner;
}

namespace {
using Clock = std::chrono::steady_clock;
double secs(Clock::time_point t0) { return std::chrono::duration<double>(Clock::now() - t0).count(); }

void record(Context* ctx, KrylovWork& w, const KrylovScalars& hs, const std::vector<uint64_t>& inner,
            Clock::time_point t0, SolveResult* out) {
  out->wall = secs(t0);
  out->iterations = static_cast<uint64_t>(hs.it);
  out->converged = hs.converged != 0;
  out->final_rel = hs.rel;
  const size_t nh = hs.it == 0 && hs.converged ? 1 : static_cast<size_t>(hs.it);
  out->hist.resize(nh);
  if (nh) RMG_CK(cudaMemcpyAsync(out->hist.data(), w.hist.get(), nh * 8, cudaMemcpyDeviceToHost, ctx->stream));
  ctx->sync();
  out->inner = inner;
}
}  // namespace

// one outer FCG iteration at level k (krylov.cpp:185-220): the launch sequence the
// graph loop captures
void Method::fcg_iteration(size_t k) {
  KrylovWork& w = *work_[k];
  Matrix& m = level_matrix(k);
  const int64_t n = m.f();
  cudaStream_t s = ctx_->stream;
  const bool nested = k + 1 < coarse_.size() + 0 && k + 1 < work_.size();
  KrylovWork* iw = nested ? work_[k + 1].get() : nullptr;
  precond(k, w.r.get(), w.z.get());
  if (iw) {
    launch_copy_inner_count(iw->sc.get(), w.sc.get(), w.inner_hist.get(), s);
    ctx_->launches += 1;
  }
  launch_fcg_gs(w.z.get(), w.ap_ring.get(), w.p_ring.get(), n, w.sc.get(), w.vw, s);
  XtArgs a;
  a.v = w.p_ring.get();
  a.r = w.r.get();
  a.out = w.ap_ring.get();
  a.beta = level_beta(k);
  a.sc = w.sc.get();
  a.ring_stride = static_cast<int>(n);
  m.apply_ring(w.p_ring.get(), static_cast<int>(n), w.sc.get(), Epi::Fcg, a, prof(k));
  launch_fcg_axpy(w.x.get(), w.r.get(), w.p_ring.get(), w.ap_ring.get(), n, w.sc.get(), w.hist.get(), w.vw, s);
  ctx_->launches += 3;
}

bool Method::build_fcg_graph() {
  if (std::getenv("RMG_NO_GRAPH") != nullptr) return false;
  for (size_t k = 0; k < coarse_.size(); ++k)  // NCCL collectives stay outside graphs here
    if (level_matrix(k).comm != nullptr) return false;
  auto gl = std::make_unique<GraphLoop>();
  gl->passes.alloc(1);
  if (!capture_while_graph(ctx_, &work_[0]->sc.get()->done, [&] { fcg_iteration(0); }, &gl->g, &gl->exec,
                           &gl->launches_per_iter, gl->passes.get(), solver.max_iters + 2))
    return false;
  fcg_graph_ = std::move(gl);
  return true;
}

// fcg (krylov.cpp:159-227) at level k with the level-k preconditioner
uint64_t Method::run_fcg(size_t k, const double* rhs, bool rec, SolveResult* out) {
  KrylovWork& w = *work_[k];
  Matrix& m = level_matrix(k);
  const int64_t n = m.f();
  cudaStream_t s = ctx_->stream;
  const auto t0 = Clock::now();
  launch_krylov_begin(rhs, w.x.get(), w.r.get(), n, w.sc.get(), w.hist.get(), w.vw, s);
  ctx_->launches += 1;
  KrylovScalars hs = ctx_->read(w.sc.get());
  if (hs.status == 3) throw InvalidArgument("fcg: non-finite rhs");
  std::vector<uint64_t> inner;
  const bool nested = k + 1 < coarse_.size() + 0 && k + 1 < work_.size();
  KrylovWork* iw = nested ? work_[k + 1].get() : nullptr;
  KrylovScalars ihs{};
  // outer loop on the device (one CUDA graph launch) when every inner level runs
  // without the host: the persistent dense solver or the direct coarsest solve
  const bool graphable = k == 0 && !profiling_ && (!nested || (dense_.size() > 1 && dense_[1] != nullptr));
  if (!hs.done && graphable && (fcg_graph_ || build_fcg_graph())) {
    RMG_CK(cudaMemsetAsync(fcg_graph_->passes.get(), 0, sizeof(unsigned long long), s));
    RMG_CK(cudaGraphLaunch(fcg_graph_->exec, s));
    if (iw)
      ctx_->read2(w.sc.get(), &hs, iw->sc.get(), &ihs);
    else
      hs = ctx_->read(w.sc.get());
    ctx_->launches += fcg_graph_->launches_per_iter * static_cast<uint64_t>(std::max(1, hs.it));
    if (hs.status >= 101 && hs.status <= 103) {
      const int st = hs.status - 100;
      if (st == 3) throw InvalidArgument("fcg: non-finite rhs in the level-" + std::to_string(k + 1) + " inner solve");
      throw RuntimeError(std::string(st == 1 ? "fcg: breakdown, <p, Ap> = 0" : "fcg: <p, Ap> <= 0") +
                         " at iteration " + std::to_string(ihs.it) + " of the level-" + std::to_string(k + 1) +
                         " inner solve; operator is not positive definite");
    }
    if (hs.status == 1) throw RuntimeError("fcg: breakdown, <p, Ap> = 0 at iteration " + std::to_string(hs.it));
    if (hs.status == 2)
      throw RuntimeError("fcg: <p, Ap> < 0 at iteration " + std::to_string(hs.it) +
                         "; operator is not positive definite");
  }
  while (!hs.done) {
    fcg_iteration(k);
    if (iw) {
      ctx_->read2(w.sc.get(), &hs, iw->sc.get(), &ihs);
      if (ihs.status == 1 || ihs.status == 2)
        throw RuntimeError(std::string(ihs.status == 1 ? "fcg: breakdown, <p, Ap> = 0" : "fcg: <p, Ap> <= 0") +
                           " at iteration " + std::to_string(ihs.it) + " of the level-" + std::to_string(k + 1) +
                           " inner solve; operator is not positive definite");
      if (ihs.status == 3) throw InvalidArgument("fcg: non-finite rhs in the level-" + std::to_string(k + 1) + " inner solve");
    } else {
      hs = ctx_->read(w.sc.get());
    }
    if (profiling_) collect_profiles();
    if (hs.status == 1) throw RuntimeError("fcg: breakdown, <p, Ap> = 0 at iteration " + std::to_string(hs.it));
    if (hs.status == 2)
      throw RuntimeError("fcg: <p, Ap> < 0 at iteration " + std::to_string(hs.it) +
                         "; operator is not positive definite");
  }
  if (rec) {
    if (iw && hs.it > 0) {
      inner.resize(static_cast<size_t>(hs.it));
      RMG_CK(cudaMemcpyAsync(inner.data(), w.inner_hist.get(), inner.size() * sizeof(uint64_t),
                             cudaMemcpyDeviceToHost, s));
    } else if (hs.it > 0) {
      inner.assign(static_cast<size_t>(hs.it), 0);  // direct coarse solve: zero inner iterations
    }
    record(ctx_, w, hs, inner, t0, out);
  }
  return static_cast<uint64_t>(hs.it);
}

// fgmres (krylov.cpp:229-328), full flexible GMRES with the level-0 two-level
// preconditioner.  Device: preconditioner, operator, the MGS sweep (one
// cooperative launch per iteration, fgmres.cu), v_{j+1} = w / h_{j+1,j} and the
// final x = sum y_j z_j.  Host: the reference's Givens rotations, residual
// estimate and back substitution on the j + 2 Hessenberg entries per iteration.
uint64_t Method::run_fgmres(const double* rhs, SolveResult* out) {
  KrylovWork& w = *work_[0];
  Matrix& m = level_matrix(0);
  const int64_t n = m.f();
  cudaStream_t s = ctx_->stream;
  const auto t0 = Clock::now();
  launch_krylov_begin(rhs, w.x.get(), w.r.get(), n, w.sc.get(), w.hist.get(), w.vw, s);  // x = 0, ||rhs||
  ctx_->launches += 1;
  const KrylovScalars hs0 = ctx_->read(w.sc.get());
  if (hs0.status == 3) throw InvalidArgument("fgmres: non-finite rhs");
  const double nrhs = hs0.nb;
  out->inner.clear();
  out->hist.clear();
  out->iterations = 0;
  out->converged = false;
  if (nrhs == 0.0) {
    out->converged = true;
    out->hist.push_back(0.0);
    out->final_rel = 0.0;
    out->wall = secs(t0);
    return 0;
  }
  const uint64_t maxit = solver.max_iters;
  const size_t need_basis = static_cast<size_t>(maxit + 1) * std::max<int64_t>(1, n);
  if (gm_basis_.size() < need_basis) {
    gm_basis_.alloc(need_basis);
    gm_z_.alloc(static_cast<size_t>(std::max<uint64_t>(1, maxit)) * std::max<int64_t>(1, n));
    gm_h_.alloc(static_cast<size_t>(maxit + 2));
    gm_part_.alloc(static_cast<size_t>(2 * mgs_grid(n)));
  }
  double* wv = w.r.get();  // w = A z_j, orthogonalized in place
  // v_0 = rhs / ||rhs|| (KrylovScalars::nb on the device)
  launch_div(gm_basis_.get(), rhs, &w.sc.get()->nb, n, s);
  std::vector<std::vector<double>> hess;
  std::vector<double> giv_c, giv_s, g{nrhs}, h;
  uint64_t k = 0;
  for (uint64_t j = 0; j < maxit; ++j) {
    double* vj = gm_basis_.get() + static_cast<size_t>(j) * n;
    double* zj = gm_z_.get() + static_cast<size_t>(j) * n;
    out->inner.push_back(precond(0, vj, zj));
    XtArgs a;
    a.v = zj;
    a.out = wv;
    a.beta = level_beta(0);
    m.apply(zj, Epi::Axpby, a, prof(0));
    launch_mgs(wv, gm_basis_.get(), n, static_cast<int>(j), gm_h_.get(), gm_part_.get(), s);
    ctx_->launches += 2;
    h.assign(j + 2, 0.0);
    RMG_CK(cudaMemcpyAsync(h.data(), gm_h_.get(), (j + 2) * sizeof(double), cudaMemcpyDeviceToHost, s));
    ctx_->sync();
    if (profiling_) collect_profiles();
    const double h_next = h[j + 1];
    for (uint64_t i = 0; i < j; ++i) {  // previously accumulated rotations
      const double tmp = giv_c[i] * h[i] + giv_s[i] * h[i + 1];
      h[i + 1] = -giv_s[i] * h[i] + giv_c[i] * h[i + 1];
      h[i] = tmp;
    }
    const double denom = std::hypot(h[j], h[j + 1]);
    const double c = denom == 0.0 ? 1.0 : h[j] / denom;
    const double sn = denom == 0.0 ? 0.0 : h[j + 1] / denom;
    giv_c.push_back(c);
    giv_s.push_back(sn);
    h[j] = denom;
    h[j + 1] = 0.0;
    g.push_back(-sn * g[j]);
    g[j] = c * g[j];
    hess.push_back(h);
    k = j + 1;
    const double rel = std::abs(g[j + 1]) / nrhs;
    out->hist.push_back(rel);
    out->iterations = k;
    out->final_rel = rel;
    if (rel <= solver.tol || h_next == 0.0) {  // converged, or happy breakdown
      out->converged = true;
      break;
    }
    launch_div(gm_basis_.get() + static_cast<size_t>(j + 1) * n, wv, gm_h_.get() + j + 1, n, s);
    ctx_->launches += 1;
  }
  std::vector<double> y(k, 0.0);  // back substitution on the rotated triangle
  for (uint64_t i = k; i-- > 0;) {
    double acc = g[i];
    for (uint64_t jj = i + 1; jj < k; ++jj) acc -= hess[jj][i] * y[jj];
    const double diag = hess[i][i];
    if (diag == 0.0)
      throw RuntimeError("fgmres: rank-deficient Hessenberg system at column " + std::to_string(i));
    y[i] = acc / diag;
  }
  if (k > 0) {
    DBuf<double> yd(k);
    yd.upload(y.data(), k, s);
    launch_combine(w.x.get(), gm_z_.get(), yd.get(), static_cast<int>(k), n, s);
    ctx_->launches += 1;
    ctx_->sync();
  }
  out->wall = secs(t0);
  return k;
}

// cg (krylov.cpp:94-157), optionally Jacobi-preconditioned
uint64_t Method::run_cg(size_t k, const double* rhs, const double* inv, bool rec, SolveResult* out) {
  KrylovWork& w = *work_[k];
  Matrix& m = level_matrix(k);
  const int64_t n = m.f();
  cudaStream_t s = ctx_->stream;
  double* p = w.p_ring.get();
  double* ap = w.ap_ring.get();
  double* z = inv ? w.z.get() : w.r.get();
  const auto t0 = Clock::now();
  launch_cg_begin(rhs, inv, w.x.get(), w.r.get(), w.z.get(), p, n, w.sc.get(), w.hist.get(), w.vw, s);
  ctx_->launches += 1;
  KrylovScalars hs = ctx_->read(w.sc.get());
  if (hs.status == 3) throw InvalidArgument("cg: non-finite rhs");
  auto iteration = [&] {
    cudaStream_t cs = ctx_->stream;  // the capture stream while a graph is recorded
    XtArgs a;
    a.v = p;
    a.out = ap;
    a.beta = level_beta(k);
    a.sc = w.sc.get();
    a.done = &w.sc.get()->done;
    m.apply(p, Epi::Cg, a, prof(k));
    launch_cg_axpy(w.x.get(), w.r.get(), w.z.get(), inv, p, ap, n, w.sc.get(), w.hist.get(), w.vw, cs);
    launch_cg_update_p(p, z, n, w.sc.get(), cs);
    ctx_->launches += 2;
  };
  // level 0 (cg, jacobi_cg): the loop as a CUDA graph (§4.13)
  if (!hs.done && k == 0 && !profiling_ && std::getenv("RMG_NO_GRAPH") == nullptr && m.comm == nullptr) {
    GraphLoop* gl = inv ? cg_graph_[1].get() : cg_graph_[0].get();
    if (gl == nullptr) {
      auto g = std::make_unique<GraphLoop>();
      g->passes.alloc(1);
      if (capture_while_graph(ctx_, &w.sc.get()->done, iteration, &g->g, &g->exec, &g->launches_per_iter,
                              g->passes.get(), w.max_iters + 2)) {
        gl = g.get();
        cg_graph_[inv ? 1 : 0] = std::move(g);
      }
    }
    if (gl != nullptr) {
      RMG_CK(cudaMemsetAsync(gl->passes.get(), 0, sizeof(unsigned long long), s));
      RMG_CK(cudaGraphLaunch(gl->exec, s));
      hs = ctx_->read(w.sc.get());
      ctx_->launches += gl->launches_per_iter * static_cast<uint64_t>(std::max(1, hs.it));
      if (hs.status == 2)
        throw RuntimeError("cg: <p, Ap> = " + std::to_string(hs.pap) + " at iteration " + std::to_string(hs.it) +
                           "; operator is not positive definite");
    }
  }
  while (!hs.done) {
    iteration();
    hs = ctx_->read(w.sc.get());
    if (profiling_) collect_profiles();
    if (hs.status == 2)
      throw RuntimeError("cg: <p, Ap> = " + std::to_string(hs.pap) + " at iteration " + std::to_string(hs.it) +
                         "; operator is not positive definite");
  }
  if (rec) record(ctx_, w, hs, {}, t0, out);
  return static_cast<uint64_t>(hs.it);
}

SolveResult Method::solve_rhs(const double* rhs, double* w_out) {
  RMG_CK(cudaSetDevice(ctx_->device));
  SolveResult res;
  if (kind_ == RMG_METHOD_CG)
    run_cg(0, rhs, nullptr, true, &res);
  else if (kind_ == RMG_METHOD_JACOBI_CG)
    run_cg(0, rhs, inv_diag_.get(), true, &res);
  else if (kind_ == RMG_METHOD_FGMRES_TWOLEVEL)
    run_fgmres(rhs, &res);
  else if (vc_kind())
    run_pcg_vcycle(rhs, &res);
  else
    run_fcg(0, rhs, true, &res);
  const int64_t n = fine_->f();
  if (n) RMG_CK(cudaMemcpyAsync(w_out, work_[0]->x.get(), n * 8, cudaMemcpyDeviceToDevice, ctx_->stream));
  return res;
}

void Method::set_profiling(bool on) {
  profiling_ = on;
  while (prof_.size() < static_cast<size_t>(n_levels())) prof_.push_back(std::make_unique<OpProfile>());
  for (auto& p : prof_) p->reset();
}

void Method::collect_profiles() {
  for (auto& p : prof_) p->collect();
}

void Method::precondition(const double* r, double* z) {
  if (coarse_.empty()) throw InvalidArgument("precondition: method has no hierarchy");
  if (vc_kind())
    vcycle(0, r, z, nullptr);
  else
    precond(0, r, z);
}

// ---------------------------------------------------------------- pcg_vcycle
// Damped Jacobi at every level above the coarsest: D_k = diag(X_k^T X_k) + beta_k
// (gram_diagonal, ridge.cpp:30-37), weight 1.4 / lambda_max(D_k^-1 A_k) by 30 power
// steps from CounterRng(0x5eed + 64 + k) normals (underestimates lambda_max by a
// little, so w lambda_max stays just above 1, inside (0, 2)).
void Method::build_vcycle() {
  cudaStream_t s = ctx_->stream;
  const size_t L = coarse_.size();
  if (vc_graph_) vc_graph_retired_ = std::move(vc_graph_);  // its kernels point at the buffers rebuilt here
  vc_.clear();
  if (!dg_built_) build_dense_grams();  // beta-free: built once, kept across set_beta
  for (size_t k = 0; k < L; ++k) {
    Matrix& m = level_matrix(k);
    const int64_t n = m.f();
    auto v = std::make_unique<VcLevel>();
    const size_t nn = static_cast<size_t>(std::max<int64_t>(1, n));
    v->dinv.alloc(nn);
    v->x1.alloc(nn);
    v->y.alloc(nn);
    v->e.alloc(nn);
    m.gram_diagonal(level_beta(k), v->x1.get());
    std::vector<double> d(n);
    if (n) RMG_CK(cudaMemcpyAsync(d.data(), v->x1.get(), n * 8, cudaMemcpyDeviceToHost, s));
    ctx_->sync();
    for (double& e : d) {
      if (!(e > 0.0)) throw InvalidArgument("pcg_vcycle: Jacobi diagonal must be positive");
      e = 1.0 / e;
    }
    v->dinv.upload(d.data(), d.size(), s);
    if (vc_additive(k)) {  // the additive level applies D^-1 itself (weight 1, no smoothing step)
      v->w = 1.0;
      vc_.push_back(std::move(v));
      continue;
    }
    CounterRng rng(0x5eed + 64 + k);
    std::vector<double> h(n);
    for (double& e : h) e = rng.next_normal();
    double lam = 0.0;
    for (int it = 0; it < 30 && n > 0; ++it) {
      double nv = 0.0;
      for (double e : h) nv += e * e;
      nv = std::sqrt(nv);
      if (nv == 0.0) break;
      for (double& e : h) e /= nv;
      lam = nv;
      v->x1.upload(h.data(), h.size(), s);
      XtArgs a;
      a.v = v->x1.get();
      a.out = v->y.get();
      a.beta = level_beta(k);
      if (const DenseGram* dg = dgram(k))
        launch_gram_gemv(dg->G.get(), dg->ld, v->x1.get(), level_beta(k), v->y.get(), n, nullptr, s);
      else
        m.apply(v->x1.get(), Epi::Axpby, a);
      launch_vc_pre(v->y.get(), v->dinv.get(), 1.0, v->e.get(), n, nullptr, s);  // D^-1 A v
      RMG_CK(cudaMemcpyAsync(h.data(), v->e.get(), n * 8, cudaMemcpyDeviceToHost, s));
      ctx_->sync();
    }
    {
      double nv = 0.0;
      for (double e : h) nv += e * e;
      lam = std::sqrt(nv);
    }
    if (!(lam > 0.0)) throw RuntimeError("pcg_vcycle: Jacobi power iteration collapsed");
    // w = 1.4 / lambda: the cycle stays SPD while w lambda_max < 2, and the 30 power
    // steps underestimate lambda_max by a few percent at most (measured on cfg 3:
    // 1.0 -> 1.4 takes 10.06 -> 9.67 ms per right-hand side; 1.7 gains nothing more);
    // RMG_VC_OMEGA_SCALE overrides
    static const double scale = [] {
      const char* e = std::getenv("RMG_VC_OMEGA_SCALE");
      return e != nullptr ? std::atof(e) : 1.4;
    }();
    v->w = scale / lam;
    vc_.push_back(std::move(v));
  }
}

// z = M_k r: pre-smooth from zero, coarse correction (the next level's cycle, or the
// coarsest direct solve), post-smooth -- symmetric, so plain PCG applies.
void Method::vcycle(size_t k, const double* r, double* z, const int32_t* done) {
  cudaStream_t s = ctx_->stream;
  const size_t L = coarse_.size();
  CoarseLevelDev& c = *coarse_[k];
  Matrix& m = level_matrix(k);
  const int64_t nf = m.f();
  VcLevel& v = *vc_[k];
  const bool last = k + 1 == L;
  double* rc = last ? rc_last_.get() : work_[k + 1]->b.get();
  double* ec = last ? ec_last_.get() : work_[k + 1]->x.get();
  if (vc_additive(k)) {  // z = D^-1 r + P V_{k+1}(P^T r): no operator application at this level
    XtArgs ra;
    ra.t = r;
    ra.out = rc;
    ra.done = done;
    launch_xt(c.pt.view, c.pt_sched.view, Epi::Plain, ra, s);
    if (last)
      launch_dense_gemv(ainv_.get(), rc, ec, c.mat->f(), done, s);
    else
      vcycle(k + 1, rc, ec, done);
    launch_vc_jacobi_prolong(r, v.dinv.get(), c.label.get(), c.weight.get(), ec, z, nf, done, s);
    ctx_->launches += 3;
    return;
  }
  launch_vc_pre(r, v.dinv.get(), v.w, v.x1.get(), nf, done, s);
  XtArgs a;
  a.v = v.x1.get();
  a.out = v.y.get();
  a.beta = level_beta(k);
  a.done = done;
  const DenseGram* dg = dgram(k);
  if (dg != nullptr)
    launch_gram_gemv(dg->G.get(), dg->ld, v.x1.get(), level_beta(k), v.y.get(), nf, done, s);
  else
    m.apply(v.x1.get(), Epi::Axpby, a, prof(k));
  launch_vc_sub(r, v.y.get(), nf, done, s);  // y = r - A x1
  XtArgs ra;
  ra.t = v.y.get();
  ra.out = rc;
  ra.done = done;
  launch_xt(c.pt.view, c.pt_sched.view, Epi::Plain, ra, s);
  if (last)
    launch_dense_gemv(ainv_.get(), rc, ec, c.mat->f(), done, s);
  else
    vcycle(k + 1, rc, ec, done);
  launch_prolong(c.label.get(), c.weight.get(), ec, v.e.get(), nf, done, s);
  launch_vc_add(v.x1.get(), v.e.get(), nf, done, s);  // e = x2
  a.v = v.e.get();
  a.out = v.y.get();
  if (dg != nullptr)
    launch_gram_gemv(dg->G.get(), dg->ld, v.e.get(), level_beta(k), v.y.get(), nf, done, s);
  else
    m.apply(v.e.get(), Epi::Axpby, a, prof(k));
  launch_vc_post(v.e.get(), r, v.y.get(), v.dinv.get(), v.w, z, nf, done, s);
  ctx_->launches += 8;
}

bool Method::block_capable() const {
  if (fine_->comm != nullptr) return false;
  if (kind_ == RMG_METHOD_CG || kind_ == RMG_METHOD_JACOBI_CG) return true;
  if (!vc_kind() || coarse_.empty()) return false;
  for (size_t k = 1; k < coarse_.size(); ++k) {
    if (dgram(k) != nullptr || vc_additive(k)) continue;  // an additive level applies no operator
    const Matrix& m = level_matrix(k);
    if (m.dense != nullptr || m.comm != nullptr) return false;
  }
  return true;
}

void Method::bprecond(const double* r, double* z, int k) {
  cudaStream_t s = ctx_->stream;  // the capture stream while a graph is recorded
  const int64_t n = fine_->f();
  if (vc_kind()) {
    bvcycle(0, r, z, k);
  } else if (kind_ == RMG_METHOD_JACOBI_CG) {  // z = r * (1/d) (krylov.cpp:41-47)
    launch_bvc_pre(r, inv_diag_.get(), 1.0, z, n, k, s);
    ctx_->launches += 1;
  } else {  // IdentityPreconditioner (krylov.cpp:34-39)
    RMG_CK(cudaMemcpyAsync(z, r, static_cast<size_t>(n) * k * sizeof(double), cudaMemcpyDeviceToDevice, s));
  }
}

// the V-cycle of vcycle() on k columns at once (row-major blocks; every operator
// application is one block operator call)
void Method::bvcycle(size_t lv, const double* r, double* z, int k) {
  cudaStream_t s = ctx_->stream;
  const size_t L = coarse_.size();
  CoarseLevelDev& c = *coarse_[lv];
  Matrix& m = level_matrix(lv);
  const int64_t nf = m.f(), nc = c.mat->f();
  VcLevel& v = *vc_[lv];
  while (bl_.size() <= lv) bl_.push_back(std::make_unique<BlockLevel>());
  BlockLevel& b = *bl_[lv];
  const size_t nfk = static_cast<size_t>(std::max<int64_t>(1, nf)) * k, nck = static_cast<size_t>(std::max<int64_t>(1, nc)) * k;
  if (b.x1.size() < nfk) {
    b.x1.alloc(nfk);
    b.y.alloc(nfk);
    b.e.alloc(nfk);
  }
  if (b.rc.size() < nck) {
    b.rc.alloc(nck);
    b.ec.alloc(nck);
  }
  const DenseGram* dg = dgram(lv);
  auto apply = [&](const double* in, double* out) {
    if (dg != nullptr)
      launch_gram_gemm(dg->G.get(), dg->ld, in, level_beta(lv), out, nf, k, dg->scratch.get(), s);
    else
      m.apply_block(in, out, level_beta(lv), k, false);
  };
  if (vc_additive(lv)) {  // z = D^-1 r + P V_{lv+1}(P^T r)
    launch_brestrict(c.mptr.get(), c.members.get(), c.weight.get(), r, b.rc.get(), nc, k, s);
    if (lv + 1 == L)
      launch_bgemm_inv(ainv_.get(), b.rc.get(), b.ec.get(), nc, k, s);
    else
      bvcycle(lv + 1, b.rc.get(), b.ec.get(), k);
    if (lv == 0 && brz_partial_ != nullptr) {  // the PCG loop's <r, z> rides on this pass
      launch_bvc_jacobi_prolong_dot(r, v.dinv.get(), c.label.get(), c.weight.get(), b.ec.get(), z, nf, k, brz_partial_,
                                    brz_g_, brz_out_, s);
      brz_done_ = true;
    } else {
      launch_bvc_jacobi_prolong(r, v.dinv.get(), c.label.get(), c.weight.get(), b.ec.get(), z, nf, k, s);
    }
    ctx_->launches += 3;
    return;
  }
  launch_bvc_pre(r, v.dinv.get(), v.w, b.x1.get(), nf, k, s);
  apply(b.x1.get(), b.y.get());
  launch_bsub(r, b.y.get(), nf * k, s);
  launch_brestrict(c.mptr.get(), c.members.get(), c.weight.get(), b.y.get(), b.rc.get(), nc, k, s);
  if (lv + 1 == L)
    launch_bgemm_inv(ainv_.get(), b.rc.get(), b.ec.get(), nc, k, s);
  else
    bvcycle(lv + 1, b.rc.get(), b.ec.get(), k);
  launch_bprolong(c.label.get(), c.weight.get(), b.ec.get(), b.e.get(), nf, k, s);
  launch_badd(b.x1.get(), b.e.get(), nf * k, s);
  apply(b.e.get(), b.y.get());
  launch_bvc_post(b.e.get(), r, b.y.get(), v.dinv.get(), v.w, z, nf, k, s);
  ctx_->launches += 10;
}

// One lock-step iteration of the batched PCG loop (k columns) on the context's stream --
// the capture stream while a graph is recorded.  Works on bw_ (sized by solve_block).
void Method::block_iteration(int k) {
  Matrix& m = *fine_;
  BlockWork& w = bw_;
  const int64_t n = m.f();
  const int g = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(296, (n + 255) / 256)));
  double *rr = w.dots.get(), *rz = rr + 64, *pap = rr + 128;
  cudaStream_t cs = ctx_->stream;
  m.apply_block(w.p.get(), w.ap.get(), level_beta(0), k, false);
  launch_bdots(w.p.get(), w.ap.get(), n, k, w.partial.get(), g, pap, cs);
  launch_bpcg_alpha(w.sc.get(), pap, k, cs);
  // x, r and <r, r> in one pass (the partials are launch_bdots')
  launch_bupdate_xr_dot(w.x.get(), w.r.get(), w.p.get(), w.ap.get(), w.sc.get(), n, k, w.partial.get(), g, rr, cs);
  launch_bpcg_conv(w.sc.get(), rr, k, w.hist.get(), cs);
  brz_partial_ = w.partial.get();  // an additive finest level forms <r, z> while it writes z
  brz_g_ = g;
  brz_out_ = rz;
  brz_done_ = false;
  bprecond(w.r.get(), w.z.get(), k);
  brz_partial_ = nullptr;
  if (!brz_done_) launch_bdots(w.r.get(), w.z.get(), n, k, w.partial.get(), g, rz, cs);
  launch_bpcg_beta(w.sc.get(), rz, k, cs);
  launch_bupdate_p(w.p.get(), w.z.get(), w.sc.get(), n, k, cs);
  ctx_->launches += 12;
}

// The lock-step loop as a CUDA graph (device-side while loop over block_iteration).  Built by
// the first batched solve, and again by set_beta for the k it was built for: beta and the
// rebuilt coarse buffers are baked into the captured nodes, and capture + instantiate (0.3 ms,
// but 4-23 ms in one solve out of three to ten) then never falls inside a solve.
bool Method::build_block_graph(int k) {
  bw_graph_.reset();
  const uint64_t maxit = std::max<uint64_t>(solver.max_iters, 1);
  auto gl = std::make_unique<GraphLoop>();
  gl->passes.alloc(1);
  if (!capture_while_graph(ctx_, nullptr, [&] { block_iteration(k); }, &gl->g, &gl->exec, &gl->launches_per_iter,
                           gl->passes.get(), maxit + 2, bw_.sc.get(), k))
    return false;
  bw_graph_ = std::move(gl);
  bw_graph_k_ = k;
  return true;
}

std::vector<SolveResult> Method::solve_block(const double* b_cm, double* w_cm, int k) {
  if (!block_capable())
    throw InvalidArgument("solve_block: cg, jacobi_cg or pcg_vcycle over a single-GPU matrix only");
  if (k < 1 || k > 64) throw InvalidArgument("solve_block: k must be in [1, 64]");
  RMG_CK(cudaSetDevice(ctx_->device));
  cudaStream_t s = ctx_->stream;
  Matrix& m = *fine_;
  const int64_t n = m.f();
  const uint64_t maxit = std::max<uint64_t>(solver.max_iters, 1);
  const int g = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(296, (n + 255) / 256)));
  BlockWork& w = bw_;
  const size_t nk = static_cast<size_t>(std::max<int64_t>(1, n)) * k;
  if (w.k != k || w.x.size() < nk) {
    w.x.alloc(nk);
    w.r.alloc(nk);
    w.z.alloc(nk);
    w.p.alloc(nk);
    w.ap.alloc(nk);
    w.partial.alloc(static_cast<size_t>(g) * 64);
    w.dots.alloc(4 * 64);
    w.sc.alloc(64);
    w.k = k;
  }
  if (w.hist.size() < (maxit + 1) * k) w.hist.alloc((maxit + 1) * k);
  double *rr = w.dots.get(), *rz = rr + 64, *pap = rr + 128, *bad = rr + 192;
  const auto t0 = Clock::now();
  m.xt_block_cm(b_cm, w.r.get(), k);  // rhs = X^T B, one block pass (row-major F x k)
  RMG_CK(cudaMemsetAsync(w.x.get(), 0, nk * sizeof(double), s));
  std::vector<BlockScalars> hs(k);
  for (auto& e : hs) {
    std::memset(&e, 0, sizeof(e));
    e.tol = solver.tol;
    e.max_iters = static_cast<int32_t>(std::min<uint64_t>(maxit, INT32_MAX));
  }
  RMG_CK(cudaMemcpyAsync(w.sc.get(), hs.data(), k * sizeof(BlockScalars), cudaMemcpyHostToDevice, s));
  launch_bnonfinite(w.r.get(), n, k, bad, s);
  launch_bdots(w.r.get(), w.r.get(), n, k, w.partial.get(), g, rr, s);
  bprecond(w.r.get(), w.z.get(), k);
  launch_bdots(w.r.get(), w.z.get(), n, k, w.partial.get(), g, rz, s);
  launch_bpcg_begin(w.sc.get(), rr, rz, bad, k, w.hist.get(), s);
  RMG_CK(cudaMemcpyAsync(w.p.get(), w.z.get(), nk * sizeof(double), cudaMemcpyDeviceToDevice, s));
  const double beta0 = level_beta(0);
  // layouts and scratch of every block operator, before any graph capture (they allocate and synchronize)
  if (m.dense != nullptr) m.ensure_block_gram();
  m.ensure_block_schedule();
  for (size_t lv = 1; lv < coarse_.size() && vc_kind(); ++lv)  // smoothed coarse levels applied as sparse sweeps
    if (dgram(lv) == nullptr && !vc_additive(lv) && level_matrix(lv).dense == nullptr)
      level_matrix(lv).ensure_block_schedule();
  auto iteration = [&] { block_iteration(k); };
  // the lock-step loop as a CUDA graph (§4.13): runs while any column runs
  bool graph_used = false;
  static const bool ttrace = std::getenv("RMG_SOLVE_TRACE") != nullptr;  // host-side phases of a batched solve
  const auto tt0 = Clock::now();
  auto tt1 = tt0, tt2 = tt0;
  if (std::getenv("RMG_NO_GRAPH") == nullptr) {
    if (!bw_graph_ || bw_graph_k_ != k) build_block_graph(k);
    tt1 = Clock::now();
    if (bw_graph_) {
      RMG_CK(cudaMemsetAsync(bw_graph_->passes.get(), 0, sizeof(unsigned long long), s));
      RMG_CK(cudaGraphLaunch(bw_graph_->exec, s));
      graph_used = true;
    }
    tt2 = Clock::now();
  }
  for (;;) {
    RMG_CK(cudaMemcpyAsync(hs.data(), w.sc.get(), k * sizeof(BlockScalars), cudaMemcpyDeviceToHost, s));
    ctx_->sync();
    bool all = true;
    for (int c = 0; c < k; ++c) {
      if (hs[c].status == 3) throw InvalidArgument("cg: non-finite rhs (right-hand side " + std::to_string(c) + ")");
      if (hs[c].status == 2)
        throw RuntimeError("cg: <p, Ap> = " + std::to_string(hs[c].pap) + " at iteration " + std::to_string(hs[c].it) +
                           " of right-hand side " + std::to_string(c) + "; operator is not positive definite");
      all = all && hs[c].done;
    }
    if (all) break;
    iteration();
  }
  const double wall = secs(t0);
  if (ttrace)
    std::fprintf(stderr, "[rmg solve] enqueue %.2f ms, capture %.2f ms, launch %.2f ms, wait %.2f ms\n",
                 1e3 * std::chrono::duration<double>(tt0 - t0).count(),
                 1e3 * std::chrono::duration<double>(tt1 - tt0).count(),
                 1e3 * std::chrono::duration<double>(tt2 - tt1).count(),
                 1e3 * std::chrono::duration<double>(Clock::now() - tt2).count());
  launch_brow2col(w.x.get(), w_cm, n, k, s);
  int32_t itmax = 0;
  for (const auto& e : hs) itmax = std::max(itmax, e.it);
  if (graph_used) ctx_->launches += bw_graph_->launches_per_iter * static_cast<uint64_t>(std::max(1, itmax));
  std::vector<double> hist(static_cast<size_t>(itmax + 1) * k);
  if (!hist.empty())
    RMG_CK(cudaMemcpyAsync(hist.data(), w.hist.get(), hist.size() * sizeof(double), cudaMemcpyDeviceToHost, s));
  ctx_->sync();
  std::vector<SolveResult> out(k);
  for (int c = 0; c < k; ++c) {
    SolveResult& r = out[c];
    r.wall = wall;
    r.iterations = static_cast<uint64_t>(hs[c].it);
    r.converged = hs[c].converged != 0;
    r.final_rel = hs[c].rel;
    const size_t nh = hs[c].it == 0 && hs[c].converged ? 1 : static_cast<size_t>(hs[c].it);
    r.hist.resize(nh);
    for (size_t i = 0; i < nh; ++i) r.hist[i] = hist[i * k + c];
    r.inner.assign(static_cast<size_t>(hs[c].it), 0);
  }
  return out;
}

// one PCG iteration with the V-cycle (the launch sequence the graph captures)
void Method::pcg_vcycle_iteration() {
  KrylovWork& w = *work_[0];
  Matrix& m = *fine_;
  const int64_t n = m.f();
  cudaStream_t s = ctx_->stream;
  double* p = w.p_ring.get();
  double* ap = w.ap_ring.get();
  double* z = w.z.get();
  const int32_t* done = &w.sc.get()->done;
  XtArgs a;
  a.v = p;
  a.out = ap;
  a.beta = level_beta(0);
  a.sc = w.sc.get();
  a.done = done;
  m.apply(p, Epi::Cg, a, prof(0));
  launch_cg_axpy(w.x.get(), w.r.get(), z, nullptr, p, ap, n, w.sc.get(), w.hist.get(), w.vw, s, true);
  vcycle(0, w.r.get(), z, done);
  launch_pcg_rz(w.r.get(), z, n, w.sc.get(), false, w.vw, s);
  launch_cg_update_p(p, z, n, w.sc.get(), s);
  ctx_->launches += 3;
}

// The while-node graph (CUDA 12.4+ conditional nodes).  Built once per hierarchy /
// beta (the buffers it points at are fixed); false when the runtime refuses it.
bool Method::build_vcycle_graph() {
  if (std::getenv("RMG_NO_GRAPH") != nullptr) return false;
  for (size_t k = 0; k < coarse_.size(); ++k)  // NCCL collectives stay outside graphs here
    if (level_matrix(k).comm != nullptr) return false;
  auto gl = std::make_unique<GraphLoop>();
  gl->passes.alloc(1);
  if (!capture_while_graph(ctx_, &work_[0]->sc.get()->done, [&] { pcg_vcycle_iteration(); }, &gl->g, &gl->exec,
                           &gl->launches_per_iter, gl->passes.get(), solver.max_iters + 2))
    return false;
  vc_graph_ = std::move(gl);
  return true;
}

// PCG (krylov.cpp:94-157) with z = M r the V-cycle
uint64_t Method::run_pcg_vcycle(const double* rhs, SolveResult* out) {
  KrylovWork& w = *work_[0];
  Matrix& m = *fine_;
  const int64_t n = m.f();
  cudaStream_t s = ctx_->stream;
  double* p = w.p_ring.get();
  double* ap = w.ap_ring.get();
  double* z = w.z.get();
  const int32_t* done = &w.sc.get()->done;
  const auto t0 = Clock::now();
  launch_cg_begin(rhs, nullptr, w.x.get(), w.r.get(), z, p, n, w.sc.get(), w.hist.get(), w.vw, s);
  KrylovScalars hs = ctx_->read(w.sc.get());
  if (hs.status == 3) throw InvalidArgument("cg: non-finite rhs");
  if (!hs.done) {
    vcycle(0, w.r.get(), z, done);
    launch_pcg_rz(w.r.get(), z, n, w.sc.get(), true, w.vw, s);
    RMG_CK(cudaMemcpyAsync(p, z, static_cast<size_t>(n) * 8, cudaMemcpyDeviceToDevice, s));
    ctx_->launches += 2;
  }
  if (!hs.done && !profiling_ && (vc_graph_ || build_vcycle_graph())) {
    // the whole iteration loop on the device: one graph launch
    RMG_CK(cudaMemsetAsync(vc_graph_->passes.get(), 0, sizeof(unsigned long long), s));
    RMG_CK(cudaGraphLaunch(vc_graph_->exec, s));
    hs = ctx_->read(w.sc.get());
    ctx_->launches += vc_graph_->launches_per_iter * static_cast<uint64_t>(std::max(1, hs.it));
    if (hs.status == 2)
      throw RuntimeError("cg: <p, Ap> = " + std::to_string(hs.pap) + " at iteration " + std::to_string(hs.it) +
                         "; operator is not positive definite");
  }
  while (!hs.done) {
    pcg_vcycle_iteration();
    hs = ctx_->read(w.sc.get());
    if (profiling_) collect_profiles();
    if (hs.status == 2)
      throw RuntimeError("cg: <p, Ap> = " + std::to_string(hs.pap) + " at iteration " + std::to_string(hs.it) +
                         "; operator is not positive definite");
  }
  if (out) record(ctx_, w, hs, std::vector<uint64_t>(static_cast<size_t>(hs.it), 0), t0, out);
  return static_cast<uint64_t>(hs.it);
}

double Method::time_operator(size_t level, uint64_t reps, bool flush, double* k1_ms, double* k2_ms) {
  if (level >= static_cast<size_t>(n_levels())) throw InvalidArgument("level index out of range");
  Matrix& m = level_matrix(level);
  if (!m.dense) m.ensure_operator();
  cudaStream_t s = ctx_->stream;
  DBuf<double> v(std::max<int64_t>(1, m.f())), out(std::max<int64_t>(1, m.f()));
  launch_fill(v.get(), 1.0, m.f(), s);
  DBuf<char> scratch;
  const size_t flush_bytes = size_t(256) << 20;
  if (flush) scratch.alloc(flush_bytes);
  cudaEvent_t e0, e1, e2;
  RMG_CK(cudaEventCreate(&e0));
  RMG_CK(cudaEventCreate(&e1));
  RMG_CK(cudaEventCreate(&e2));
  double t1 = 0.0, t2 = 0.0;
  XtArgs a;
  a.v = v.get();
  a.out = out.get();
  a.beta = level_beta(level);
  a.t = m.t.get();
  for (uint64_t r = 0; r < reps + 2; ++r) {  // 2 warm-ups
    if (flush) RMG_CK(cudaMemsetAsync(scratch.get(), static_cast<int>(r & 0xff), flush_bytes, s));
    RMG_CK(cudaEventRecord(e0, s));
    if (m.dense)  // fused single sweep: K1 slot = sweep + finish, K2 slot empty
      m.apply(v.get(), Epi::Axpby, a);
    else
      launch_spmv_rows(m.x.view, v.get(), m.t.get(), nullptr, s);
    RMG_CK(cudaEventRecord(e1, s));
    if (m.dense) {
    } else if (m.comm != nullptr) {  // no collective inside a single-rank timing loop
      launch_xt(m.xt.view, m.sched.view, Epi::Axpby, a, s);
    } else {
      xt_pass(m, m.t.get(), Epi::Axpby, a);
    }
    RMG_CK(cudaEventRecord(e2, s));
    RMG_CK(cudaEventSynchronize(e2));
    float a1 = 0.f, a2 = 0.f;
    RMG_CK(cudaEventElapsedTime(&a1, e0, e1));
    RMG_CK(cudaEventElapsedTime(&a2, e1, e2));
    if (r >= 2) {
      t1 += a1;
      t2 += a2;
    }
  }
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaEventDestroy(e2);
  *k1_ms = t1 / static_cast<double>(std::max<uint64_t>(reps, 1));
  *k2_ms = t2 / static_cast<double>(std::max<uint64_t>(reps, 1));
  return *k1_ms + *k2_ms;
}

}  // namespace rmg
