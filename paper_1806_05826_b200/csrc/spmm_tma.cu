// Block-operator gather passes on TMA gather4 (spmm_tma.cuh).
#include <cuda.h>
#include <cudaTypedefs.h>

#include <cstdlib>
#include <cstring>
#include <mutex>
#include <stdexcept>
#include <string>

#include "spmm_tma.cuh"

namespace rmg {
namespace {

constexpr int kTW = 8;        // warps per CTA (one CTA per SM: the stages fill shared memory)
constexpr int kTS = 3;        // pipeline stages per warp
constexpr int kTP = 64;       // entries per piece (16 gather4 instructions)
constexpr int kTCols = 16;    // columns per pass (one 128-byte row)
constexpr size_t kStageRows = static_cast<size_t>(kTP) * kTCols * sizeof(double);  // 8 KB
constexpr size_t kStageVals = kTP * sizeof(double);
constexpr size_t kSmemBytes = static_cast<size_t>(kTW) * kTS * (kStageRows + kStageVals) + kTW * kTS * 8;

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
  asm volatile(
      "{\n .reg .pred p;\n"
      "WAIT_%=:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra WAIT_%=;\n"
      "}\n" ::"r"(bar),
      "r"(parity)
      : "memory");
}

// one warp's walk over its units (unit indices gw, gw + nw, ...), piece by piece
struct PieceIt {
  int ui, row, e0, len, seg, off;
  bool valid;
  __device__ __forceinline__ void load(const int4* __restrict__ units, int n_units) {
    valid = ui < n_units;
    if (valid) {
      const int4 u = units[ui];
      row = u.x;
      e0 = u.y;
      len = u.z - u.y;
      seg = u.w;
    }
    off = 0;
  }
  __device__ __forceinline__ int count() const { return min(kTP, len - off); }
  __device__ __forceinline__ bool last() const { return off + kTP >= len; }
  __device__ __forceinline__ void next(const int4* __restrict__ units, int n_units, int nw) {
    if (!last()) {
      off += kTP;
    } else {
      ui += nw;
      load(units, n_units);
    }
  }
};

// EPI 0: Y[row] = sum (K1).  EPI 1: the chunked X^T epilogue (k_xt_block's).
template <bool PAT, int EPI>
__global__ void __launch_bounds__(kTW * 32, 1)
    k_spmm_tma(const __grid_constant__ CUtensorMap tmap, const int4* __restrict__ units, int n_units,
               const int32_t* __restrict__ idx, const double* __restrict__ val, int c0, int kc,
               double* __restrict__ Y, int ldy, const double* __restrict__ V, double beta, double* __restrict__ seg,
               int first, int last) {
  extern __shared__ __align__(1024) unsigned char smem[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, h = lane >> 4, q = lane & 15;
  double* rows = reinterpret_cast<double*>(smem) + static_cast<size_t>(warp) * kTS * kTP * kTCols;
  double* vals = reinterpret_cast<double*>(smem + static_cast<size_t>(kTW) * kTS * kStageRows) +
                 static_cast<size_t>(warp) * kTS * kTP;
  uint64_t* bars =
      reinterpret_cast<uint64_t*>(smem + static_cast<size_t>(kTW) * kTS * (kStageRows + kStageVals)) + warp * kTS;
  if (lane == 0) {
    for (int s = 0; s < kTS; ++s) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(bars + s)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  }
  __syncwarp();
  const int nw = gridDim.x * kTW;
  PieceIt P, C;  // producer (issues piece p + kTS), consumer (piece p)
  P.ui = C.ui = blockIdx.x * kTW + warp;
  P.load(units, n_units);
  C.load(units, n_units);

  // entry indices / values of the producer's piece: lane l holds entries l, 32 + l
  int ci0 = 0, ci1 = 0;
  double x0 = 0.0, x1 = 0.0;
  auto fetch = [&]() {
    const int cnt = P.count();
    const int b = P.e0 + P.off;
    ci0 = lane < cnt ? idx[b + lane] : -1;
    ci1 = 32 + lane < cnt ? idx[b + 32 + lane] : -1;
    x0 = (PAT || lane >= cnt) ? 1.0 : val[b + lane];
    x1 = (PAT || 32 + lane >= cnt) ? 1.0 : val[b + 32 + lane];
  };
  auto issue = [&](int stage) {
    const int cnt = P.count();
    const int ng = (cnt + 3) >> 2;
    double* sv = vals + stage * kTP;
    sv[lane] = x0;
    sv[32 + lane] = x1;
    // padded slots of the last gather4 repeat entry 0's row (always in bounds)
    const int pad = __shfl_sync(0xffffffffu, ci0, 0);
    const int a0 = ci0 < 0 ? pad : ci0, a1 = ci1 < 0 ? pad : ci1;
    int r[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int s0 = __shfl_sync(0xffffffffu, a0, (4 * lane + j) & 31);
      const int s1 = __shfl_sync(0xffffffffu, a1, (4 * lane + j) & 31);
      r[j] = lane < 8 ? s0 : s1;
    }
    const uint32_t bar = smem_u32(bars + stage);
    if (lane == 0)
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(ng * 4 * kTCols * 8)
                   : "memory");
    __syncwarp();
    if (lane < ng) {
      const uint32_t dst = smem_u32(rows + (static_cast<size_t>(stage) * kTP + 4 * lane) * kTCols);
      asm volatile(
          "cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes"
          " [%0], [%1, {%2, %3, %4, %5, %6}], [%7];" ::"r"(dst),
          "l"(reinterpret_cast<uint64_t>(&tmap)), "r"(c0), "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(bar)
          : "memory");
    }
  };

  // prologue: the first kTS pieces in flight
  int issued = 0;
  for (; issued < kTS && P.valid; ++issued) {
    fetch();
    issue(issued);
    P.next(units, n_units, nw);
  }
  double acc = 0.0;
  for (int p = 0; C.valid; ++p) {
    const int stage = p % kTS;
    const bool more = P.valid;
    if (more) fetch();  // the loads overlap the wait and the consumption below
    mbar_wait(smem_u32(bars + stage), static_cast<uint32_t>((p / kTS) & 1));
    const int cnt = C.count();
    const double* sr = rows + static_cast<size_t>(stage) * kTP * kTCols;
    const double* sv = vals + stage * kTP;
    const int base = h * 32, n_mine = min(32, cnt - base);
#pragma unroll 8
    for (int u = 0; u < n_mine; ++u) {
      const double m = sr[(base + u) * kTCols + q];
      acc = PAT ? acc + m : fma(sv[base + u], m, acc);
    }
    if (C.last()) {
      const double tot = acc + __shfl_xor_sync(0xffffffffu, acc, 16);
      acc = 0.0;
      if (h == 0 && q < kc) {
        if (EPI == 0) {
          Y[static_cast<int64_t>(C.row) * ldy + c0 + q] = tot;
        } else if (C.seg < 0) {
          const int64_t o = static_cast<int64_t>(C.row) * ldy + c0 + q;
          double r = first ? tot : Y[o] + tot;
          if (last) r = r + beta * V[o];
          Y[o] = r;
        } else {
          seg[static_cast<int64_t>(C.seg) * 16 + q] = tot;
        }
      }
    }
    C.next(units, n_units, nw);
    __syncwarp();  // every lane has read the stage before TMA refills it
    if (more) {
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      issue(stage);
      P.next(units, n_units, nw);
    }
  }
  // the barriers' phases are complete (every issued piece was consumed)
}

PFN_cuTensorMapEncodeTiled_v12000 encoder() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q{};
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  });
  if (fn == nullptr) throw std::runtime_error("cuTensorMapEncodeTiled unavailable");
  return fn;
}

CUtensorMap row_map(const double* M, int64_t m_rows, int ld) {
  CUtensorMap map;
  std::memset(&map, 0, sizeof(map));
  const cuuint64_t dims[2] = {static_cast<cuuint64_t>(ld), static_cast<cuuint64_t>(m_rows)};
  const cuuint64_t strides[1] = {static_cast<cuuint64_t>(ld) * sizeof(double)};
  const cuuint32_t box[2] = {kTCols, 1};
  const cuuint32_t estr[2] = {1, 1};
  const CUresult r = encoder()(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, const_cast<double*>(M), dims, strides, box,
                               estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                               CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) throw std::runtime_error("cuTensorMapEncodeTiled failed: " + std::to_string(r));
  return map;
}

int grid_ctas() {
  static int sms = 0;
  if (sms == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (sms <= 0) sms = 148;
  }
  return sms;
}

template <bool PAT, int EPI>
void launch(const TmaSpmm& u, const double* M, int64_t m_rows, int ld, int c0, int kc, double* Y, const double* V,
            double beta, double* seg, int first, int last, cudaStream_t s) {
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(k_spmm_tma<PAT, EPI>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         static_cast<int>(kSmemBytes));
    attr = true;
  }
  const CUtensorMap map = row_map(M, m_rows, ld);
  const int grid = static_cast<int>(std::min<int64_t>(grid_ctas(), (u.n_units + kTW - 1) / kTW));
  k_spmm_tma<PAT, EPI><<<std::max(grid, 1), kTW * 32, kSmemBytes, s>>>(map, u.units, u.n_units, u.idx, u.val, c0, kc,
                                                                      Y, ld, V, beta, seg, first, last);
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) throw std::runtime_error(std::string("spmm_tma: ") + cudaGetErrorString(e));
}

}  // namespace

bool tma_spmm_enabled() {
  const char* e = std::getenv("RMG_BLOCK_TMA");
  return e != nullptr && std::string(e) == "1";
}

bool tma_spmm_ok(const void* m, int ld) {
  return tma_spmm_enabled() && m != nullptr && ld > 0 && ld % 2 == 0 && reinterpret_cast<uintptr_t>(m) % 16 == 0;
}

void launch_spmm_tma_rows(const TmaSpmm& u, const double* M, int64_t m_rows, int ld, int c0, int kc, double* T,
                          cudaStream_t s) {
  if (u.n_units <= 0) return;
  if (u.val == nullptr)
    launch<true, 0>(u, M, m_rows, ld, c0, kc, T, nullptr, 0.0, nullptr, 1, 1, s);
  else
    launch<false, 0>(u, M, m_rows, ld, c0, kc, T, nullptr, 0.0, nullptr, 1, 1, s);
}

void launch_spmm_tma_xt(const TmaSpmm& u, const double* M, int64_t m_rows, int ld, int c0, int kc, double* out,
                        const double* V, double beta, double* seg, int first, int last, cudaStream_t s) {
  if (u.n_units <= 0) return;
  if (u.val == nullptr)
    launch<true, 1>(u, M, m_rows, ld, c0, kc, out, V, beta, seg, first, last, s);
  else
    launch<false, 1>(u, M, m_rows, ld, c0, kc, out, V, beta, seg, first, last, s);
}

}  // namespace rmg
