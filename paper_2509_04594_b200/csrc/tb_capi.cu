// tb_capi.cu — the extern "C" boundary (include/tbgpu.h): launch validation
// with the reference's status codes, variant dispatch, TMA descriptor
// encoding, kernel-only CUDA-event timing, the host-buffer flat entry and the
// cuBLAS DGEMM baseline.
#include <cublas_v2.h>
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <chrono>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <vector>
#include <atomic>
#include <map>
#include <mutex>

#include "../../include/tbgpu.h"
#include "dgemm_dmma.cuh"
#include "dgemm_paper.cuh"

#ifndef TB_VERSION
#define TB_VERSION "tbgpu 0.1.0 (sm_100a)"
#endif

namespace {

// Pipeline shapes (sub-slabs per stage x stages). kProdCfg is the tuned
// default; TB_KCFG=<index> selects another for A/B measurements.
struct KCfg {
  int sub, stages;
};
constexpr KCfg kCfgs[] = {{1, 6}, {1, 7}, {2, 3}};
constexpr int kNumCfgs = sizeof(kCfgs) / sizeof(kCfgs[0]);
constexpr int kProdCfg = 0;

int active_cfg() {
  static const int idx = [] {
    const char* e = std::getenv("TB_KCFG");
    const int v = e ? std::atoi(e) : kProdCfg;
    return (v >= 0 && v < kNumCfgs) ? v : kProdCfg;
  }();
  return idx;
}

template <int SUB, int STAGES>
struct KernelSet {
  static void* tma() { return (void*)tb::dgemm_dmma_kernel<SUB, STAGES, tb::Loader::TMA>; }
  static void* cpasync() { return (void*)tb::dgemm_dmma_kernel<SUB, STAGES, tb::Loader::CPASYNC>; }
  static void* dfma(bool tma) {
    return tma ? (void*)tb::dgemm_dmma_kernel<SUB, STAGES, tb::Loader::TMA, tb::Math::DFMA>
               : (void*)tb::dgemm_dmma_kernel<SUB, STAGES, tb::Loader::CPASYNC, tb::Math::DFMA>;
  }
  static constexpr int smem() { return tb::dmma_smem_bytes<SUB, STAGES>(); }
};

void* cfg_kernel(int idx, bool tma, bool dfma = false) {
  if (dfma) return KernelSet<1, 6>::dfma(tma);  // DFMA comparison variant: one pipeline shape
  switch (idx) {
    case 1: return tma ? KernelSet<1, 7>::tma() : KernelSet<1, 7>::cpasync();
    case 2: return tma ? KernelSet<2, 3>::tma() : KernelSet<2, 3>::cpasync();
    default: return tma ? KernelSet<1, 6>::tma() : KernelSet<1, 6>::cpasync();
  }
}

int cfg_smem(int idx) {
  switch (idx) {
    case 1: return KernelSet<1, 7>::smem();
    case 2: return KernelSet<2, 3>::smem();
    default: return KernelSet<1, 6>::smem();
  }
}

// 64-row tiles for small problems (DmmaCfgT<64>): 24 KB stages, 8 deep.
constexpr int kSmallStages = 8;
void* small_kernel(bool tma) {
  return tma ? (void*)tb::dgemm_dmma_kernel<1, kSmallStages, tb::Loader::TMA, tb::Math::DMMA, 64>
             : (void*)tb::dgemm_dmma_kernel<1, kSmallStages, tb::Loader::CPASYNC, tb::Math::DMMA, 64>;
}
constexpr int small_smem() { return tb::dmma_smem_bytes<1, kSmallStages, 64>(); }

// The host pipeline's fused phase-1 kernel (PIPE mode, dgemm_dmma.cuh).
void* pipe_kernel() { return (void*)tb::dgemm_dmma_kernel<1, 6, tb::Loader::TMA, tb::Math::DMMA, 128, true>; }

// Edge-strip tile shapes (TMA + DMMA): the remainder columns / rows of a
// large product, so the main launch runs on whole 128 x 128 tiles and only a
// narrow strip pads (N = 10000: the last tile column and row had 16 valid
// columns / rows of 128, 2.2 % of all DMMAs on zeros).
enum StripCfg : int {
  kStripNone = 0,
  kStrip128x16,
  kStrip128x32,
  kStrip128x64,
  kStrip16x128,
  kStrip32x128,
  kStrip64x128
};
constexpr int kStripStages = 8;
template <int BM, int BN, int WM>
struct StripK {
  static void* fn() {
    return (void*)tb::dgemm_dmma_kernel<1, kStripStages, tb::Loader::TMA, tb::Math::DMMA, BM, false, BN, WM>;
  }
  static constexpr int smem() { return tb::dmma_smem_bytes<1, kStripStages, BM, BN>(); }
};
struct StripInfo {
  int bm, bn;
  void* fn;
  int smem;
};
StripInfo strip_info(int c) {
  switch (c) {
    case kStrip128x16: return {128, 16, StripK<128, 16, 8>::fn(), StripK<128, 16, 8>::smem()};
    case kStrip128x32: return {128, 32, StripK<128, 32, 8>::fn(), StripK<128, 32, 8>::smem()};
    case kStrip128x64: return {128, 64, StripK<128, 64, 4>::fn(), StripK<128, 64, 4>::smem()};
    case kStrip16x128: return {16, 128, StripK<16, 128, 1>::fn(), StripK<16, 128, 1>::smem()};
    case kStrip32x128: return {32, 128, StripK<32, 128, 1>::fn(), StripK<32, 128, 1>::smem()};
    default: return {0, 0, nullptr, 0};
  }
}

// Tile rows for a DMMA launch (measured, profiles/r01_bm_ab.txt). 64-row
// tiles run ~2 % less efficiently per flop than 128-row tiles (warp tile
// 32 x 32: more fragment loads per DMMA) but double the tile count and can
// halve the row padding:
//  - fewer than two waves of 128-row tiles (and not a >= 90 % single wave,
//    which runs data-parallel): 64 rows — parallelism wins (N = 600 / 1000 /
//    1200 / 1700 / 2000: +33 / +10 / +14 / +5 / +1 %);
//  - otherwise 64 rows only if its padded row count, weighted by that 2 %,
//    is smaller (N = 2223 / 3000 take 64; 4000 / 5000 / 8000 / 10000 and the
//    1250-row shard keep 128).
// TB_BM=64|128 forces (A/B experiments).
int choose_bm(int64_t m, int64_t n, int sms, bool dfma) {
  static const int forced = [] {
    const char* e = std::getenv("TB_BM");
    return e ? std::atoi(e) : 0;
  }();
  if (dfma) return 128;
  if (forced == 64 || forced == 128) return forced;
  const int64_t t128 = ((m + 127) / 128) * ((n + 127) / 128);
  const bool dp_wave = t128 < sms && 10 * t128 >= 9 * (int64_t)sms;  // 128-row DP wave (N = 1500)
  if (t128 < 2 * (int64_t)sms && !dp_wave) return 64;
  const double rows64 = (double)((m + 63) / 64 * 64) * 1.021, rows128 = (double)((m + 127) / 128 * 128);
  return rows64 < rows128 ? 64 : 128;
}
constexpr int kMaxDevices = 64;
constexpr int kMaxBlockThreads = 1024;     // limits.ts:20-24 maxThreadsPerBlock

thread_local char g_err[512] = "";
std::atomic<long long> g_launches{0};  // kernels this library has launched (tb_kernel_launches)

void set_err(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
}

int cuda_fail(cudaError_t e, const char* what) {
  set_err("%s: %s", what, cudaGetErrorString(e));
  return TB_STATUS_RUNTIME;
}

#define TB_CUDA(call, what)                          \
  do {                                               \
    cudaError_t e_ = (call);                         \
    if (e_ != cudaSuccess) return cuda_fail(e_, what); \
  } while (0)

struct DeviceState {
  std::mutex mu;       // device attributes, kernel attributes, cuBLAS handle
  std::mutex host_mu;  // host-buffer entry: workspace + stream
  bool ready = false;
  int sms = 0;
  int smem_optin = 0;
  bool attrs_set = false;
  cublasHandle_t cublas = nullptr;
  cudaStream_t host_stream = nullptr;  // host-buffer entry: compute streams (even / odd row blocks)
  cudaStream_t host_stream2 = nullptr;
  cudaStream_t h2d_stream = nullptr;   // host-buffer entry: host-to-device copies
  cudaStream_t d2h_stream = nullptr;   // host-buffer entry: device-to-host copies
  double* ws = nullptr;                // host-entry device workspace (A | B | C)
  size_t ws_bytes = 0;
  struct SplitWs {                     // stream-K partial tiles + tile counters, per stream
    double* partials = nullptr;
    size_t partial_elems = 0;
    int* counters = nullptr;
    size_t counter_elems = 0;
  };
  std::map<cudaStream_t, SplitWs> split_ws;
  struct StageWs {  // even-pitch copies of misaligned operands (TMA staging), per stream
    double* buf = nullptr;
    size_t elems = 0;
  };
  std::map<cudaStream_t, StageWs> stage_ws;
  std::vector<cudaEvent_t> ev_pool[2];  // host-buffer entry: [timing, no-timing] events
  int* dtab = nullptr;                  // host-buffer entry: [0,128) panel flags, [128,256) panel k-stages
  int* htab = nullptr;                  // pinned: [0,128) zeros, [128,256) panel k-stages, [256] = 1
};

DeviceState g_dev[kMaxDevices];

PFN_cuTensorMapEncodeTiled_v12000 g_encode = nullptr;
std::once_flag g_encode_once;

int device_count_raw() {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  return n;
}

// RAII: switch to `dev` for the call, restore the caller's device after.
struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int dev) {
    if (cudaGetDevice(&prev) != cudaSuccess) prev = -1;
    if (prev != dev) cudaSetDevice(dev);
  }
  ~DeviceGuard() {
    int cur = -1;
    if (prev >= 0 && cudaGetDevice(&cur) == cudaSuccess && cur != prev) cudaSetDevice(prev);
  }
};

int ensure_device(int dev) {
  DeviceState& st = g_dev[dev];
  std::lock_guard<std::mutex> lk(st.mu);
  if (st.ready) return TB_STATUS_OK;
  TB_CUDA(cudaDeviceGetAttribute(&st.sms, cudaDevAttrMultiProcessorCount, dev), "query SM count");
  TB_CUDA(cudaDeviceGetAttribute(&st.smem_optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev),
          "query shared memory opt-in");
  st.ready = true;
  return TB_STATUS_OK;
}

int ensure_kernel_attrs(int dev) {
  DeviceState& st = g_dev[dev];
  std::lock_guard<std::mutex> lk(st.mu);
  if (st.attrs_set) return TB_STATUS_OK;
  for (bool tma : {true, false})
    TB_CUDA(cudaFuncSetAttribute(cfg_kernel(0, tma, true), cudaFuncAttributeMaxDynamicSharedMemorySize, cfg_smem(0)),
            "set smem attribute (dfma)");
  for (int i = 0; i < kNumCfgs; ++i) {
    if (cfg_smem(i) > st.smem_optin) continue;  // validate() rejects the active one if it does not fit
    TB_CUDA(cudaFuncSetAttribute(cfg_kernel(i, true), cudaFuncAttributeMaxDynamicSharedMemorySize, cfg_smem(i)),
            "set smem attribute (dmma_tma)");
    TB_CUDA(cudaFuncSetAttribute(cfg_kernel(i, false), cudaFuncAttributeMaxDynamicSharedMemorySize, cfg_smem(i)),
            "set smem attribute (dmma_cpasync)");
  }
  if (cfg_smem(0) <= st.smem_optin)
    TB_CUDA(cudaFuncSetAttribute(pipe_kernel(), cudaFuncAttributeMaxDynamicSharedMemorySize, cfg_smem(0)),
            "set smem attribute (pipe)");
  for (int c = kStrip128x16; c <= kStrip32x128; ++c) {
    const StripInfo si = strip_info(c);
    if (si.smem <= st.smem_optin)
      TB_CUDA(cudaFuncSetAttribute(si.fn, cudaFuncAttributeMaxDynamicSharedMemorySize, si.smem),
              "set smem attribute (strip)");
  }
  if (small_smem() <= st.smem_optin)
    for (bool tma : {true, false})
      TB_CUDA(cudaFuncSetAttribute(small_kernel(tma), cudaFuncAttributeMaxDynamicSharedMemorySize, small_smem()),
              "set smem attribute (64-row tiles)");
  TB_CUDA(cudaFuncSetAttribute(tb::dgemm_paper_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               st.smem_optin),
          "set smem attribute (paper)");
  st.attrs_set = true;
  return TB_STATUS_OK;
}

int get_encoder() {
  std::call_once(g_encode_once, [] {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      g_encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
    else
      cudaGetLastError();
  });
  if (!g_encode) {
    set_err("cuTensorMapEncodeTiled unavailable from the driver");
    return TB_STATUS_RUNTIME;
  }
  return TB_STATUS_OK;
}

// Row-major [rows][cols] float64 with leading dim ld, box [box_rows][16 cols], SWIZZLE_128B.
int encode_map(CUtensorMap* map, const double* base, int64_t rows, int64_t cols, int64_t ld, uint32_t box_rows) {
  cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)ld * sizeof(double)};
  cuuint32_t box[2] = {16u, box_rows};
  cuuint32_t estr[2] = {1u, 1u};
  CUresult r = g_encode(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, const_cast<double*>(base), dims, strides, box,
                        estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                        CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    set_err("cuTensorMapEncodeTiled failed (CUresult %d) for %lldx%lld ld=%lld", (int)r, (long long)rows,
            (long long)cols, (long long)ld);
    return TB_STATUS_RUNTIME;
  }
  return TB_STATUS_OK;
}

bool tma_ok(const void* A, int64_t lda, const void* B, int64_t ldb) {
  // TMA: 16-byte aligned global base and 16-byte multiple strides (cuda.h
  // cuTensorMapEncodeTiled requirements), i.e. even leading dims for float64.
  return ((reinterpret_cast<uintptr_t>(A) | reinterpret_cast<uintptr_t>(B)) & 15u) == 0 && (lda % 2 == 0) &&
         (ldb % 2 == 0);
}

int resolve(const void* A, int64_t lda, const void* B, int64_t ldb, int variant) {
  if (variant == TB_VARIANT_AUTO) return tma_ok(A, lda, B, ldb) ? TB_VARIANT_DMMA_TMA : TB_VARIANT_DMMA_CPASYNC;
  if (variant == TB_VARIANT_DMMA_TMA && !tma_ok(A, lda, B, ldb)) return TB_VARIANT_DMMA_CPASYNC;
  return variant;  // DFMA picks its loader at launch (TMA when aligned)
}

// validateLaunch (limits.ts:58-79) plus this kernel family's own limits.
int validate(int64_t m, int64_t k, int64_t n, int32_t tile_edge, int32_t variant, int dev) {
  if (m < 1 || k < 1 || n < 1) {
    set_err("dimensions must be positive integers, got %lldx%lld @ %lldx%lld", (long long)m, (long long)k,
            (long long)k, (long long)n);
    return TB_STATUS_BAD_DIMS;
  }
  if (variant < 0 || variant >= TB_NUM_VARIANTS) {
    set_err("unknown kernel variant %d", variant);
    return TB_STATUS_BAD_DIMS;
  }
  if (tile_edge < 1) {
    set_err("tile edge must be a positive integer, got %d", tile_edge);
    return TB_STATUS_BAD_DIMS;
  }
  const int64_t threads = (int64_t)tile_edge * tile_edge;
  if (threads > kMaxBlockThreads) {
    set_err("block of %lld threads (%dx%d) exceeds the device limit of %d threads per block", (long long)threads,
            tile_edge, tile_edge, kMaxBlockThreads);
    return TB_STATUS_OVER_LIMITS;
  }
  const int64_t lim = 0x7fffffff;
  if (m > lim || k > lim || n > lim) {
    set_err("dimension over the 2^31-1 element limit of this kernel family");
    return TB_STATUS_OVER_LIMITS;
  }
  if (dev >= 0) {
    const DeviceState& st = g_dev[dev];
    const int64_t shared = 2 * threads * (int64_t)sizeof(double);  // limits.ts:45-47
    if (variant == TB_VARIANT_PAPER) {
      if (shared > st.smem_optin) {
        set_err("shared tiles need %lld bytes, over the per-block limit of %d bytes", (long long)shared,
                st.smem_optin);
        return TB_STATUS_OVER_LIMITS;
      }
      if ((m + tile_edge - 1) / tile_edge > 65535) {
        set_err("grid of %lld tile rows exceeds gridDim.y 65535", (long long)((m + tile_edge - 1) / tile_edge));
        return TB_STATUS_OVER_LIMITS;
      }
    } else if (cfg_smem(active_cfg()) > st.smem_optin) {
      set_err("dmma pipeline needs %d bytes of shared memory, device allows %d", cfg_smem(active_cfg()),
              st.smem_optin);
      return TB_STATUS_OVER_LIMITS;
    }
  }
  return TB_STATUS_OK;
}

int check_device(int32_t device) {
  const int count = device_count_raw();
  if (count <= 0 || device < 0 || device >= count || device >= kMaxDevices) {
    set_err("no CUDA device %d (found %d)", device, count);
    return TB_STATUS_NO_DEVICE;
  }
  return ensure_device(device);
}

// Persistent schedule (dgemm_dmma.cuh): data-parallel tiles round-robin over
// the CTAs, then a stream-K region whose k-iterations are split evenly across
// them. Three shapes, chosen on the host (the kernel is the same):
//  - stream-K: the last (T mod P) + P tiles split over P = #SM CTAs;
//  - data-parallel: no split when a single wave is >= 75 % full — splitting
//    every tile costs partial-tile traffic and fixups that an idle 10 % does
//    not (measured: with several waves the stream-K tail still wins);
//  - split-K: T <= P/2 tiles each split into exactly s = P / T equal k-ranges
//    on s*T CTAs (num_k padded up to a multiple of s with k-slabs past K,
//    which the loaders zero-fill), so every CTA owns exactly one segment and
//    every tile exactly s — the stream-K split of so few tiles would give
//    3-4 segments per tile and two fixups to some CTAs.
// TB_SCHED=dp|sk forces data-parallel / the plain stream-K shape (A/B experiments).
struct Schedule {
  int grid, dp, sk, ipc, max_seg, num_k;
};

Schedule plan_schedule(int64_t tiles, int num_k, int sms) {
  static const int forced = [] {
    const char* e = std::getenv("TB_SCHED");
    if (e && std::strcmp(e, "dp") == 0) return 1;
    if (e && std::strcmp(e, "sk") == 0) return 2;  // always the stream-K shape (previous default)
    return 0;
  }();
  Schedule sc{sms, (int)tiles, 0, 1, 1, num_k};
  const int64_t rem = tiles % sms;
  if (forced == 1 || rem == 0) return sc;
  // A single wave >= 75 % full runs data-parallel: splitting every tile of a single wave costs about a
  // quarter of a tile's k-loop in partial traffic and fixups (N = 1500, 144 tiles: 28.6 -> 31.2;
  // N = 1000 on 64-row tiles, 128 tiles: 23.3 -> 25.9; N = 900, 120 tiles: 19.5 -> 20.5; at 61 %,
  // N = 800, stream-K stays ahead 18.2 vs 15.9 TFLOP/s). With more waves the stream-K tail wins
  // (N = 4000 / 6000 at 92 %: 34.12 / 35.84 vs 33.99 / 35.76).
  if (forced == 0 && tiles < sms && 4 * tiles >= 3 * sms) return sc;
  const int64_t min_seg = num_k < 8 ? num_k : 8;      // keep segments long enough to amortise the fixup
  if (forced == 0 && 2 * tiles <= sms) {
    int64_t split = std::min<int64_t>(sms / tiles, num_k / min_seg);
    if (split >= 2) {
      const int64_t ipc = (num_k + split - 1) / split;
      sc.num_k = (int)(ipc * split);
      sc.grid = (int)(split * tiles);
      sc.dp = 0;
      sc.sk = (int)tiles;
      sc.ipc = (int)ipc;
      sc.max_seg = (int)split;
      return sc;
    }
  }
  sc.sk = (int)(tiles > sms ? rem + sms : tiles);
  sc.dp = (int)(tiles - sc.sk);
  const int64_t total = (int64_t)sc.sk * num_k;
  int64_t ipc = (total + sms - 1) / sms;
  if (ipc < min_seg) ipc = min_seg;
  sc.ipc = (int)ipc;
  int max_seg = 1;
  for (int64_t st = 0; st < sc.sk; ++st) {
    const int64_t first = st * num_k;
    const int64_t nseg = (first + num_k - 1) / ipc - first / ipc + 1;
    if (nseg > max_seg) max_seg = (int)nseg;
  }
  sc.max_seg = max_seg;
  return sc;
}

int split_workspace(int dev, cudaStream_t stream, size_t partial_elems, size_t counter_elems, double** partials,
                    int** counters) {
  DeviceState& st = g_dev[dev];
  std::lock_guard<std::mutex> lk(st.mu);
  DeviceState::SplitWs& w = st.split_ws[stream];
  // Size for the schedule's bound on first use (plan_schedule: at most
  // 2P - 1 stream-K tiles of at most 2 segments when T > P, at most P + T
  // slots when T <= P), so a stream never regrows while its earlier launches
  // may still be queued.
  partial_elems = std::max(partial_elems, (size_t)4 * st.sms * tb::DmmaCfg::TILE_ELEMS);
  counter_elems = std::max(counter_elems, (size_t)2 * st.sms);
  if ((w.partial_elems < partial_elems && w.partials) || (w.counter_elems < counter_elems && w.counters))
    TB_CUDA(cudaStreamSynchronize(stream), "stream-K workspace regrow");  // earlier launches may use it
  if (w.partial_elems < partial_elems) {
    if (w.partials) cudaFree(w.partials);
    w.partials = nullptr;
    w.partial_elems = 0;
    TB_CUDA(cudaMalloc(&w.partials, partial_elems * sizeof(double)), "stream-K workspace allocation");
    w.partial_elems = partial_elems;
  }
  if (w.counter_elems < counter_elems) {
    if (w.counters) cudaFree(w.counters);
    w.counters = nullptr;
    w.counter_elems = 0;
    TB_CUDA(cudaMalloc(&w.counters, counter_elems * sizeof(int)), "stream-K counter allocation");
    // Counters start at zero once; each launch's last segment resets its tile's
    // counter. Zeroed on the launching stream: a legacy-stream memset is not
    // ordered before kernels on non-blocking streams.
    TB_CUDA(cudaMemsetAsync(w.counters, 0, counter_elems * sizeof(int), stream), "stream-K counter init");
    w.counter_elems = counter_elems;
  }
  *partials = w.partials;
  *counters = w.counters;
  return TB_STATUS_OK;
}

// Enqueue one GEMM on `stream` (current device = dev). Assumes validated args.
// AUTO on operands TMA cannot address (odd leading dimension or a base not
// 16-byte aligned — the reference's odd-N cases) would run the cp.async
// loader at ~92 % of the TMA path's speed. For large products the operands
// are instead copied once, on the launching stream, into even-pitch
// workspace buffers (HBM copy: ~1 % of the GEMM time at N = 9999) and the
// TMA kernel runs on those. Small products keep the cp.async loader.
constexpr double kStageMinFlops = 2e10;
constexpr size_t kStageMaxBytes = size_t(16) << 30;

// Row re-pitch for staging: dst (16-byte aligned, even pitch) <- src (any
// 8-byte alignment/pitch). One block row-slab per blockIdx.y, coalesced 8-byte
// loads, 16-byte stores where the destination allows.
__global__ void __launch_bounds__(256) repitch_kernel(const double* __restrict__ src, int64_t lds,
                                                      double* __restrict__ dst, int64_t ldd, int64_t rows,
                                                      int64_t cols) {
  for (int64_t r = blockIdx.y; r < rows; r += gridDim.y) {
    const double* s = src + r * lds;
    double2* d = reinterpret_cast<double2*>(dst + r * ldd);
    for (int64_t c = 2 * ((int64_t)blockIdx.x * blockDim.x + threadIdx.x); c < cols;
         c += 2 * (int64_t)gridDim.x * blockDim.x) {
      const double x = s[c];
      const double y = c + 1 < cols ? s[c + 1] : 0.0;
      d[c >> 1] = make_double2(x, y);  // ldd even and >= cols + (cols & 1): the pad column takes 0
    }
  }
}

int repitch(const double* src, int64_t lds, double* dst, int64_t ldd, int64_t rows, int64_t cols,
            cudaStream_t stream) {
  const int64_t pairs = (cols + 1) / 2;
  const unsigned gx = (unsigned)std::min<int64_t>((pairs + 255) / 256, 8);
  const unsigned gy = (unsigned)std::min<int64_t>(rows, 65535);
  repitch_kernel<<<dim3(gx, gy), 256, 0, stream>>>(src, lds, dst, ldd, rows, cols);
  TB_CUDA(cudaGetLastError(), "staging copy launch");
  g_launches.fetch_add(1, std::memory_order_relaxed);
  return TB_STATUS_OK;
}

bool misaligned(const void* p, int64_t ld) { return (reinterpret_cast<uintptr_t>(p) & 15u) != 0 || (ld % 2) != 0; }

int stage_workspace(int dev, cudaStream_t stream, size_t elems, double** buf) {
  DeviceState& st = g_dev[dev];
  std::lock_guard<std::mutex> lk(st.mu);
  DeviceState::StageWs& w = st.stage_ws[stream];
  if (w.elems < elems) {
    if (w.buf) {
      TB_CUDA(cudaStreamSynchronize(stream), "staging workspace regrow");  // earlier launches may use it
      cudaFree(w.buf);
    }
    w.buf = nullptr;
    w.elems = 0;
    TB_CUDA(cudaMalloc(&w.buf, elems * sizeof(double)), "staging workspace allocation");
    w.elems = elems;
  }
  *buf = w.buf;
  return TB_STATUS_OK;
}

int launch_tiles(int dev, const double* A, int64_t lda, const double* B, int64_t ldb, double* Cm, int64_t ldc,
                 int64_t m, int64_t k, int64_t n, int accumulate, int tile_edge, int variant, cudaStream_t stream,
                 int strip);

// Enqueue one GEMM on `stream` (current device = dev). Assumes validated args.
// Stages misaligned operands (large AUTO calls), then, for a large TMA-fed
// DMMA product whose m or n is not a multiple of 128, runs the whole-tile
// part and the remainder strips as separate launches (TB_SPLIT=0: one
// launch, A/B).
int launch(int dev, const double* A, int64_t lda, const double* B, int64_t ldb, double* Cm, int64_t ldc, int64_t m,
           int64_t k, int64_t n, int accumulate, int tile_edge, int variant, cudaStream_t stream) {
  int s = ensure_kernel_attrs(dev);
  if (s) return s;
  if (variant == TB_VARIANT_AUTO && !tma_ok(A, lda, B, ldb) && 2.0 * (double)m * (double)n * (double)k >= kStageMinFlops) {
    const bool sa = misaligned(A, lda), sb = misaligned(B, ldb);
    const int64_t lda2 = (k + 1) & ~int64_t(1), ldb2 = (n + 1) & ~int64_t(1);
    const size_t ea = sa ? (size_t)(m * lda2 + 32) : 0, eb = sb ? (size_t)(k * ldb2) : 0;
    if ((ea + eb) * sizeof(double) <= kStageMaxBytes) {
      double* buf = nullptr;
      if ((s = stage_workspace(dev, stream, ea + eb + 32, &buf))) return s;
      double* a2 = buf;
      double* b2 = buf + ((ea + 31) & ~size_t(31));  // 256-byte aligned
      if (sa) {
        if ((s = repitch(A, lda, a2, lda2, m, k, stream))) return s;
        A = a2;
        lda = lda2;
      }
      if (sb) {
        if ((s = repitch(B, ldb, b2, ldb2, k, n, stream))) return s;
        B = b2;
        ldb = ldb2;
      }
    }
  }
  variant = resolve(A, lda, B, ldb, variant);
  static const bool split_env = !(std::getenv("TB_SPLIT") && std::strcmp(std::getenv("TB_SPLIT"), "0") == 0);
  if (split_env && variant == TB_VARIANT_DMMA_TMA && (m % 128 != 0 || n % 128 != 0)) {
    const int64_t hb = m % 128, wr = n % 128;
    const int bcfg = hb == 0 ? kStripNone : hb <= 16 ? kStrip16x128 : hb <= 32 ? kStrip32x128
                                                      : hb <= 64 ? kStrip64x128 : kStripNone;
    const int rcfg = wr == 0 ? kStripNone : wr <= 16 ? kStrip128x16 : wr <= 32 ? kStrip128x32
                                                      : wr <= 64 ? kStrip128x64 : kStripNone;
    const int64_t m1 = bcfg != kStripNone ? m - hb : m, n1 = rcfg != kStripNone ? n - wr : n;
    if ((bcfg != kStripNone || rcfg != kStripNone) && m1 >= 128 && n1 >= 128 &&
        choose_bm(m1, n1, g_dev[dev].sms, false) == 128) {
      // Main part on whole 128 x 128 tiles, then the right strip (all rows)
      // and the bottom strip (the main part's columns); disjoint parts of C.
      if ((s = launch_tiles(dev, A, lda, B, ldb, Cm, ldc, m1, k, n1, accumulate, tile_edge, variant, stream, -1)))
        return s;
      if (rcfg != kStripNone &&
          (s = launch_tiles(dev, A, lda, B + n1, ldb, Cm + n1, ldc, m, k, n - n1, accumulate, tile_edge, variant,
                            stream, rcfg)))
        return s;
      if (bcfg != kStripNone &&
          (s = launch_tiles(dev, A + m1 * lda, lda, B, ldb, Cm + m1 * ldc, ldc, m - m1, k, n1, accumulate,
                            tile_edge, variant, stream, bcfg)))
        return s;
      return TB_STATUS_OK;
    }
  }
  return launch_tiles(dev, A, lda, B, ldb, Cm, ldc, m, k, n, accumulate, tile_edge, variant, stream, kStripNone);
}

// One launch on resolved operands. strip: kStripNone = choose_bm's tile
// height, -1 = 128 x 128 forced, else an edge-strip shape.
int launch_tiles(int dev, const double* A, int64_t lda, const double* B, int64_t ldb, double* Cm, int64_t ldc,
                 int64_t m, int64_t k, int64_t n, int accumulate, int tile_edge, int variant, cudaStream_t stream,
                 int strip) {
  int s = TB_STATUS_OK;
  if (variant == TB_VARIANT_PAPER) {
    const int K = tile_edge;
    dim3 block(K, K);
    dim3 grid((unsigned)((n + K - 1) / K), (unsigned)((m + K - 1) / K));
    tb::dgemm_paper_kernel<<<grid, block, 2 * K * K * sizeof(double), stream>>>(
        A, lda, B, ldb, Cm, ldc, (int)m, (int)k, (int)n, K, accumulate);
    g_launches.fetch_add(1, std::memory_order_relaxed);
  } else {
    using Cfg = tb::DmmaCfg;
    tb::GemmParams p;
    p.A = A;
    p.B = B;
    p.C = Cm;
    p.lda = lda;
    p.ldb = ldb;
    p.ldc = ldc;
    p.m = (int)m;
    p.n = (int)n;
    p.k = (int)k;
    const bool dfma = variant == TB_VARIANT_DFMA;
    const StripInfo si = strip > 0 ? strip_info(strip) : StripInfo{0, 0, nullptr, 0};
    const bool narrow = si.fn != nullptr;  // an edge-strip shape (TMA only)
    const int bm = narrow ? si.bm : strip == kStrip64x128 ? 64 : strip < 0 ? 128 : choose_bm(m, n, g_dev[dev].sms, dfma);
    const int bn = narrow ? si.bn : Cfg::BN;
    p.tiles_m = (int)((m + bm - 1) / bm);
    p.tiles_n = (int)((n + bn - 1) / bn);
    p.accumulate = accumulate;
    p.vec_store = ((reinterpret_cast<uintptr_t>(Cm) & 15u) == 0 && ldc % 2 == 0) ? 1 : 0;
    const int64_t tiles = (int64_t)p.tiles_m * p.tiles_n;
    if (tiles > 0x7fffffff) {
      set_err("too many output tiles");
      return TB_STATUS_OVER_LIMITS;
    }
    const int cfg = dfma ? 0 : active_cfg();
    const int64_t kstage = (bm == 64 || narrow) ? (int64_t)Cfg::BK : (int64_t)Cfg::BK * kCfgs[cfg].sub;
    p.num_k = (int)((k + kstage - 1) / kstage);
    const Schedule sc = plan_schedule(tiles, p.num_k, g_dev[dev].sms);
    p.num_k = sc.num_k;  // split-K pads the k-slab count (extra slabs read as zeros)
    p.dp_tiles = sc.dp;
    p.sk_tiles = sc.sk;
    p.sk_ipc = sc.ipc;
    p.max_seg = sc.max_seg;
    p.partials = nullptr;
    p.counters = nullptr;
#ifdef TB_TIMELINE
    unsigned long long* tl_buf = nullptr;
    p.timeline = nullptr;
    if (std::getenv("TB_TIMELINE")) {
      TB_CUDA(cudaMalloc(&tl_buf, (size_t)sc.grid * 8 * sizeof(unsigned long long)), "timeline alloc");
      TB_CUDA(cudaMemsetAsync(tl_buf, 0, (size_t)sc.grid * 8 * sizeof(unsigned long long), stream), "timeline");
      p.timeline = tl_buf;
    }
#endif
    if (sc.sk > 0 &&
        (s = split_workspace(dev, stream, (size_t)sc.sk * sc.max_seg * Cfg::TILE_ELEMS, (size_t)sc.sk, &p.partials,
                             &p.counters)))
      return s;
    CUtensorMap mA, mB;
    std::memset(&mA, 0, sizeof(mA));
    std::memset(&mB, 0, sizeof(mB));
    const bool use_tma = variant == TB_VARIANT_DMMA_TMA || (dfma && tma_ok(A, lda, B, ldb));
    if (use_tma) {
      if ((s = get_encoder())) return s;
      if ((s = encode_map(&mA, A, m, k, lda, (uint32_t)bm))) return s;
      if ((s = encode_map(&mB, B, k, n, ldb, Cfg::BK))) return s;
    }
    void* args[] = {&mA, &mB, &p};
    if (narrow && !use_tma) {
      set_err("edge-strip launch needs TMA-addressable operands");
      return TB_STATUS_RUNTIME;
    }
    TB_CUDA(cudaLaunchKernel(narrow ? si.fn : bm == 64 ? small_kernel(use_tma) : cfg_kernel(cfg, use_tma, dfma),
                             dim3((unsigned)sc.grid), dim3(Cfg::THREADS), args,
                             (size_t)(narrow ? si.smem : bm == 64 ? small_smem() : cfg_smem(cfg)), stream),
            "kernel launch");
    g_launches.fetch_add(1, std::memory_order_relaxed);
#ifdef TB_TIMELINE
    if (tl_buf) {
      // Per-CTA stamps (ns): [0] entry [1] first stage landed [2] last main-loop end [3] last unit done
      // [4] units [5] fixup ns [6] epilogue ns [7] main-loop ns.
      std::vector<unsigned long long> h((size_t)sc.grid * 8);
      TB_CUDA(cudaStreamSynchronize(stream), "timeline sync");
      TB_CUDA(cudaMemcpy(h.data(), tl_buf, h.size() * sizeof(unsigned long long), cudaMemcpyDeviceToHost), "tl");
      cudaFree(tl_buf);
      unsigned long long t0 = ~0ull, tend = 0;
      double first = 0, mainl = 0, fix = 0, epi = 0, units = 0, endmax = 0, endmin = 1e30, lastml = 0;
      for (int c = 0; c < sc.grid; ++c) {
        const unsigned long long* r = &h[(size_t)c * 8];
        t0 = std::min(t0, r[0]);
        tend = std::max(tend, r[3]);
      }
      for (int c = 0; c < sc.grid; ++c) {
        const unsigned long long* r = &h[(size_t)c * 8];
        first += (double)(r[1] - t0);
        lastml += (double)(r[2] - t0);
        mainl += (double)r[7];
        fix += (double)r[5];
        epi += (double)r[6];
        units += (double)r[4];
        endmax = std::max(endmax, (double)(r[3] - t0));
        endmin = std::min(endmin, (double)(r[3] - t0));
      }
      const double g = sc.grid;
      std::fprintf(stderr,
                   "TBTIMELINE m=%lld n=%lld k=%lld grid=%d dp=%d sk=%d ipc=%d maxseg=%d span_us=%.2f "
                   "first_stage_us=%.2f mainloop_us=%.2f last_mainloop_end_us=%.2f fixup_us=%.2f epilogue_us=%.2f "
                   "units=%.2f end_min_us=%.2f end_max_us=%.2f\n",
                   (long long)m, (long long)n, (long long)k, sc.grid, sc.dp, sc.sk, sc.ipc, sc.max_seg,
                   (tend - t0) / 1e3, first / g / 1e3, mainl / g / 1e3, lastml / g / 1e3, fix / g / 1e3,
                   epi / g / 1e3, units / g, endmin / 1e3, endmax / 1e3);
    }
#endif
  }
  TB_CUDA(cudaGetLastError(), "kernel launch");
  return TB_STATUS_OK;
}

// One persistent launch for the host pipeline's phase 1 (PIPE mode): C =
// A·B over all k, k-panel q (k-stages [panel_it[q], panel_it[q+1]), panel_it
// in device memory) consumed once flags[q] != 0. TMA operands (even pitch,
// 16-byte aligned) only.
int launch_pipe(int dev, const double* A, int64_t lda, const double* B, int64_t ldb, double* Cm, int64_t ldc,
                int64_t m, int64_t k, int64_t n, const int* panel_it_d, const int* flags_d, int Q,
                cudaStream_t stream) {
  int s = ensure_kernel_attrs(dev);
  if (s) return s;
  using Cfg = tb::DmmaCfg;
  tb::GemmParams p;
  std::memset(&p, 0, sizeof(p));
  p.A = A;
  p.B = B;
  p.C = Cm;
  p.lda = lda;
  p.ldb = ldb;
  p.ldc = ldc;
  p.m = (int)m;
  p.n = (int)n;
  p.k = (int)k;
  p.tiles_m = (int)((m + Cfg::BM - 1) / Cfg::BM);
  p.tiles_n = (int)((n + Cfg::BN - 1) / Cfg::BN);
  p.num_k = (int)((k + Cfg::BK - 1) / Cfg::BK);
  p.accumulate = 0;
  p.vec_store = ((reinterpret_cast<uintptr_t>(Cm) & 15u) == 0 && ldc % 2 == 0) ? 1 : 0;
  const int64_t tiles = (int64_t)p.tiles_m * p.tiles_n;
  p.dp_tiles = (int)tiles;
  p.sk_tiles = Q;                                        // PIPE: panel count
  p.sk_ipc = 1;
  p.max_seg = 1;
  p.counters = const_cast<int*>(panel_it_d);             // PIPE: panel k-stage bounds
  p.partials = reinterpret_cast<double*>(const_cast<int*>(flags_d));  // PIPE: panel flags
  if ((s = get_encoder())) return s;
  CUtensorMap mA, mB;
  if ((s = encode_map(&mA, A, m, k, lda, Cfg::BM))) return s;
  if ((s = encode_map(&mB, B, k, n, ldb, Cfg::BK))) return s;
  void* args[] = {&mA, &mB, &p};
  const int grid = (int)std::min<int64_t>(tiles, g_dev[dev].sms);
  TB_CUDA(cudaLaunchKernel(pipe_kernel(), dim3((unsigned)grid), dim3(Cfg::THREADS), args, (size_t)cfg_smem(0), stream),
          "kernel launch (pipe)");
  g_launches.fetch_add(1, std::memory_order_relaxed);
  return TB_STATUS_OK;
}

struct EventPair {
  cudaEvent_t a = nullptr, b = nullptr;
  ~EventPair() {
    if (a) cudaEventDestroy(a);
    if (b) cudaEventDestroy(b);
  }
  int create() {
    TB_CUDA(cudaEventCreate(&a), "event create");
    TB_CUDA(cudaEventCreate(&b), "event create");
    return TB_STATUS_OK;
  }
};

int timed_gemm(int dev, const double* A, const double* B, double* Cm, int64_t m, int64_t k, int64_t n,
               int tile_edge, int variant, cudaStream_t stream, double* out_seconds, bool use_cublas) {
  EventPair ev;
  int s = ev.create();
  if (s) return s;
  TB_CUDA(cudaEventRecord(ev.a, stream), "event record");
  if (use_cublas) {
    DeviceState& st = g_dev[dev];
    {
      std::lock_guard<std::mutex> lk(st.mu);
      if (!st.cublas && cublasCreate(&st.cublas) != CUBLAS_STATUS_SUCCESS) {
        set_err("cublasCreate failed");
        return TB_STATUS_RUNTIME;
      }
    }
    cublasSetStream(st.cublas, stream);
    const double one = 1.0, zero = 0.0;
    // Row-major C = A·B  <=>  column-major C^T = B^T · A^T.
    if (cublasDgemm(st.cublas, CUBLAS_OP_N, CUBLAS_OP_N, (int)n, (int)m, (int)k, &one, B, (int)n, A, (int)k, &zero,
                    Cm, (int)n) != CUBLAS_STATUS_SUCCESS) {
      set_err("cublasDgemm failed");
      return TB_STATUS_RUNTIME;
    }
  } else {
    s = launch(dev, A, k, B, n, Cm, n, m, k, n, 0, tile_edge, variant, stream);
    if (s) return s;
  }
  TB_CUDA(cudaEventRecord(ev.b, stream), "event record");
  TB_CUDA(cudaEventSynchronize(ev.b), "kernel execution");
  float ms = 0.f;
  TB_CUDA(cudaEventElapsedTime(&ms, ev.a, ev.b), "event elapsed");
  if (out_seconds) *out_seconds = (double)ms * 1e-3;
  return TB_STATUS_OK;
}

int dgemm_common(const double* A, const double* B, double* Cm, int64_t m, int64_t k, int64_t n, int32_t tile_edge,
                 int32_t variant, int32_t device, void* cuda_stream, double* out_seconds, bool use_cublas) {
  int s = check_device(device);
  if (s) return s;
  if (!A || !B || !Cm || !out_seconds) {
    set_err("null buffer pointer");
    return TB_STATUS_BAD_DIMS;
  }
  if ((s = validate(m, k, n, tile_edge, variant, device))) return s;
  DeviceGuard guard(device);
  return timed_gemm(device, A, B, Cm, m, k, n, tile_edge, variant, static_cast<cudaStream_t>(cuda_stream),
                    out_seconds, use_cublas);
}

}  // namespace

// The host pipeline's shape (pure; exported as tb_pipeline_plan for tests).
struct PipePlan {
  int64_t Mq = 0;
  bool fused = false;          // phase 1 as one PIPE-mode launch
  std::vector<int64_t> pk;     // phase-1 K-panel bounds
  std::vector<int64_t> gb;     // phase-1 row groups (one per compute stream)
  std::vector<int64_t> rb;     // phase-2 row-block bounds, rb[0] = Mq
};

PipePlan plan_pipeline(int64_t m, int64_t k, int64_t n, int sms, bool fused_ok) {
  PipePlan pl;
  int64_t& Mq = pl.Mq;
  bool& fused = pl.fused;
  std::vector<int64_t>& pk = pl.pk;
  std::vector<int64_t>& gb = pl.gb;
  std::vector<int64_t>& rb = pl.rb;
  Mq = m;
  pk = {0, k};
  gb = {0, m};
  rb = {m};
  const double flops = 2.0 * (double)m * (double)n * (double)k;
  if (flops >= 1e11) {
    constexpr double kH2D = 55e9, kRate = 36e12;  // B/s (PCIe gen5 x16, measured), flop/s (FP64 DMMA)
    const double den = (double)n * kH2D - 4.0 * kRate;
    int64_t mq = den > 0 ? (int64_t)(1.2 * 4.0 * kRate * (double)n / den) : m;
    int64_t kp0 = 256, kp_max = 2048, blk = 1536, groups = 2;
    // TB_PIPE=mq,kp0,kp_max,blk[,groups] overrides the shape (tuning experiments).
    if (const char* e = std::getenv("TB_PIPE")) {
      long long a0 = 0, a1 = 0, a2 = 0, a3 = 0, a4 = 2;
      if (std::sscanf(e, "%lld,%lld,%lld,%lld,%lld", &a0, &a1, &a2, &a3, &a4) >= 4 && a0 >= 1 && a1 >= 2 &&
          a2 >= 2 && a3 >= 1 && a4 >= 1) {
        mq = a0;
        kp0 = a1;
        kp_max = a2;
        blk = a3;
        groups = a4;
      }
    }
    mq = (mq + 127) / 128 * 128;
    // Phase 1 as one persistent launch that waits on per-panel flags (PIPE
    // mode) rather than a launch per panel and row group; TB_PIPE_FUSED=0
    // restores the launch-per-panel form (A/B).
    const char* fe = std::getenv("TB_PIPE_FUSED");
    fused = fused_ok && !(fe && std::strcmp(fe, "0") == 0);
    if (fused && !std::getenv("TB_PIPE")) {
      // The fused launch gives CTA c the phase-1 tiles c, c + P, ...: pick
      // the tile-row count (>= the compute-cover minimum, up to 8 more) whose
      // tile count leaves the least imbalance, ceil(T/P) - T/P (N = 10000:
      // 34 rows -> 18.15 tiles per CTA, 59.1 ms; 41 rows -> 21.89, 58.0 ms;
      // profiles/r01_pipe_trace_mq_sweep.txt).
      const int64_t tn = (n + 127) / 128, P_sm = sms;
      int64_t best_r = mq / 128;
      double best_imb = 2.0;
      for (int64_t rr = mq / 128; rr <= mq / 128 + 8 && rr * 128 < m - blk / 2; ++rr) {
        const double per = (double)(rr * tn) / (double)P_sm;
        const double imb = std::ceil(per) - per;
        if (imb < best_imb - 1e-9) {
          best_imb = imb;
          best_r = rr;
        }
      }
      mq = best_r * 128;
    }
    Mq = mq >= m - blk / 2 ? m : mq;
    const int64_t kal = fused ? 16 : 2;  // panel bounds on k-stage (PIPE) or TMA (even k0) boundaries
    // Panel sizes: after a small first panel, each panel is as large as can
    // land (transfer model) before the GEMMs queued so far drain (compute
    // model), so the panels grow geometrically by the compute/transfer ratio
    // without opening a compute gap; capped at kp_max.
    const double tr_per_k = 8.0 * (double)(Mq + n) / kH2D, c_per_k = 2.0 * (double)Mq * (double)n / kRate;
    pk.assign(1, 0);
    double arrive = 0.0, finish = 0.0;
    for (int64_t at = 0, step = kp0; at < k;) {
      int64_t nx = at + step >= k - step / 2 ? k : ((at + step) / kal * kal);
      if (nx <= at) nx = std::min<int64_t>(k, at + kal);
      arrive += tr_per_k * (double)(nx - at);
      finish = std::max(finish, arrive) + c_per_k * (double)(nx - at);
      pk.push_back(nx);
      at = nx;
      step = std::min<int64_t>(kp_max, std::max<int64_t>(kp0, (int64_t)((finish - arrive) / tr_per_k)));
    }
    gb = (groups >= 2 && Mq >= 2048) ? std::vector<int64_t>{0, (Mq / 2 + 127) / 128 * 128, Mq}
                                     : std::vector<int64_t>{0, Mq};
    int64_t r = m - Mq;
    std::vector<int64_t> tail;
    for (int64_t t : {std::min<int64_t>(128, blk / 4), blk / 2})  // shrinking tail: the last D2H is ~10-20 MB
      if (t > 0 && r >= 2 * t) {
        tail.push_back(t);
        r -= t;
      }
    rb.assign(1, Mq);
    const int64_t nb = (r + blk - 1) / blk;
    // Block bounds on 128-row tile boundaries: a block of, say, 1413 rows
    // would pad its last tile row to 1536 (8 % of its DMMAs on zeros).
    for (int64_t i = 1; i <= nb; ++i) {
      const int64_t bnd = i == nb ? Mq + r : std::min(Mq + r, Mq + (r * i / nb + 64) / 128 * 128);
      if (bnd > rb.back()) rb.push_back(bnd);  // no empty blocks
    }
    for (auto it = tail.rbegin(); it != tail.rend(); ++it) rb.push_back(rb.back() + *it);
    // Interior bounds on tile rows (Mq is a multiple of 128): only the last
    // block may be ragged.
    std::vector<int64_t> al{rb.front()};
    for (size_t i = 1; i + 1 < rb.size(); ++i) {
      const int64_t v = (rb[i] + 64) / 128 * 128;
      if (v > al.back() && v < m) al.push_back(v);
    }
    if (m > al.back()) al.push_back(m);
    rb.swap(al);
  }
  if (pl.pk.size() - 1 < 2 || pl.pk.size() - 1 > 120) pl.fused = false;  // table holds <= 120 panels
  return pl;
}

extern "C" {

int tb_device_count(void) { return device_count_raw(); }

const char* tb_last_error(void) { return g_err; }

const char* tb_version(void) { return TB_VERSION; }

const char* tb_variant_name(int32_t variant) {
  switch (variant) {
    case TB_VARIANT_AUTO: return "auto";
    case TB_VARIANT_PAPER: return "paper";
    case TB_VARIANT_DMMA_TMA: return "dmma_tma";
    case TB_VARIANT_DMMA_CPASYNC: return "dmma_cpasync";
    case TB_VARIANT_DFMA: return "dfma";
    default: return nullptr;
  }
}

int tb_resolve_variant(const void* A, int64_t lda, const void* B, int64_t ldb, int32_t variant) {
  if (variant < 0 || variant >= TB_NUM_VARIANTS) return -1;
  return resolve(A, lda, B, ldb, variant);
}

int tb_validate_launch(int64_t m, int64_t k, int64_t n, int32_t tile_edge, int32_t variant, int32_t device) {
  int s = check_device(device);
  if (s) return s;
  return validate(m, k, n, tile_edge, variant, device);
}

int tb_dgemm(const double* A, const double* B, double* C, int64_t m, int64_t k, int64_t n, int32_t tile_edge,
             int32_t variant, int32_t device, void* cuda_stream, double* out_kernel_seconds) {
  return dgemm_common(A, B, C, m, k, n, tile_edge, variant, device, cuda_stream, out_kernel_seconds, false);
}

int tb_cublas_dgemm(const double* A, const double* B, double* C, int64_t m, int64_t k, int64_t n, int32_t tile_edge,
                    int32_t variant, int32_t device, void* cuda_stream, double* out_kernel_seconds) {
  return dgemm_common(A, B, C, m, k, n, tile_edge, variant, device, cuda_stream, out_kernel_seconds, true);
}

int tb_dgemm_launch(const double* A, int64_t lda, const double* B, int64_t ldb, double* C, int64_t ldc, int64_t m,
                    int64_t k, int64_t n, int32_t accumulate, int32_t tile_edge, int32_t variant, void* cuda_stream) {
  int dev = -1;
  if (cudaGetDevice(&dev) != cudaSuccess) {
    cudaGetLastError();
    set_err("no current CUDA device");
    return TB_STATUS_NO_DEVICE;
  }
  int s = check_device(dev);
  if (s) return s;
  if (!A || !B || !C) {
    set_err("null buffer pointer");
    return TB_STATUS_BAD_DIMS;
  }
  if ((s = validate(m, k, n, tile_edge, variant, dev))) return s;
  if (lda < k || ldb < n || ldc < n) {
    set_err("leading dimensions too small (lda=%lld ldb=%lld ldc=%lld)", (long long)lda, (long long)ldb,
            (long long)ldc);
    return TB_STATUS_BAD_DIMS;
  }
  return launch(dev, A, lda, B, ldb, C, ldc, m, k, n, accumulate, tile_edge, variant,
                static_cast<cudaStream_t>(cuda_stream));
}

int tb_gpu_tiled_multiply_flat_ex(int32_t device, const double* a, const double* b, int64_t m, int64_t k, int64_t n,
                                  int32_t tile_edge, int32_t variant, double* out_c, int64_t out_c_len,
                                  double* out_seconds, double* out_e2e_seconds) {
  const auto h_entry = std::chrono::steady_clock::now();
  int s = check_device(device);  // multiply.ts:65 — no device is a status, not a throw
  if (s) return s;
  if (!a || !b || !out_c || !out_seconds || m < 1 || k < 1 || n < 1 || out_c_len != m * n) {
    set_err("bad dimensions or output buffer (out_c_len=%lld, m*n=%lld)", (long long)out_c_len,
            (long long)(m * n));
    return TB_STATUS_BAD_DIMS;  // multiply.ts:66
  }
  if ((s = validate(m, k, n, tile_edge, variant, device))) return s;
  DeviceGuard guard(device);
  DeviceState& st = g_dev[device];
  std::lock_guard<std::mutex> lk(st.host_mu);  // one in-flight call per backend
  // Device copies use even pitches so odd k / n still get the TMA loader and
  // 16-byte C stores / batched accumulate loads (the 2D copies re-pitch for free).
  const int64_t lda_d = (k + 1) & ~int64_t(1), ldb_d = (n + 1) & ~int64_t(1), ldc_d = ldb_d;
  const size_t na = (size_t)(m * lda_d), nb = (size_t)(k * ldb_d), nc = (size_t)(m * ldc_d);
  auto up = [](size_t x) { return (x + 31) & ~size_t(31); };  // 256-byte aligned sub-buffers
  const size_t need = (up(na) + up(nb) + up(nc)) * sizeof(double);
  for (cudaStream_t* sp : {&st.host_stream, &st.host_stream2, &st.h2d_stream, &st.d2h_stream})
    if (!*sp) TB_CUDA(cudaStreamCreateWithFlags(sp, cudaStreamNonBlocking), "stream create");
  if (st.ws_bytes < need) {
    if (st.ws) cudaFree(st.ws);
    st.ws = nullptr;
    st.ws_bytes = 0;
    TB_CUDA(cudaMalloc(&st.ws, need), "device workspace allocation");
    st.ws_bytes = need;
  }
  double* dA = st.ws;
  double* dB = dA + up(na);
  double* dC = dB + up(nb);
  const cudaStream_t hs = st.h2d_stream, ds = st.d2h_stream;
  const cudaStream_t css[2] = {st.host_stream, st.host_stream2};

  // Copy/compute/copy pipeline over four streams (H2D, two compute, D2H).
  //  Phase 1 (rank-k panels): the first Mq rows of C are computed as
  //    C[0:Mq] (+)= A[0:Mq, panel p] · B[panel p, :]
  //  while the panels stream in (A's panel slice by a 2D copy, B's panel as
  //  contiguous rows). The first panel is small, so the GEMM starts early;
  //  Mq is sized so a panel's GEMM (2·Mq·kp·n flops) outlasts its transfer
  //  (8·kp·(Mq+n) bytes) and compute does not wait on PCIe afterwards.
  //  Phase 2 (row blocks): the remaining rows of A arrive as contiguous
  //  blocks and run full-K GEMMs; every finished part of C is copied back at
  //  once, and the last blocks shrink so the final D2H is short.
  // Small problems degenerate to copy, GEMM, copy.
  const bool fused_ok = variant != TB_VARIANT_PAPER && variant != TB_VARIANT_DFMA &&
                        variant != TB_VARIANT_DMMA_CPASYNC && cfg_smem(0) <= g_dev[device].smem_optin;
  const PipePlan plan = plan_pipeline(m, k, n, g_dev[device].sms, fused_ok);
  const int64_t Mq = plan.Mq;
  bool fused = plan.fused;
  const std::vector<int64_t>& pk = plan.pk;  // phase-1 K-panel bounds
  const std::vector<int64_t>& gb = plan.gb;  // phase-1 row groups (launch-per-panel form)
  const std::vector<int64_t>& rb = plan.rb;  // phase-2 row-block bounds, rb[0] = Mq
  const int P = (int)pk.size() - 1, G = (int)gb.size() - 1, R = (int)rb.size() - 1;
  // Ragged n (<= 64 columns past a multiple of 128) on the fused path: every
  // launch covers the first n1 columns on whole tiles and one edge-strip
  // launch computes the remaining columns for all rows.
  const int64_t wr = n % 128;
  const bool strip_n = fused && wr > 0 && wr <= 64 && n >= 256 &&
                       !(std::getenv("TB_SPLIT") && std::strcmp(std::getenv("TB_SPLIT"), "0") == 0);
  const int64_t n1 = strip_n ? n - wr : n;

  // Events come from a per-device pool reused across calls (every call
  // drains its streams before returning), so the host does not create and
  // destroy ~100 events per call.
  size_t used[2] = {0, 0};
  bool ev_fail = false;
  auto mk = [&](unsigned flags) -> cudaEvent_t {
    const int kind = flags == cudaEventDisableTiming ? 1 : 0;
    std::vector<cudaEvent_t>& pool = st.ev_pool[kind];
    if (used[kind] == pool.size()) {
      cudaEvent_t e = nullptr;
      if (cudaEventCreateWithFlags(&e, flags) != cudaSuccess) {
        ev_fail = true;
        return nullptr;
      }
      pool.push_back(e);
    }
    return pool[used[kind]++];
  };
  cudaEvent_t e_start = mk(cudaEventDefault), e_end = mk(cudaEventDefault);
  std::vector<cudaEvent_t> evP(P), evA(R), kt0, kt1;
  for (auto& e : evP) e = mk(cudaEventDisableTiming);
  for (auto& e : evA) e = mk(cudaEventDisableTiming);
  if (ev_fail) return cuda_fail(cudaGetLastError(), "event create");

  // TB_PIPE_TRACE=1: print every copy / GEMM's device interval (ms from the
  // pipeline start) to stderr — tooling for tools/pipe_trace.py.
  static const bool trace = std::getenv("TB_PIPE_TRACE") != nullptr;
  struct TraceRec {
    const char* what;
    int idx;
    cudaEvent_t t0, t1;
    double bytes;
  };
  std::vector<TraceRec> tr;
  auto trace_begin = [&](cudaStream_t sm) -> cudaEvent_t {
    if (!trace) return nullptr;
    cudaEvent_t e = mk(cudaEventDefault);
    if (e) cudaEventRecord(e, sm);
    return e;
  };
  auto trace_end = [&](const char* what, int idx, cudaEvent_t t0, cudaStream_t sm, double bytes) {
    if (!trace || !t0) return;
    cudaEvent_t e = mk(cudaEventDefault);
    if (!e) return;
    cudaEventRecord(e, sm);
    tr.push_back({what, idx, t0, e, bytes});
  };
  // Rows [r0, r1) x columns [c0, c1) of a row-major host matrix with `cols`
  // columns into the same place of its device copy of pitch `dld` (>= cols).
  auto h2d = [&](double* dst, int64_t dld, const double* src, int64_t cols, int64_t r0, int64_t r1, int64_t c0,
                 int64_t c1, const char* what, int idx) -> int {
    cudaEvent_t t0 = trace_begin(hs);
    const size_t pitch = (size_t)cols * sizeof(double);
    if (c0 == 0 && c1 == cols && dld == cols)
      TB_CUDA(cudaMemcpyAsync(dst + r0 * cols, src + r0 * cols, (size_t)(r1 - r0) * pitch, cudaMemcpyHostToDevice,
                              hs),
              "host to device copy");
    else
      TB_CUDA(cudaMemcpy2DAsync(dst + r0 * dld + c0, (size_t)dld * sizeof(double), src + r0 * cols + c0, pitch,
                                (size_t)(c1 - c0) * sizeof(double), (size_t)(r1 - r0), cudaMemcpyHostToDevice, hs),
              "host to device copy");
    trace_end(what, idx, t0, hs, (double)(r1 - r0) * (double)(c1 - c0) * sizeof(double));
    return TB_STATUS_OK;
  };
  auto gemm = [&](cudaStream_t cs, int64_t r0, int64_t r1, int64_t k0, int64_t k1, bool acc) -> int {
    cudaEvent_t t0 = mk(cudaEventDefault), t1 = mk(cudaEventDefault);
    if (!t0 || !t1) return cuda_fail(cudaGetLastError(), "event create");
    kt0.push_back(t0);
    kt1.push_back(t1);
    TB_CUDA(cudaEventRecord(t0, cs), "event record");
    int rc = launch(device, dA + r0 * lda_d + k0, lda_d, dB + k0 * ldb_d, ldb_d, dC + r0 * ldc_d, ldc_d, r1 - r0,
                    k1 - k0, n1, acc ? 1 : 0, tile_edge, variant, cs);
    if (rc) return rc;
    TB_CUDA(cudaEventRecord(t1, cs), "event record");
    return TB_STATUS_OK;
  };
  int nd2h = 0;
  // Rows [r0, r1) x columns [c0, c1) of C back to the host, after `cs`'s work so far.
  auto d2h = [&](cudaStream_t cs, int64_t r0, int64_t r1, int64_t c0, int64_t c1) -> int {
    cudaEvent_t done = mk(cudaEventDisableTiming);
    if (!done) return cuda_fail(cudaGetLastError(), "event create");
    TB_CUDA(cudaEventRecord(done, cs), "event record");
    TB_CUDA(cudaStreamWaitEvent(ds, done, 0), "stream wait");
    cudaEvent_t t0 = trace_begin(ds);
    if (ldc_d == n && c0 == 0 && c1 == n)
      TB_CUDA(cudaMemcpyAsync(out_c + r0 * n, dC + r0 * n, (size_t)((r1 - r0) * n) * sizeof(double),
                              cudaMemcpyDeviceToHost, ds),
              "device to host copy");
    else
      TB_CUDA(cudaMemcpy2DAsync(out_c + r0 * n + c0, (size_t)n * sizeof(double), dC + r0 * ldc_d + c0,
                                (size_t)ldc_d * sizeof(double), (size_t)(c1 - c0) * sizeof(double),
                                (size_t)(r1 - r0), cudaMemcpyDeviceToHost, ds),
              "device to host copy");
    trace_end("d2h_C", nd2h++, t0, ds, (double)(r1 - r0) * (c1 - c0) * sizeof(double));
    return TB_STATUS_OK;
  };

  const auto h_start = std::chrono::steady_clock::now();
  TB_CUDA(cudaEventRecord(e_start, hs), "event record");
  for (cudaStream_t cs : css) TB_CUDA(cudaStreamWaitEvent(cs, e_start, 0), "stream wait");
  TB_CUDA(cudaStreamWaitEvent(ds, e_start, 0), "stream wait");
  cudaEvent_t evTab = nullptr;
  if (fused) {
    // PIPE tables: flags zeroed and panel k-stage bounds uploaded on the copy
    // stream (copy engine, no SM: the phase-1 kernel may occupy every SM).
    if (!st.dtab) {
      TB_CUDA(cudaMalloc(&st.dtab, 512 * sizeof(int)), "pipeline table allocation");
      TB_CUDA(cudaHostAlloc(&st.htab, 512 * sizeof(int), cudaHostAllocDefault), "pipeline table allocation");
      std::memset(st.htab, 0, 512 * sizeof(int));
      st.htab[256] = 1;
    }
    for (int q = 0; q <= P; ++q) st.htab[128 + q] = (int)((pk[q] + 15) / 16);
    TB_CUDA(cudaMemcpyAsync(st.dtab, st.htab, (size_t)P * sizeof(int), cudaMemcpyHostToDevice, hs), "flags reset");
    TB_CUDA(cudaMemcpyAsync(st.dtab + 128, st.htab + 128, (size_t)(P + 1) * sizeof(int), cudaMemcpyHostToDevice, hs),
            "panel table");
    if (!(evTab = mk(cudaEventDisableTiming))) return cuda_fail(cudaGetLastError(), "event create");
    TB_CUDA(cudaEventRecord(evTab, hs), "event record");
  }
  // H2D: phase-1 panels (A slice, then B rows; in fused mode then the
  // panel's flag, copied after its data on the same stream), then the
  // phase-2 row blocks.
  for (int p = 0; p < P; ++p) {
    if (Mq > 0 && (s = h2d(dA, lda_d, a, k, 0, Mq, pk[p], pk[p + 1], "h2d_Ap", p))) return s;
    if ((s = h2d(dB, ldb_d, b, n, pk[p], pk[p + 1], 0, n, "h2d_Bp", p))) return s;
    TB_CUDA(cudaEventRecord(evP[p], hs), "event record");
    if (fused)
      TB_CUDA(cudaMemcpyAsync(st.dtab + p, st.htab + 256, sizeof(int), cudaMemcpyHostToDevice, hs), "panel flag");
  }
  for (int r = 0; r < R; ++r) {
    if ((s = h2d(dA, lda_d, a, k, rb[r], rb[r + 1], 0, k, "h2d_A", r))) return s;
    TB_CUDA(cudaEventRecord(evA[r], hs), "event record");
  }
  if (fused) {
    // Phase 1: one persistent launch; its producer waits on each panel's flag.
    const cudaStream_t cs = css[0];
    TB_CUDA(cudaStreamWaitEvent(cs, evTab, 0), "stream wait");
    cudaEvent_t t0 = mk(cudaEventDefault), t1 = mk(cudaEventDefault);
    if (!t0 || !t1) return cuda_fail(cudaGetLastError(), "event create");
    kt0.push_back(t0);
    kt1.push_back(t1);
    TB_CUDA(cudaEventRecord(t0, cs), "event record");
    if ((s = launch_pipe(device, dA, lda_d, dB, ldb_d, dC, ldc_d, Mq, k, n1, st.dtab + 128, st.dtab, P, cs))) return s;
    TB_CUDA(cudaEventRecord(t1, cs), "event record");
    if ((s = d2h(cs, 0, Mq, 0, n1))) return s;
  } else {
    // Phase 1: panel p of every row group once it has landed; row group g
    // stays on stream g, so its partial sums accumulate in panel order.
    for (int p = 0; p < P; ++p)
      for (int g = 0; g < G; ++g) {
        TB_CUDA(cudaStreamWaitEvent(css[g], evP[p], 0), "stream wait");
        if ((s = gemm(css[g], gb[g], gb[g + 1], pk[p], pk[p + 1], p > 0))) return s;
        if (p == P - 1 && (s = d2h(css[g], gb[g], gb[g + 1], 0, n1))) return s;
      }
  }
  // Phase 2: full-K row blocks, alternating streams (the first one on the
  // stream the fused phase-1 launch does not hold).
  // The column strip needs all of A and B; it is enqueued after the block
  // two from the end, on that block's stream, so it overlaps the last blocks
  // instead of trailing them.
  auto strip = [&](cudaStream_t cs) -> int {
    if (R > 0) TB_CUDA(cudaStreamWaitEvent(cs, evA[R - 1], 0), "stream wait");
    TB_CUDA(cudaStreamWaitEvent(cs, evP[P - 1], 0), "stream wait");
    cudaEvent_t t0 = mk(cudaEventDefault), t1 = mk(cudaEventDefault);
    if (!t0 || !t1) return cuda_fail(cudaGetLastError(), "event create");
    kt0.push_back(t0);
    kt1.push_back(t1);
    TB_CUDA(cudaEventRecord(t0, cs), "event record");
    int rc = launch_tiles(device, dA, lda_d, dB + n1, ldb_d, dC + n1, ldc_d, m, k, wr, 0, tile_edge,
                          TB_VARIANT_DMMA_TMA, cs, wr <= 16 ? kStrip128x16 : wr <= 32 ? kStrip128x32 : kStrip128x64);
    if (rc) return rc;
    TB_CUDA(cudaEventRecord(t1, cs), "event record");
    return d2h(cs, 0, m, n1, n);
  };
  const int strip_after = std::max(0, R - 3);
  if (strip_n && R == 0 && (s = strip(css[1]))) return s;
  for (int r = 0; r < R; ++r) {
    const cudaStream_t cs = css[(r + (fused ? 1 : 0)) & 1];
    TB_CUDA(cudaStreamWaitEvent(cs, evP[P - 1], 0), "stream wait");
    TB_CUDA(cudaStreamWaitEvent(cs, evA[r], 0), "stream wait");
    if ((s = gemm(cs, rb[r], rb[r + 1], 0, k, false))) return s;
    if ((s = d2h(cs, rb[r], rb[r + 1], 0, n1))) return s;
    if (strip_n && r == strip_after && (s = strip(cs))) return s;
  }
  TB_CUDA(cudaEventRecord(e_end, ds), "event record");
  const auto h_enq = std::chrono::steady_clock::now();
  // The call is synchronous: spin on the last D2H's event rather than a
  // blocking wait, whose wake-up latency would add to every call.
  static const bool block_sync = std::getenv("TB_SYNC_BLOCK") != nullptr;
  if (block_sync) {
    TB_CUDA(cudaEventSynchronize(e_end), "kernel execution");
  } else {
    cudaError_t q;
    while ((q = cudaEventQuery(e_end)) == cudaErrorNotReady) {
    }
    TB_CUDA(q, "kernel execution");
  }
  for (cudaStream_t cs : css) TB_CUDA(cudaStreamSynchronize(cs), "kernel execution");
  const auto h_sync = std::chrono::steady_clock::now();
  double ksum = 0.0;
  for (size_t i = 0; i < kt0.size(); ++i) {
    float ms = 0.f;
    TB_CUDA(cudaEventElapsedTime(&ms, kt0[i], kt1[i]), "event elapsed");
    ksum += ms;
  }
  float e_ms = 0.f;
  TB_CUDA(cudaEventElapsedTime(&e_ms, e_start, e_end), "event elapsed");
  if (trace) {
    auto us = [](std::chrono::steady_clock::time_point x, std::chrono::steady_clock::time_point y) {
      return std::chrono::duration<double, std::micro>(y - x).count();
    };
    std::fprintf(stderr, "TBHOST entry_to_start_us %.1f enqueue_us %.1f wait_us %.1f post_us %.1f\n",
                 us(h_entry, h_start), us(h_start, h_enq), us(h_enq, h_sync),
                 us(h_sync, std::chrono::steady_clock::now()));
    for (size_t i = 0; i < kt0.size(); ++i) tr.push_back({"gemm", (int)i, kt0[i], kt1[i], 0.0});
    for (const TraceRec& t : tr) {
      float a0 = 0.f, a1 = 0.f;
      cudaEventElapsedTime(&a0, e_start, t.t0);
      cudaEventElapsedTime(&a1, e_start, t.t1);
      std::fprintf(stderr, "TBTRACE %s %d %.4f %.4f %.0f\n", t.what, t.idx, a0, a1, t.bytes);
    }
  }
  *out_seconds = ksum * 1e-3;  // kernel-only: sum of the GEMM launch durations
  if (out_e2e_seconds) *out_e2e_seconds = (double)e_ms * 1e-3;
  return TB_STATUS_OK;
}

int tb_gpu_tiled_multiply_flat(int32_t device, const double* a, const double* b, int64_t m, int64_t k, int64_t n,
                               int32_t tile_edge, double* out_c, int64_t out_c_len, double* out_seconds) {
  return tb_gpu_tiled_multiply_flat_ex(device, a, b, m, k, n, tile_edge, TB_VARIANT_AUTO, out_c, out_c_len,
                                       out_seconds, nullptr);
}

int tb_pipeline_plan(int64_t m, int64_t k, int64_t n, int32_t sms, int32_t fused_ok, int64_t* out_mq,
                     int32_t* out_fused, int64_t* out_panels, int32_t max_panels, int32_t* out_npanels,
                     int64_t* out_blocks, int32_t max_blocks, int32_t* out_nblocks) {
  if (m < 1 || k < 1 || n < 1 || sms < 1 || !out_mq || !out_fused || !out_npanels || !out_nblocks) {
    set_err("bad pipeline-plan arguments");
    return TB_STATUS_BAD_DIMS;
  }
  const PipePlan pl = plan_pipeline(m, k, n, sms, fused_ok != 0);
  *out_mq = pl.Mq;
  *out_fused = pl.fused ? 1 : 0;
  *out_npanels = (int32_t)pl.pk.size();
  *out_nblocks = (int32_t)pl.rb.size();
  if ((int32_t)pl.pk.size() > max_panels || (int32_t)pl.rb.size() > max_blocks || !out_panels || !out_blocks) {
    set_err("plan needs %d panel and %d block bounds", (int)pl.pk.size(), (int)pl.rb.size());
    return TB_STATUS_OVER_LIMITS;
  }
  std::copy(pl.pk.begin(), pl.pk.end(), out_panels);
  std::copy(pl.rb.begin(), pl.rb.end(), out_blocks);
  return TB_STATUS_OK;
}

long long tb_kernel_launches(void) { return g_launches.load(std::memory_order_relaxed); }

void tb_release(void) {
  const int count = device_count_raw();
  for (int d = 0; d < count && d < kMaxDevices; ++d) {
    DeviceState& st = g_dev[d];
    std::lock_guard<std::mutex> lk_host(st.host_mu);
    std::lock_guard<std::mutex> lk(st.mu);
    DeviceGuard guard(d);
    if (st.ws) cudaFree(st.ws);
    st.ws = nullptr;
    st.ws_bytes = 0;
    if (st.cublas) cublasDestroy(st.cublas);
    st.cublas = nullptr;
    for (cudaStream_t* sp : {&st.host_stream, &st.host_stream2, &st.h2d_stream, &st.d2h_stream}) {
      if (*sp) cudaStreamDestroy(*sp);
      *sp = nullptr;
    }
    if (st.dtab) cudaFree(st.dtab);
    if (st.htab) cudaFreeHost(st.htab);
    st.dtab = nullptr;
    st.htab = nullptr;
    for (auto& pool : st.ev_pool) {
      for (cudaEvent_t e : pool) cudaEventDestroy(e);
      pool.clear();
    }
    for (auto& kv : st.stage_ws)
      if (kv.second.buf) cudaFree(kv.second.buf);
    st.stage_ws.clear();
    for (auto& kv : st.split_ws) {
      if (kv.second.partials) cudaFree(kv.second.partials);
      if (kv.second.counters) cudaFree(kv.second.counters);
    }
    st.split_ws.clear();
  }
}

}  // extern "C"
