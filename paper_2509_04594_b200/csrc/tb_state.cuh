// tb_state.cuh — library-internal state and tables (included by tb_capi.cu
// only): kernel instantiation tables (pipeline shapes, 64-row / edge-strip /
// PIPE kernels, choose_bm), error reporting, per-device state, TMA descriptor
// encoding, operand checks and launch validation (limits.ts:58-79).
#pragma once

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
  kStrip64x128,
  // Main-tile shapes besides 128 x 128 / 64 x 128 (TMA + DMMA), for small
  // and ragged problems (tile_for_shape).
  kTile64x64,
  kTile96x128,
  kTile128x96,
  kTile96x96,
  kTile64x96,
  kTile128x64,
  kTile64x128,  // TMA 64 x 128 with 32-deep stages (the 64-row kernel kStrip64x128 keeps 16-deep ones)
  kTile64x64d,  // 64 x 64 with 64-deep stages (SUB 4 x 3): fewer stage boundaries, shallower ring
  kTile96x96t,  // 96 x 96 with 48-deep stages (SUB 3 x 3)
  kNumStripCfgs
};
// Narrow tiles do little work per 16-deep k-slab, so a strip stage holds
// several sub-slabs (SUB x 16 k) to amortise the per-stage barrier round trip.
template <int BM, int BN, int WM, int SUB, int STAGES>
struct StripK {
  static void* fn() {
    return (void*)tb::dgemm_dmma_kernel<SUB, STAGES, tb::Loader::TMA, tb::Math::DMMA, BM, false, BN, WM>;
  }
  static constexpr int smem() { return tb::dmma_smem_bytes<SUB, STAGES, BM, BN>(); }
};
struct StripInfo {
  int bm, bn, sub;
  void* fn;
  int smem;
};
StripInfo strip_info(int c) {
  switch (c) {
    case kStrip128x16: return {128, 16, 4, StripK<128, 16, 8, 4, 3>::fn(), StripK<128, 16, 8, 4, 3>::smem()};
    case kStrip128x32: return {128, 32, 2, StripK<128, 32, 8, 2, 5>::fn(), StripK<128, 32, 8, 2, 5>::smem()};
    case kStrip128x64: return {128, 64, 2, StripK<128, 64, 4, 2, 4>::fn(), StripK<128, 64, 4, 2, 4>::smem()};
    case kStrip16x128: return {16, 128, 4, StripK<16, 128, 1, 4, 3>::fn(), StripK<16, 128, 1, 4, 3>::smem()};
    case kStrip32x128: return {32, 128, 2, StripK<32, 128, 1, 2, 5>::fn(), StripK<32, 128, 1, 2, 5>::smem()};
    case kTile64x64: return {64, 64, 2, StripK<64, 64, 2, 2, 6>::fn(), StripK<64, 64, 2, 2, 6>::smem()};
    case kTile64x64d: return {64, 64, 4, StripK<64, 64, 2, 4, 3>::fn(), StripK<64, 64, 2, 4, 3>::smem()};
    case kTile96x128: return {96, 128, 1, StripK<96, 128, 2, 1, 7>::fn(), StripK<96, 128, 2, 1, 7>::smem()};
    case kTile128x96: return {128, 96, 1, StripK<128, 96, 4, 1, 7>::fn(), StripK<128, 96, 4, 1, 7>::smem()};
    case kTile96x96: return {96, 96, 2, StripK<96, 96, 4, 2, 4>::fn(), StripK<96, 96, 4, 2, 4>::smem()};
    case kTile96x96t: return {96, 96, 3, StripK<96, 96, 4, 3, 3>::fn(), StripK<96, 96, 4, 3, 3>::smem()};
    case kTile64x96: return {64, 96, 2, StripK<64, 96, 4, 2, 5>::fn(), StripK<64, 96, 4, 2, 5>::smem()};
    case kTile64x128: return {64, 128, 2, StripK<64, 128, 2, 2, 4>::fn(), StripK<64, 128, 2, 2, 4>::smem()};
    case kTile128x64: return {128, 64, 2, StripK<128, 64, 4, 2, 4>::fn(), StripK<128, 64, 4, 2, 4>::smem()};
    default: return {0, 0, 1, nullptr, 0};
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
constexpr int kAbortReadback = 300;  // DeviceState::htab slot
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
  std::mutex stage_mu;   // a staged launch's re-pitch + GEMM enqueue (tb_launch.cuh launch())
  std::mutex cublas_mu;  // cublasSetStream + cublasDgemm on the shared handle
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
  struct SideStream {  // per caller stream: the edge-strip launches' stream + fork / join events
    cudaStream_t s = nullptr;
    cudaEvent_t fork = nullptr, join = nullptr;
  };
  std::map<cudaStream_t, SideStream> side;
  std::mutex side_mu;  // one fork / launch / join sequence at a time per device
  std::vector<cudaEvent_t> ev_pool[2];  // host-buffer entry: [timing, no-timing] events
  int* dtab = nullptr;                  // host-buffer entry: [0,128) panel flags (+ abort word at
                                        // tb::kPipeAbortWord), [128,256) panel k-stages
  int* htab = nullptr;                  // pinned: [0,128) zeros, [128,256) panel k-stages, [256] = 1,
                                        // [kAbortReadback] the last fused launch's abort word
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

// The per-device cuBLAS handle for the baseline, created once with the math
// mode pinned to CUBLAS_DEFAULT_MATH: native FP64 DGEMM (the math-mode bits
// that enable tensor-op / emulated paths apply to FP32 only in cuBLAS 12.x,
// and no FP64 emulation exists before CUDA 13), recorded by tb_runtime_info.
int ensure_cublas(int dev) {
  DeviceState& st = g_dev[dev];
  std::lock_guard<std::mutex> lk(st.mu);
  if (st.cublas) return TB_STATUS_OK;
  cublasHandle_t h = nullptr;
  if (cublasCreate(&h) != CUBLAS_STATUS_SUCCESS) {
    set_err("cublasCreate failed");
    return TB_STATUS_RUNTIME;
  }
  if (cublasSetMathMode(h, CUBLAS_DEFAULT_MATH) != CUBLAS_STATUS_SUCCESS) {
    cublasDestroy(h);
    set_err("cublasSetMathMode(CUBLAS_DEFAULT_MATH) failed");
    return TB_STATUS_RUNTIME;
  }
  st.cublas = h;
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
  for (int c = kStrip128x16; c < kNumStripCfgs; ++c) {
    const StripInfo si = strip_info(c);
    if (si.fn && si.smem <= st.smem_optin)  // kStrip64x128 is the 64-row kernel (small_kernel), set below
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


}  // namespace
