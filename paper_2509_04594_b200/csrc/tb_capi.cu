// tb_capi.cu — the extern "C" boundary (include/tbgpu.h): status codes,
// the device-pointer entries (kernel-only CUDA-event timing), the host-buffer
// flat entry with its copy/compute pipeline, the cuBLAS DGEMM baseline and
// introspection. Internals: tb_state.cuh (state, tables, validation),
// tb_launch.cuh (schedules, workspaces, launches), tb_pipeline.cuh (the host
// pipeline's shape). One translation unit.
#include <cublas_v2.h>
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>
#include <dlfcn.h>

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
#include <string>

#include "../../include/tbgpu.h"
#include "dgemm_dmma.cuh"
#include "dgemm_paper.cuh"

#ifndef TB_VERSION
#define TB_VERSION "tbgpu 0.1.0 (sm_100a)"
#endif

#include "tb_state.cuh"
#include "tb_launch.cuh"
#include "tb_pipeline.cuh"
#include "tb_staging.cuh"
#include "tb_mgpu.cuh"

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
  // Pageable operands / output go through the pinned staging ring
  // (tb_staging.cuh); TB_STAGE=0 keeps plain pageable copies (A/B).
  const bool stage_ok = !(std::getenv("TB_STAGE") && std::strcmp(std::getenv("TB_STAGE"), "0") == 0);
  const bool pin_a = is_pinned(a), pin_b = is_pinned(b), pin_c = is_pinned(out_c);
  const bool stage_a = stage_ok && !pin_a, stage_b = stage_ok && !pin_b, stage_c = stage_ok && !pin_c;
  // A plain pageable cudaMemcpyAsync blocks the host (and can wait on device
  // work), so it must not be issued behind the flag-spinning fused phase-1
  // launch: without staging, pageable buffers take the event-gated
  // launch-per-panel form.
  const bool direct_pageable = !(pin_a || stage_a) || !(pin_b || stage_b) || !(pin_c || stage_c);
  StageRing& ring = g_ring[device];
  if ((stage_a || stage_b || stage_c) && (s = ring.ensure())) return s;
  struct PoolSession {  // copy workers spin (not sleep) between this call's staging copies
    CopyPool* pool;
    explicit PoolSession(CopyPool* p) : pool(p) {
      if (pool) pool->set_active(true);
    }
    ~PoolSession() {
      if (pool) pool->set_active(false);
    }
  } pool_session((stage_a || stage_b || stage_c) ? ring.pool.get() : nullptr);

  // Copy/compute/copy pipeline over four streams (H2D, two compute, D2H).
  //  Phase 1 (rank-k panels): the first Mq rows of C are computed as
  //    C[0:Mq] (+)= A[0:Mq, panel p] · B[panel p, :]
  //  while the panels stream in (A's panel slice by a 2D copy, B's panel as
  //  contiguous rows). The first panel is small, so the GEMM starts early;
  //  Mq is sized so a panel's GEMM (2·Mq·kp·n flops) outlasts its transfer
  //  (8·kp·(Mq+n) bytes) and compute does not wait on PCIe afterwards,
  //  capped so phase 2 still hides phase 1's C on its way back (the rates
  //  depend on which buffers are staged; tb_pipeline.cuh).
  //  Phase 2 (row blocks): the remaining rows of A arrive as contiguous
  //  blocks and run full-K GEMMs; every finished part of C is copied back at
  //  once, and the last blocks shrink so the final D2H is short.
  // Small problems degenerate to copy, GEMM, copy.
  const bool fused_ok = variant != TB_VARIANT_PAPER && variant != TB_VARIANT_DFMA &&
                        variant != TB_VARIANT_DMMA_CPASYNC && cfg_smem(0) <= g_dev[device].smem_optin &&
                        !direct_pageable;
  const PipePlan plan = plan_pipeline(m, k, n, g_dev[device].sms, fused_ok, stage_a || stage_b, stage_c);
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
    if ((src == a && stage_a) || (src == b && stage_b)) {
      // Pageable source: fill pinned slots on the host (pool threads), then
      // DMA each slot; a slot is refilled once its previous copy completed.
      // Rows wider than a slot go in column chunks of at most one slot.
      for (int64_t cc0 = c0; cc0 < c1; cc0 += StageRing::kSlotCols) {
        const int64_t cc1 = std::min(c1, cc0 + StageRing::kSlotCols);
        const size_t w = (size_t)(cc1 - cc0) * sizeof(double);
        const int64_t rows_per = std::max<int64_t>(1, (int64_t)(StageRing::kSlotBytes / w));
        for (int64_t r = r0; r < r1; r += rows_per) {
          const int64_t nr = std::min(rows_per, r1 - r);
          const int i = ring.next;
          ring.next = (ring.next + 1) % StageRing::kSlots;
          TB_CUDA(cudaEventSynchronize(ring.ev[i]), "staging slot wait");
          pool_copy_rows(*ring.pool, ring.slot[i], w, reinterpret_cast<const char*>(src + r * cols + cc0), pitch, w,
                         (size_t)nr);
          TB_CUDA(cudaMemcpy2DAsync(dst + r * dld + cc0, (size_t)dld * sizeof(double), ring.slot[i], w, w,
                                    (size_t)nr, cudaMemcpyHostToDevice, hs),
                  "host to device copy");
          TB_CUDA(cudaEventRecord(ring.ev[i], hs), "event record");
        }
      }
    } else if (c0 == 0 && c1 == cols && dld == cols)
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
    if (r1 <= r0) return TB_STATUS_OK;  // empty phase 1 (Mq = 0)
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
  // Rows [r0, r1) x columns [c0, c1) of C back to the host, after `cs`'s work
  // so far. A pageable output is drained through the staging ring at the end
  // of the enqueue (drain_c).
  struct D2HJob {
    cudaEvent_t ready;
    int64_t r0, r1, c0, c1;
  };
  std::vector<D2HJob> djobs;
  auto d2h = [&](cudaStream_t cs, int64_t r0, int64_t r1, int64_t c0, int64_t c1) -> int {
    if (r1 <= r0 || c1 <= c0) return TB_STATUS_OK;
    cudaEvent_t done = mk(cudaEventDisableTiming);
    if (!done) return cuda_fail(cudaGetLastError(), "event create");
    TB_CUDA(cudaEventRecord(done, cs), "event record");
    if (stage_c) {
      djobs.push_back({done, r0, r1, c0, c1});
      return TB_STATUS_OK;
    }
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
    st.htab[kAbortReadback] = 0;
    // Every flag and the abort word (tb::kPipeAbortWord) back to zero.
    TB_CUDA(cudaMemcpyAsync(st.dtab, st.htab, tb::kPipeFlagWords * sizeof(int), cudaMemcpyHostToDevice, hs),
            "flags reset");
    TB_CUDA(cudaMemcpyAsync(st.dtab + 128, st.htab + 128, (size_t)(P + 1) * sizeof(int), cudaMemcpyHostToDevice, hs),
            "panel table");
    if (!(evTab = mk(cudaEventDisableTiming))) return cuda_fail(cudaGetLastError(), "event create");
    TB_CUDA(cudaEventRecord(evTab, hs), "event record");
  }
  // Enqueue in data order, so that host-staged copies (which block this
  // thread while it fills pinned slots) never delay compute that could run:
  // the fused phase-1 launch first (its flags gate it), then per K-panel the
  // copies (+ the unfused form's panel GEMMs), then per row block its copy
  // and GEMM; the column strip once all of A has been enqueued.
  // Test hook (tests/test_gpu_parity.py): TB_PIPE_TEST_WITHHOLD=q never sets
  // panel q's flag, so the fused launch must abort on its flag-wait timeout.
  const char* wh = std::getenv("TB_PIPE_TEST_WITHHOLD");
  const int withhold = wh ? std::atoi(wh) : -1;
  // Any error return after the fused launch is enqueued sets its abort word
  // (on the H2D stream, which never waits on compute) and drains the call's
  // streams, so no launch is left spinning on flags that will not come.
  struct AbortGuard {
    DeviceState& st;
    cudaStream_t hs;
    const cudaStream_t* css;
    cudaStream_t ds;
    bool armed = false, done = false;
    ~AbortGuard() {
      if (!armed || done) return;
      cudaMemcpyAsync(st.dtab + tb::kPipeAbortWord, st.htab + 256, sizeof(int), cudaMemcpyHostToDevice, hs);
      for (cudaStream_t x : {hs, css[0], css[1], ds}) cudaStreamSynchronize(x);
      cudaGetLastError();
    }
  } abort_guard{st, hs, css, ds};
  auto phase1 = [&]() -> int {
    // Phase 1: one persistent launch; its producer waits on each panel's flag.
    const cudaStream_t cs = css[0];
    TB_CUDA(cudaStreamWaitEvent(cs, evTab, 0), "stream wait");
    cudaEvent_t t0 = mk(cudaEventDefault), t1 = mk(cudaEventDefault);
    if (!t0 || !t1) return cuda_fail(cudaGetLastError(), "event create");
    kt0.push_back(t0);
    kt1.push_back(t1);
    TB_CUDA(cudaEventRecord(t0, cs), "event record");
    int rc = launch_pipe(device, dA, lda_d, dB, ldb_d, dC, ldc_d, Mq, k, n1, st.dtab + 128, st.dtab, P,
                         pipe_timeout_ms(), cs);
    if (rc) return rc;
    abort_guard.armed = true;
    TB_CUDA(cudaEventRecord(t1, cs), "event record");
    // The launch's abort word, read back once the launch is done.
    TB_CUDA(cudaMemcpyAsync(st.htab + kAbortReadback, st.dtab + tb::kPipeAbortWord, sizeof(int),
                            cudaMemcpyDeviceToHost, cs),
            "abort word readback");
    return d2h(cs, 0, Mq, 0, n1);
  };
  // With pinned operands every panel copy and flag is enqueued (microseconds)
  // before the flag-spinning launch, so the running kernel never depends on
  // host progress: another thread's device-synchronising call (cudaFreeHost,
  // ...) cannot block an enqueue the kernel is spinning on. Staged operands
  // are enqueued while the pool fills slots (tens of ms), so there the launch
  // goes first and the call must not overlap such calls from other threads
  // (include/tbgpu.h).
  const bool phase1_first = fused && (stage_a || stage_b);
  if (phase1_first && (s = phase1())) return s;
  // H2D of phase-1 panels: A slice, then B rows; in fused mode then the
  // panel's flag, copied after its data on the same stream.
  for (int p = 0; p < P; ++p) {
    if (Mq > 0 && (s = h2d(dA, lda_d, a, k, 0, Mq, pk[p], pk[p + 1], "h2d_Ap", p))) return s;
    if ((s = h2d(dB, ldb_d, b, n, pk[p], pk[p + 1], 0, n, "h2d_Bp", p))) return s;
    TB_CUDA(cudaEventRecord(evP[p], hs), "event record");
    if (fused) {
      if (p != withhold)
        TB_CUDA(cudaMemcpyAsync(st.dtab + p, st.htab + 256, sizeof(int), cudaMemcpyHostToDevice, hs), "panel flag");
    } else {
      // Phase 1, unfused: panel p of every row group once it has landed; row
      // group g stays on stream g, so its partial sums accumulate in panel order.
      for (int g = 0; g < G; ++g) {
        TB_CUDA(cudaStreamWaitEvent(css[g], evP[p], 0), "stream wait");
        if ((s = gemm(css[g], gb[g], gb[g + 1], pk[p], pk[p + 1], p > 0))) return s;
        if (p == P - 1 && (s = d2h(css[g], gb[g], gb[g + 1], 0, n1))) return s;
      }
    }
  }
  if (fused && !phase1_first && (s = phase1())) return s;
  // The column strip needs all of A and B; it goes on the stream the last
  // row block does not use, after the block before it, so it overlaps the
  // last block instead of trailing it.
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
  if (strip_n && R == 0 && (s = strip(css[1]))) return s;
  // Phase 2: full-K row blocks, alternating streams (the first one on the
  // stream the fused phase-1 launch does not hold).
  for (int r = 0; r < R; ++r) {
    if ((s = h2d(dA, lda_d, a, k, rb[r], rb[r + 1], 0, k, "h2d_A", r))) return s;
    TB_CUDA(cudaEventRecord(evA[r], hs), "event record");
    const cudaStream_t cs = css[(r + (fused ? 1 : 0)) & 1];
    if (strip_n && r == R - 1 && (s = strip(css[(r + (fused ? 1 : 0) + 1) & 1]))) return s;
    TB_CUDA(cudaStreamWaitEvent(cs, evP[P - 1], 0), "stream wait");
    TB_CUDA(cudaStreamWaitEvent(cs, evA[r], 0), "stream wait");
    if ((s = gemm(cs, rb[r], rb[r + 1], 0, k, false))) return s;
    if ((s = d2h(cs, rb[r], rb[r + 1], 0, n1))) return s;
  }
  // Pageable output: drain C through the staging ring, in job order; up to
  // kSlots D2H copies in flight while the host copies finished slots out.
  if (stage_c) {
    struct Pending {
      int slot;
      double* dst;
      size_t w;
      int64_t rows;
    };
    std::vector<Pending> inflight;  // FIFO (front = oldest)
    size_t head = 0;
    auto pop = [&]() -> int {
      const Pending& pd = inflight[head++];
      TB_CUDA(cudaEventSynchronize(ring.ev[pd.slot]), "device to host copy");
      pool_copy_rows(*ring.pool, reinterpret_cast<char*>(pd.dst), (size_t)n * sizeof(double), ring.slot[pd.slot],
                     pd.w, pd.w, (size_t)pd.rows);
      return TB_STATUS_OK;
    };
    for (const D2HJob& jb : djobs) {
      TB_CUDA(cudaStreamWaitEvent(ds, jb.ready, 0), "stream wait");
      for (int64_t cc0 = jb.c0; cc0 < jb.c1; cc0 += StageRing::kSlotCols) {  // rows wider than a slot: chunks
        const int64_t cc1 = std::min(jb.c1, cc0 + StageRing::kSlotCols);
        const size_t w = (size_t)(cc1 - cc0) * sizeof(double);
        const int64_t rows_per = std::max<int64_t>(1, (int64_t)(StageRing::kSlotBytes / w));
        for (int64_t r = jb.r0; r < jb.r1; r += rows_per) {
          const int64_t nr = std::min(rows_per, jb.r1 - r);
          if (inflight.size() - head == (size_t)StageRing::kSlots && (s = pop())) return s;
          const int i = ring.next;
          ring.next = (ring.next + 1) % StageRing::kSlots;
          TB_CUDA(cudaStreamWaitEvent(ds, ring.ev[i], 0), "stream wait");  // the slot's last H2D has read it
          TB_CUDA(cudaMemcpy2DAsync(ring.slot[i], w, dC + r * ldc_d + cc0, (size_t)ldc_d * sizeof(double), w,
                                    (size_t)nr, cudaMemcpyDeviceToHost, ds),
                  "device to host copy");
          TB_CUDA(cudaEventRecord(ring.ev[i], ds), "event record");
          inflight.push_back({i, out_c + r * n + cc0, w, nr});
        }
      }
    }
    TB_CUDA(cudaEventRecord(e_end, ds), "event record");
    while (head < inflight.size())
      if ((s = pop())) return s;
  }
  if (!stage_c) TB_CUDA(cudaEventRecord(e_end, ds), "event record");
  const auto h_enq = std::chrono::steady_clock::now();
  // The call is synchronous: spin on the last D2H's event rather than a
  // blocking wait, whose wake-up latency would add to every call.
  static const bool block_sync = std::getenv("TB_SYNC_BLOCK") != nullptr;
  const char* what = "kernel execution";
  if (block_sync) {
    TB_CUDA(cudaEventSynchronize(e_end), what);
  } else {
    cudaError_t q;
    while ((q = cudaEventQuery(e_end)) == cudaErrorNotReady) {
    }
    TB_CUDA(q, what);
  }
  for (cudaStream_t cs : css) TB_CUDA(cudaStreamSynchronize(cs), "kernel execution");
  abort_guard.done = true;
  const auto h_sync = std::chrono::steady_clock::now();
  if (fused && st.htab[kAbortReadback] != 0) {
    set_err("kernel execution: fused phase-1 launch aborted, K-panel %d's flag not observed within %d ms "
            "(was this thread blocked while enqueueing? include/tbgpu.h); the product is invalid",
            st.htab[kAbortReadback] - 1, pipe_timeout_ms());
    return TB_STATUS_RUNTIME;
  }
#ifdef TB_TIMELINE
  pipe_timeline_report();
#endif
  // Kernel-only seconds (outSeconds): the union of the GEMM launches'
  // intervals — launches on the two compute streams overlap, so their sum
  // would count shared time twice.
  std::vector<std::pair<float, float>> iv(kt0.size());
  for (size_t i = 0; i < kt0.size(); ++i) {
    TB_CUDA(cudaEventElapsedTime(&iv[i].first, e_start, kt0[i]), "event elapsed");
    TB_CUDA(cudaEventElapsedTime(&iv[i].second, e_start, kt1[i]), "event elapsed");
  }
  std::sort(iv.begin(), iv.end());
  double ksum = 0.0, cover = -1e30;
  for (const auto& x : iv) {
    const double lo = std::max<double>(x.first, cover);
    if (x.second > lo) ksum += x.second - lo;
    cover = std::max<double>(cover, x.second);
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
  *out_seconds = ksum * 1e-3;
  if (out_e2e_seconds) *out_e2e_seconds = (double)e_ms * 1e-3;
  return TB_STATUS_OK;
}

int tb_gpu_tiled_multiply_flat(int32_t device, const double* a, const double* b, int64_t m, int64_t k, int64_t n,
                               int32_t tile_edge, double* out_c, int64_t out_c_len, double* out_seconds) {
  return tb_gpu_tiled_multiply_flat_ex(device, a, b, m, k, n, tile_edge, TB_VARIANT_AUTO, out_c, out_c_len,
                                       out_seconds, nullptr);
}

int tb_pipeline_plan(int64_t m, int64_t k, int64_t n, int32_t sms, int32_t fused_ok, int32_t staging,
                     int64_t* out_mq,
                     int32_t* out_fused, int64_t* out_panels, int32_t max_panels, int32_t* out_npanels,
                     int64_t* out_blocks, int32_t max_blocks, int32_t* out_nblocks) {
  if (m < 1 || k < 1 || n < 1 || sms < 1 || !out_mq || !out_fused || !out_npanels || !out_nblocks) {
    set_err("bad pipeline-plan arguments");
    return TB_STATUS_BAD_DIMS;
  }
  const PipePlan pl = plan_pipeline(m, k, n, sms, fused_ok != 0, (staging & 1) != 0, (staging & 2) != 0);
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

int tb_dgemm_mgpu(int32_t ndev, const int32_t* devices, const double* const* A_rows, const double* B_root,
                  double* const* B_replicas, double* const* C_rows, const int64_t* rows, int64_t k, int64_t n,
                  int32_t variant, double* out_kernel_seconds_max, double* out_total_seconds) {
  return mgpu_run(ndev, devices, A_rows, B_root, B_replicas, C_rows, rows, k, n, variant, out_kernel_seconds_max,
                  out_total_seconds);
}

int tb_copy2d_async(void* dst, int64_t dpitch_bytes, const void* src, int64_t spitch_bytes, int64_t width_bytes,
                    int64_t rows, void* cuda_stream) {
  if (!dst || !src || width_bytes < 0 || rows < 0 || dpitch_bytes < width_bytes || spitch_bytes < width_bytes) {
    set_err("bad 2D copy arguments");
    return TB_STATUS_BAD_DIMS;
  }
  if (width_bytes == 0 || rows == 0) return TB_STATUS_OK;
  TB_CUDA(cudaMemcpy2DAsync(dst, (size_t)dpitch_bytes, src, (size_t)spitch_bytes, (size_t)width_bytes, (size_t)rows,
                            cudaMemcpyDefault, static_cast<cudaStream_t>(cuda_stream)),
          "2D copy");
  return TB_STATUS_OK;
}

long long tb_kernel_launches(void) { return g_launches.load(std::memory_order_relaxed); }

namespace {
void json_str(std::string& js, const char* key, const char* val) {
  js += "\"";
  js += key;
  js += "\":";
  if (!val) {
    js += "null,";
    return;
  }
  js += "\"";
  for (const char* c = val; *c; ++c) {
    if (*c == '"' || *c == '\\') js += '\\';
    if ((unsigned char)*c >= 0x20) js += *c;
  }
  js += "\",";
}
void json_num(std::string& js, const char* key, long long v) {
  js += "\"";
  js += key;
  js += "\":" + std::to_string(v) + ",";
}
int json_out(std::string& js, char* buf, int64_t len) {
  if (!js.empty() && js.back() == ',') js.pop_back();
  if ((int64_t)js.size() + 1 > len) {
    set_err("buffer of %lld bytes too small for %lld bytes of JSON", (long long)len, (long long)js.size() + 1);
    return TB_STATUS_OVER_LIMITS;
  }
  std::memcpy(buf, js.c_str(), js.size() + 1);
  return TB_STATUS_OK;
}
const char* loaded_from(const void* sym) {
  Dl_info di;
  return dladdr(sym, &di) && di.dli_fname ? di.dli_fname : nullptr;
}
}  // namespace

int tb_runtime_info(int32_t device, char* buf, int64_t buf_len) {
  if (!buf || buf_len < 3) {
    set_err("null or tiny output buffer");
    return TB_STATUS_BAD_DIMS;
  }
  std::string js = "{";
  json_str(js, "library", TB_VERSION);
  json_str(js, "library_path", loaded_from((const void*)&tb_runtime_info));
  int rt = 0, drv = 0;
  if (cudaRuntimeGetVersion(&rt) != cudaSuccess) cudaGetLastError();
  if (cudaDriverGetVersion(&drv) != cudaSuccess) cudaGetLastError();
  json_num(js, "cuda_runtime_version", rt);
  json_num(js, "cuda_driver_version", drv);
  json_num(js, "cuda_runtime_header_version", CUDART_VERSION);
  // The cuBLAS that is actually loaded: in a process that imported torch
  // first, the dynamic linker binds libcublas.so.12 to torch's wheel copy,
  // not the toolkit's (same soname), so report the runtime version and path.
  int cmaj = -1, cmin = -1, cpat = -1;
  cublasGetProperty(MAJOR_VERSION, &cmaj);
  cublasGetProperty(MINOR_VERSION, &cmin);
  cublasGetProperty(PATCH_LEVEL, &cpat);
  char ver[64];
  std::snprintf(ver, sizeof(ver), "%d.%d.%d", cmaj, cmin, cpat);
  json_str(js, "cublas_version", ver);
  json_num(js, "cublas_header_version", CUBLAS_VERSION);
  const char* cub_path = loaded_from((const void*)&cublasCreate_v2);
  json_str(js, "cublas_path", cub_path);
  // FP64 emulation: cuBLAS 12.x's emulation API and its math-mode bits
  // cover FP32 (BF16x9) only; probe the API by name (absent before 12.9).
  void* h = cub_path ? dlopen(cub_path, RTLD_NOLOAD | RTLD_LAZY) : nullptr;
  using GetEmu = int (*)(cublasHandle_t, int*);
  GetEmu get_emu = h ? reinterpret_cast<GetEmu>(dlsym(h, "cublasGetEmulationStrategy")) : nullptr;
  json_str(js, "cublas_emulation_strategy_env", std::getenv("CUBLAS_EMULATION_STRATEGY"));
  json_str(js, "fp64_emulation", "none: no FP64 emulation in cuBLAS 12.x (emulation enums are FP32-only)");
  const int count = device_count_raw();
  json_num(js, "device_count", count);
  if (device >= 0 && device < count && device < kMaxDevices) {
    DeviceGuard guard(device);
    cudaDeviceProp pr;
    if (cudaGetDeviceProperties(&pr, device) == cudaSuccess) {
      json_num(js, "device", device);
      json_str(js, "gpu_name", pr.name);
      json_num(js, "sm_count", pr.multiProcessorCount);
      json_num(js, "compute_capability", pr.major * 10 + pr.minor);
      json_num(js, "l2_bytes", pr.l2CacheSize);
      json_num(js, "hbm_bytes", (long long)pr.totalGlobalMem);
      json_num(js, "smem_optin_bytes", (long long)pr.sharedMemPerBlockOptin);
      int clk = 0, mclk = 0;
      cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, device);
      cudaDeviceGetAttribute(&mclk, cudaDevAttrMemoryClockRate, device);
      json_num(js, "sm_clock_max_khz", clk);
      json_num(js, "mem_clock_max_khz", mclk);
    } else {
      cudaGetLastError();
    }
    if (ensure_cublas(device) == TB_STATUS_OK) {
      cublasMath_t mode = CUBLAS_DEFAULT_MATH;
      cublasGetMathMode(g_dev[device].cublas, &mode);
      json_num(js, "cublas_math_mode", (int)mode);
      json_str(js, "cublas_math_mode_name", mode == CUBLAS_DEFAULT_MATH ? "CUBLAS_DEFAULT_MATH" : "other");
      int emu = -1;
      if (get_emu && get_emu(g_dev[device].cublas, &emu) == 0)
        json_num(js, "cublas_emulation_strategy", emu);
      else
        json_str(js, "cublas_emulation_strategy", nullptr);
    }
  }
  if (h) dlclose(h);
  if (js.back() == ',') js.pop_back();
  js += "}";
  return json_out(js, buf, buf_len);
}

int tb_launch_plan(int64_t m, int64_t k, int64_t n, int32_t variant, int32_t sms, char* buf, int64_t buf_len) {
  if (m < 1 || k < 1 || n < 1 || sms < 1 || variant < 0 || variant >= TB_NUM_VARIANTS || !buf || buf_len < 3) {
    set_err("bad launch-plan arguments");
    return TB_STATUS_BAD_DIMS;
  }
  PlanRec rec;
  rec.sms = sms;
  rec.json = "[";
  g_plan = &rec;
  // Packed, 16-byte aligned operands (torch CUDA tensors); nothing is read.
  const double* fake = reinterpret_cast<const double*>(256);
  const int s = launch(0, fake, k, fake, n, const_cast<double*>(fake), n, m, k, n, 0, TB_DEFAULT_TILE_EDGE, variant,
                       nullptr);
  g_plan = nullptr;
  if (s) return s;
  if (rec.json.back() == ',') rec.json.pop_back();
  rec.json += "]";
  return json_out(rec.json, buf, buf_len);
}

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
    g_ring[d].release();
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
    {
      std::lock_guard<std::mutex> lk_side(st.side_mu);
      for (auto& kv : st.side) {
        if (kv.second.s) cudaStreamSynchronize(kv.second.s);
        if (kv.second.s) cudaStreamDestroy(kv.second.s);
        if (kv.second.fork) cudaEventDestroy(kv.second.fork);
        if (kv.second.join) cudaEventDestroy(kv.second.join);
      }
      st.side.clear();
    }
  }
}

}  // extern "C"
