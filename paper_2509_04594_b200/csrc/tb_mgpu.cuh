// tb_mgpu.cuh — tb_dgemm_mgpu: the row-sharded multi-GPU GEMM from ONE
// process driving several devices (included by
// tb_capi.cu only). The one-process-per-GPU form is multigpu.ShardedGemm
// over torch.distributed / NCCL; this entry is for a host that owns all the
// devices (the reference's executor model, executor.ts:78-147).
//
// Device i owns rows rows[i] of A and C (A_rows[i], C_rows[i], packed,
// row-major). B lives on devices[0] and is forwarded in K-panels along the
// chain devices[0] -> devices[1] -> ... with peer copies (cudaMemcpyPeerAsync:
// copy engines over NVLink / NVSwitch, no SM time); device i's panel-p GEMM
// C_i (+)= A_i[:, panel] · B[panel, :] runs as soon as panel p has landed
// there, so the forward of panel p+1 overlaps the GEMM of panel p. Every link
// of the chain carries B once (a flat broadcast from devices[0] would push
// (ndev-1)·8kn bytes through one GPU's NVLink ports). The first panel is
// short: only its forward is exposed before the last device starts.
#pragma once

namespace {

constexpr int kMaxMgpu = 64;

// K-panel bounds: one panel when nothing is forwarded; else a short first
// panel (128 rows of B: the only forward exposed before the chain's last
// device starts), then panels growing 4x up to TB_MGPU_PANEL (default 4096)
// rows. Forwarding is ~6x faster per k-row than a 1250-row shard multiplies
// (8n / ~700 GB/s vs 2·rows·n / 36 TF/s), so panel p+1 lands well before
// panel p's GEMM ends, and few panels keep the per-panel cost (a C re-read
// plus a wave tail: N = 10000, one entry, 1024-row panels 58.3 ms, 4096
// 56.3 ms, single GEMM 55.3 ms) small. Bounds are even, so every panel's A
// slice and B rows keep 16-byte alignment for TMA.
std::vector<int64_t> mgpu_panels(int64_t k, int ndev) {
  std::vector<int64_t> pk{0};
  int64_t cap = 4096;
  if (const char* e = std::getenv("TB_MGPU_PANEL")) {
    const long long v = std::atoll(e);
    if (v >= 2) cap = v & ~1LL;
  }
  for (int64_t at = 0, step = std::min<int64_t>(128, cap); ndev > 1 && at < k;) {
    const int64_t nx = at + step >= k - step / 4 ? k : at + step;
    pk.push_back(nx);
    at = nx;
    step = std::min(cap, step * 4);
  }
  if (pk.back() != k) pk.push_back(k);
  return pk;
}

struct MgpuEvents {  // destroyed on every exit path
  std::vector<std::pair<int, cudaEvent_t>> evs;
  cudaEvent_t make(int dev, unsigned flags) {
    DeviceGuard g(dev);
    cudaEvent_t e = nullptr;
    if (cudaEventCreateWithFlags(&e, flags) != cudaSuccess) return nullptr;
    evs.emplace_back(dev, e);
    return e;
  }
  ~MgpuEvents() {
    for (auto& de : evs) {
      DeviceGuard g(de.first);
      cudaEventDestroy(de.second);
    }
  }
};

int mgpu_run(int32_t ndev, const int32_t* devices, const double* const* A_rows, const double* B_root,
             double* const* B_replicas, double* const* C_rows, const int64_t* rows, int64_t k, int64_t n,
             int32_t variant, double* out_kernel_seconds_max, double* out_total_seconds) {
  if (ndev < 1 || ndev > kMaxMgpu || !devices || !A_rows || !B_root || !C_rows || !rows ||
      !out_kernel_seconds_max || (ndev > 1 && !B_replicas)) {
    set_err("bad multi-device arguments (ndev %d, 1..%d devices, non-null tables)", ndev, kMaxMgpu);
    return TB_STATUS_BAD_DIMS;
  }
  if (k < 1 || n < 1) {
    set_err("dimensions must be positive integers, got k=%lld n=%lld", (long long)k, (long long)n);
    return TB_STATUS_BAD_DIMS;
  }
  int s = TB_STATUS_OK;
  for (int i = 0; i < ndev; ++i) {
    if ((s = check_device(devices[i]))) return s;
    if (rows[i] < 0 || (rows[i] > 0 && (!A_rows[i] || !C_rows[i])) || (i > 0 && !B_replicas[i])) {
      set_err("device entry %d: bad rows (%lld) or null buffer", i, (long long)rows[i]);
      return TB_STATUS_BAD_DIMS;
    }
    if (rows[i] > 0 && (s = validate(rows[i], k, n, TB_DEFAULT_TILE_EDGE, variant, devices[i]))) return s;
  }
  if (variant == TB_VARIANT_PAPER) {
    set_err("the paper kernel has no accumulate form; use auto / dmma / dfma");
    return TB_STATUS_BAD_DIMS;
  }
  // One in-flight host call per device; lock in device
  // order so concurrent multi-device calls cannot deadlock.
  std::vector<int> uniq(devices, devices + ndev);
  std::sort(uniq.begin(), uniq.end());
  uniq.erase(std::unique(uniq.begin(), uniq.end()), uniq.end());
  std::vector<std::unique_lock<std::mutex>> locks;
  for (int d : uniq) locks.emplace_back(g_dev[d].host_mu);
  DeviceGuard restore(devices[0]);
  for (int d : uniq) {
    DeviceState& st = g_dev[d];
    TB_CUDA(cudaSetDevice(d), "set device");
    for (cudaStream_t* sp : {&st.host_stream, &st.h2d_stream})
      if (!*sp) TB_CUDA(cudaStreamCreateWithFlags(sp, cudaStreamNonBlocking), "stream create");
  }
  // Peer access along the chain (each device pulls from its predecessor).
  for (int i = 1; i < ndev; ++i) {
    const int d = devices[i], src = devices[i - 1];
    if (d == src) continue;
    int can = 0;
    TB_CUDA(cudaDeviceCanAccessPeer(&can, d, src), "peer query");
    if (!can) continue;  // cudaMemcpyPeerAsync still works (staged by the driver)
    TB_CUDA(cudaSetDevice(d), "set device");
    const cudaError_t e = cudaDeviceEnablePeerAccess(src, 0);
    if (e == cudaErrorPeerAccessAlreadyEnabled) cudaGetLastError();
    else TB_CUDA(e, "enable peer access");
  }
  const std::vector<int64_t> pk = mgpu_panels(k, ndev);
  const int P = (int)pk.size() - 1;
  auto bsrc = [&](int i) -> const double* { return i == 0 ? B_root : B_replicas[i]; };
  MgpuEvents ev;
  std::vector<std::vector<cudaEvent_t>> landed(ndev, std::vector<cudaEvent_t>(P, nullptr));
  std::vector<cudaEvent_t> t0(ndev, nullptr), t1(ndev, nullptr);
  for (int i = 0; i < ndev; ++i) {
    if (rows[i] > 0 && (!(t0[i] = ev.make(devices[i], cudaEventDefault)) ||
                        !(t1[i] = ev.make(devices[i], cudaEventDefault))))
      return cuda_fail(cudaGetLastError(), "event create");
    for (int p = 0; i > 0 && p < P; ++p)
      if (!(landed[i][p] = ev.make(devices[i], cudaEventDisableTiming)))
        return cuda_fail(cudaGetLastError(), "event create");
  }
  const auto h0 = std::chrono::steady_clock::now();
  for (int p = 0; p < P; ++p) {
    const int64_t k0 = pk[p], k1 = pk[p + 1];
    // Forward panel p one hop down the chain.
    for (int i = 1; i < ndev; ++i) {
      const int d = devices[i];
      const cudaStream_t cp = g_dev[d].h2d_stream;
      TB_CUDA(cudaSetDevice(d), "set device");
      if (i >= 2) TB_CUDA(cudaStreamWaitEvent(cp, landed[i - 1][p], 0), "stream wait");
      TB_CUDA(cudaMemcpyPeerAsync(B_replicas[i] + k0 * n, d, bsrc(i - 1) + k0 * n, devices[i - 1],
                                  (size_t)((k1 - k0) * n) * sizeof(double), cp),
              "peer copy of a B panel");
      TB_CUDA(cudaEventRecord(landed[i][p], cp), "event record");
    }
    // Panel-p GEMMs where the panel has landed.
    for (int i = 0; i < ndev; ++i) {
      if (rows[i] == 0) continue;
      const int d = devices[i];
      const cudaStream_t cs = g_dev[d].host_stream;
      TB_CUDA(cudaSetDevice(d), "set device");
      if (i > 0) TB_CUDA(cudaStreamWaitEvent(cs, landed[i][p], 0), "stream wait");
      if (p == 0) TB_CUDA(cudaEventRecord(t0[i], cs), "event record");
      if ((s = launch(d, A_rows[i] + k0, k, bsrc(i) + k0 * n, n, C_rows[i], n, rows[i], k1 - k0, n, p > 0,
                      TB_DEFAULT_TILE_EDGE, variant, cs)))
        return s;
      if (p == P - 1) TB_CUDA(cudaEventRecord(t1[i], cs), "event record");
    }
  }
  for (int d : uniq) {
    TB_CUDA(cudaSetDevice(d), "set device");
    TB_CUDA(cudaStreamSynchronize(g_dev[d].h2d_stream), "peer copy");
    TB_CUDA(cudaStreamSynchronize(g_dev[d].host_stream), "kernel execution");
  }
  const double total = std::chrono::duration<double>(std::chrono::steady_clock::now() - h0).count();
  double kmax = 0.0;
  for (int i = 0; i < ndev; ++i) {
    if (rows[i] == 0) continue;
    float ms = 0.f;
    TB_CUDA(cudaSetDevice(devices[i]), "set device");
    TB_CUDA(cudaEventElapsedTime(&ms, t0[i], t1[i]), "event elapsed");
    kmax = std::max(kmax, (double)ms * 1e-3);
  }
  *out_kernel_seconds_max = kmax;
  if (out_total_seconds) *out_total_seconds = total;
  return TB_STATUS_OK;
}

}  // namespace
