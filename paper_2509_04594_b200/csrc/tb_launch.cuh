// tb_launch.cuh — enqueueing GEMMs (included by tb_capi.cu only): the
// persistent schedule shapes, stream-K / staging workspaces, the re-pitch
// staging kernel, launch() with its edge-strip split, launch_tiles(), the
// host pipeline's PIPE-mode launch and the event-timed synchronous call.
#pragma once

namespace {

// Dry-run recorder (tb_launch_plan): while set on this thread, launch() and
// launch_tiles() describe the launches they would enqueue (JSON objects
// appended to `json`) on a device with `sms` SMs instead of enqueueing them.
struct PlanRec {
  std::string json;
  int sms = 148;
};
thread_local PlanRec* g_plan = nullptr;
int dev_sms(int dev) { return g_plan ? g_plan->sms : g_dev[dev].sms; }

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

// dp_only: the cost model's data-parallel alternative (choose_tile).
Schedule plan_schedule(int64_t tiles, int num_k, int sms, bool dp_only = false) {
  static const int forced = [] {
    const char* e = std::getenv("TB_SCHED");
    if (e && std::strcmp(e, "dp") == 0) return 1;
    if (e && std::strcmp(e, "sk") == 0) return 2;  // always the stream-K shape (previous default)
    return 0;
  }();
  Schedule sc{sms, (int)tiles, 0, 1, 1, num_k};
  const int64_t rem = tiles % sms;
  if (forced == 1 || rem == 0 || dp_only) {
    sc.grid = (int)std::min<int64_t>(tiles, sms);  // no idle CTAs for a partial single wave
    return sc;
  }
  // A single wave >= 75 % full runs data-parallel: splitting every tile of a single wave costs about a
  // quarter of a tile's k-loop in partial traffic and fixups (N = 1500, 144 tiles: 28.6 -> 31.2;
  // N = 1000 on 64-row tiles, 128 tiles: 23.3 -> 25.9; N = 900, 120 tiles: 19.5 -> 20.5; at 61 %,
  // N = 800, stream-K stays ahead 18.2 vs 15.9 TFLOP/s). With more waves the stream-K tail wins
  // (N = 4000 / 6000 at 92 %: 34.12 / 35.84 vs 33.99 / 35.76).
  if (forced == 0 && tiles < sms && 4 * tiles >= 3 * sms) {
    sc.grid = (int)tiles;
    return sc;
  }
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
  // Segments per tile: a tile's num_k iterations meet at most
  // floor((num_k - 1) / ipc) + 2 CTA ranges (an upper bound — it only sizes
  // the partial-tile workspace; the kernel derives each tile's exact count).
  const int max_seg = (int)std::min<int64_t>((num_k - 1) / ipc + 2, sms);
  sc.max_seg = max_seg;
  return sc;
}

// ----------------------------------------------------------------------------
// Tile-shape chooser (TMA + DMMA launches). Every main-tile configuration the
// library instantiates, under its stream-K schedule (plan_schedule) and
// purely data-parallel, is costed with one launch model and the cheapest runs:
//
//   t = w * t_stage + fixups * F * s + units * E * s + R,   s = bm*bn / 8192
//
// w = k-stages on the busiest CTA (data-parallel tiles + its stream-K
// iterations), t_stage = bm*bn*16*SUB FMAs at 64 FMA/clk/SM times the
// configuration's steady-state efficiency, fixups = the stream-K segment
// reductions on that CTA (2 when the launch splits tiles), units = its tile
// epilogues, R = launch + pipeline fill. The efficiencies, F = 2.31 us and
// E = 0.34 us were fitted (tools/tile_model_fit.py, rms log error 0.55 %) to
// the kernel-only sweep of all eleven configurations x both schedules at
// N = 1000..3000 step 50 and 3500..8192 on one B200
// (profiles/r02_tile_sched_sweep.jsonl); there the model's pick is within
// 2.3 % of the fastest measured (configuration, schedule) at every N and
// 0.2 % off on the geometric mean (tests/test_tile_model.py replays it).
// R cancels between single launches; 4 us per extra launch prices the
// edge-strip plan: wide problems with ragged m / n run as 128 x 128 main
// tiles plus remainder strips, each a launch of its own (see launch()).
struct TileCfg {
  int slot;  // launch_tiles' `strip` argument: -1 = 128 x 128, kStrip64x128 = 64-row kernel, else kTile*
  int bm, bn, sub;
  double eff;
};
// Largest tiles first: a later (smaller) shape must beat the best so far by
// kPreferLarger to be picked, so near-ties go to the shape with less
// operand traffic per flop (long-K shards re-read panels from DRAM, §3.1 of
// 128 x 64 and 128 x 128 are equally fast at N = 8192, but the
// larger tile halves B's reads).
constexpr TileCfg kTileCfgs[] = {
    {-1, 128, 128, 1, 0.9691},         {kTile128x96, 128, 96, 1, 0.9701}, {kTile96x128, 96, 128, 1, 0.9705},
    {kTile128x64, 128, 64, 2, 0.9710}, {kTile64x128, 64, 128, 2, 0.9670}, {kStrip64x128, 64, 128, 1, 0.9530},
    {kTile96x96t, 96, 96, 3, 0.9776},  {kTile96x96, 96, 96, 2, 0.9731},   {kTile64x96, 64, 96, 2, 0.9688},
    {kTile64x64d, 64, 64, 4, 0.9632},  {kTile64x64, 64, 64, 2, 0.9480},
};
constexpr double kPreferLarger = 2e-3;
// Edge-strip shapes (their launches carry the narrow tiles' lower efficiency:
// N = 10000 strips measured 23.5 TFLOP/s including their fixups).
constexpr double kStripEff = 0.70;
constexpr double kModelF = 2.31e-6, kModelE = 0.344e-6, kModelR = 4e-6;
constexpr double kSmFmaPerSec = 64.0 * 1.965e9;

double model_seconds(int64_t m, int64_t n, int64_t k, int bm, int bn, int sub, double eff, int sms,
                     bool dp_only = false) {
  const int64_t tiles = ((m + bm - 1) / bm) * ((n + bn - 1) / bn);
  const int num_k = (int)((k + 16 * sub - 1) / (16 * sub));
  const Schedule sc = plan_schedule(tiles, num_k, sms, dp_only);
  const double t_stage = (double)bm * bn * 16 * sub / (kSmFmaPerSec * eff);
  const double s = (double)bm * bn / 8192.0;
  double w, units, fix;
  if (sc.sk == 0) {
    units = (double)((tiles + sc.grid - 1) / sc.grid);
    w = units * sc.num_k;
    fix = 0;
  } else {
    const double dpw = (double)(sc.dp / sc.grid);
    w = dpw * sc.num_k + sc.ipc;
    units = dpw + (double)((sc.ipc + sc.num_k - 1) / sc.num_k) + 1;
    fix = 2;
  }
  return w * t_stage + fix * kModelF * s + units * kModelE * s + kModelR;
}

struct TileChoice {
  int slot;     // launch_tiles' strip argument for a single launch
  bool split;   // 128 x 128 main part + edge-strip launches instead
  bool dp;      // the single launch runs data-parallel (no stream-K split)
  double seconds;
};

// Edge-strip plan of launch(): bottom / right strip shapes for the ragged
// remainders (kStripNone when the remainder is 0 or wider than 64).
void strip_cfgs(int64_t m, int64_t n, int& bcfg, int& rcfg) {
  const int64_t hb = m % 128, wr = n % 128;
  bcfg = hb == 0 ? kStripNone : hb <= 16 ? kStrip16x128 : hb <= 32 ? kStrip32x128 : hb <= 64 ? kStrip64x128
                                                                                             : kStripNone;
  rcfg = wr == 0 ? kStripNone : wr <= 16 ? kStrip128x16 : wr <= 32 ? kStrip128x32 : wr <= 64 ? kStrip128x64
                                                                                             : kStripNone;
}

// split_mode: 0 = costed, -1 = never split, 1 = split whenever the shape allows.
TileChoice choose_tile_uncached(int64_t m, int64_t n, int64_t k, int sms, int split_mode) {
  TileChoice best{-1, false, false, 1e30};
  for (const TileCfg& c : kTileCfgs)
    for (bool dp : {false, true}) {
      const double t = model_seconds(m, n, k, c.bm, c.bn, c.sub, c.eff, sms, dp);
      const bool same_shape = best.slot == c.slot && best.seconds < 1e30;
      if (t < best.seconds * (same_shape ? 1.0 : 1.0 - kPreferLarger)) best = {c.slot, false, dp, t};
    }
  if (split_mode >= 0 && (m % 128 != 0 || n % 128 != 0)) {
    int bcfg, rcfg;
    strip_cfgs(m, n, bcfg, rcfg);
    const int64_t m1 = bcfg != kStripNone ? m - m % 128 : m, n1 = rcfg != kStripNone ? n - n % 128 : n;
    if ((bcfg != kStripNone || rcfg != kStripNone) && m1 >= 128 && n1 >= 128) {
      double t = model_seconds(m1, n1, k, 128, 128, 1, kTileCfgs[0].eff, sms);
      if (rcfg != kStripNone) {
        const StripInfo si = strip_info(rcfg);
        t += model_seconds(m, n - n1, k, si.bm, si.bn, si.sub, kStripEff, sms);
      }
      if (bcfg != kStripNone) {
        const int sbm = bcfg == kStrip64x128 ? 64 : strip_info(bcfg).bm;
        const int ssub = bcfg == kStrip64x128 ? 1 : strip_info(bcfg).sub;
        t += model_seconds(m - m1, n1, k, sbm, 128, ssub, bcfg == kStrip64x128 ? 0.9530 : kStripEff, sms);
      }
      if (t < best.seconds || split_mode == 1) best = {-1, true, false, t};
    }
  }
  return best;
}

// The choice is a few microseconds of host arithmetic; a per-thread cache of
// recent shapes keeps it off repeated calls (a synchronous call's kernel-only
// clock starts before the host enqueues).
TileChoice choose_tile(int64_t m, int64_t n, int64_t k, int sms, int split_mode) {
  struct Entry {
    int64_t m, n, k;
    int sms, split_mode;
    TileChoice tc;
  };
  thread_local Entry cache[8];
  thread_local int next = 0, used = 0;
  for (int i = 0; i < used; ++i) {
    const Entry& e = cache[i];
    if (e.m == m && e.n == n && e.k == k && e.sms == sms && e.split_mode == split_mode) return e.tc;
  }
  const TileChoice tc = choose_tile_uncached(m, n, k, sms, split_mode);
  cache[next] = {m, n, k, sms, split_mode, tc};
  next = (next + 1) % 8;
  if (used < 8) ++used;
  return tc;
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

// Staging. AUTO on operands TMA cannot address (odd leading dimension or a base not
// 16-byte aligned — the reference's odd-N cases) would run the cp.async
// loader, which lacks the TMA path's tile shapes and chooser. From 2e6 flops
// (N ~ 100) the operands are instead copied once, on the launching stream,
// into even-pitch workspace buffers (HBM copy: ~1 % of the GEMM time at
// N = 9999) and the TMA kernel runs on those: round 2 lowered the threshold
// from 2e10 after a same-box A/B (profiles/r02_odd_n_staging.txt, kernel-only
// TFLOP/s cp.async -> staged: N = 1001 19.5 -> 23.0, 1501 25.0 -> 28.8,
// 1999 25.8 -> 32.4 (cuBLAS 31.8); 129 30.5 -> 22.2 us; N = 65 equal).
// Tiny products keep the cp.async loader.
constexpr double kStageMinFlops = 2e6;
constexpr size_t kStageMaxBytes = size_t(16) << 30;

// Row re-pitch for staging: dst (16-byte aligned, even pitch) <- src (any
// 8-byte alignment/pitch). One block row-slab per blockIdx.y, coalesced 8-byte
// loads, 16-byte stores where the destination allows.
struct RepitchJob {
  const double* src;
  int64_t lds;
  double* dst;
  int64_t ldd, rows, cols;
};

// One launch re-pitches up to two operands (blockIdx.z picks the job). Each
// thread moves up to U pairs per step with all loads issued before the
// stores (bytes in flight bound this HBM copy).
template <int U>
__global__ void __launch_bounds__(256) repitch_kernel(RepitchJob j0, RepitchJob j1) {
  const RepitchJob& j = blockIdx.z == 0 ? j0 : j1;
  const int64_t pairs = (j.cols + 1) / 2;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t r = blockIdx.y; r < j.rows; r += gridDim.y) {
    const double* s = j.src + r * j.lds;
    double2* d = reinterpret_cast<double2*>(j.dst + r * j.ldd);
    for (int64_t p0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p0 < pairs; p0 += U * stride) {
      double x[U], y[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int64_t c = 2 * (p0 + u * stride);
        x[u] = c < j.cols ? __ldg(s + c) : 0.0;
        y[u] = c + 1 < j.cols ? __ldg(s + c + 1) : 0.0;  // ldd even, >= cols + (cols & 1): pad column 0
      }
#pragma unroll
      for (int u = 0; u < U; ++u)
        if (p0 + u * stride < pairs) d[p0 + u * stride] = make_double2(x[u], y[u]);
    }
  }
}

// Re-pitch job j0 and, if j1.rows > 0, j1 too, in one launch.
int repitch(const RepitchJob& j0, const RepitchJob& j1, cudaStream_t stream) {
  constexpr int U = 4;
  const int64_t rows = std::max(j0.rows, j1.rows), cols = std::max(j0.cols, j1.cols);
  const int64_t pairs = (cols + 1) / 2;
  const unsigned gx = (unsigned)std::min<int64_t>((pairs + 256 * U - 1) / (256 * U), 8);
  const unsigned gy = (unsigned)std::min<int64_t>(rows, 65535);
  repitch_kernel<U><<<dim3(gx, gy, j1.rows > 0 ? 2 : 1), 256, 0, stream>>>(j0, j1);
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
                 int strip, bool dp_only = false);

// Enqueue one GEMM on `stream` (current device = dev). Assumes validated args.
// Stages misaligned operands (large AUTO calls), then, for a TMA-fed DMMA
// product, runs the tile shape the cost model picks (choose_tile): one launch
// on one of the main-tile shapes, or — for wide problems with ragged m / n —
// a whole 128 x 128-tile launch plus the remainder strips as launches of
// their own.
int launch(int dev, const double* A, int64_t lda, const double* B, int64_t ldb, double* Cm, int64_t ldc, int64_t m,
           int64_t k, int64_t n, int accumulate, int tile_edge, int variant, cudaStream_t stream) {
  int s = g_plan ? TB_STATUS_OK : ensure_kernel_attrs(dev);
  if (s) return s;
  // Per device: a staged call's re-pitch and GEMM are enqueued together, so
  // two host threads on one stream cannot interleave repitch(A1), repitch(A2),
  // gemm1, gemm2 on the shared stream-keyed staging buffer.
  std::unique_lock<std::mutex> stage_lk(g_dev[dev].stage_mu, std::defer_lock);
  static const double stage_min = [] {  // TB_STAGE_MIN_FLOPS: A/B override of kStageMinFlops
    const char* e = std::getenv("TB_STAGE_MIN_FLOPS");
    return e ? std::atof(e) : kStageMinFlops;
  }();
  if (variant == TB_VARIANT_AUTO && !tma_ok(A, lda, B, ldb) && 2.0 * (double)m * (double)n * (double)k >= stage_min) {
    const bool sa = misaligned(A, lda), sb = misaligned(B, ldb);
    const int64_t lda2 = (k + 1) & ~int64_t(1), ldb2 = (n + 1) & ~int64_t(1);
    const size_t ea = sa ? (size_t)(m * lda2 + 32) : 0, eb = sb ? (size_t)(k * ldb2) : 0;
    if ((ea + eb) * sizeof(double) <= kStageMaxBytes && g_plan) {
      g_plan->json += std::string("{\"repitch\":\"") + (sa ? "A" : "") + (sb ? "B" : "") + "\"},";
      if (sa) {
        A = reinterpret_cast<const double*>(256);
        lda = lda2;
      }
      if (sb) {
        B = reinterpret_cast<const double*>(256);
        ldb = ldb2;
      }
    } else if ((ea + eb) * sizeof(double) <= kStageMaxBytes) {
      stage_lk.lock();
      double* buf = nullptr;
      if ((s = stage_workspace(dev, stream, ea + eb + 32, &buf))) return s;
      double* a2 = buf;
      double* b2 = buf + ((ea + 31) & ~size_t(31));  // 256-byte aligned
      const RepitchJob ja{A, lda, a2, lda2, m, k}, jb{B, ldb, b2, ldb2, k, n}, none{nullptr, 0, nullptr, 0, 0, 0};
      if ((s = repitch(sa ? ja : jb, sa && sb ? jb : none, stream))) return s;
      if (sa) {
        A = a2;
        lda = lda2;
      }
      if (sb) {
        B = b2;
        ldb = ldb2;
      }
    }
  }
  variant = resolve(A, lda, B, ldb, variant);
  // Test / A-B hooks, read per call (tests switch them in-process):
  // TB_TILE=<bm>x<bn> forces one main-tile shape with no edge split;
  // TB_SPLIT=0 never splits off edge strips, TB_SPLIT=1 always does when the
  // shape allows it (strip-kernel parity tests); unset: the cost model decides.
  const int forced_tile = [] {
    const char* e = std::getenv("TB_TILE");
    if (!e) return 0;
    for (int c = kStrip64x128; c < kNumStripCfgs; ++c) {
      const StripInfo si = strip_info(c);
      char name[32];
      std::snprintf(name, sizeof(name), "%dx%d%s", c == kStrip64x128 ? 64 : si.bm, c == kStrip64x128 ? 128 : si.bn,
                    c == kTile64x64d || c == kTile64x128 ? "d" : c == kTile96x96t ? "t" : "");
      if (std::strcmp(e, name) == 0) return c;
    }
    return std::strcmp(e, "128x128") == 0 ? -1 : 0;
  }();
  if (forced_tile && variant == TB_VARIANT_DMMA_TMA)
    return launch_tiles(dev, A, lda, B, ldb, Cm, ldc, m, k, n, accumulate, tile_edge, variant, stream, forced_tile);
  const char* split_e = std::getenv("TB_SPLIT");
  const int split_mode = !split_e ? 0 : std::strcmp(split_e, "0") == 0 ? -1 : std::strcmp(split_e, "1") == 0 ? 1 : 0;
  if (variant == TB_VARIANT_DMMA_TMA) {
    // Costed choice between every main-tile shape and the edge-strip plan (choose_tile).
    const TileChoice tc = choose_tile(m, n, k, dev_sms(dev), split_mode);
    if (!tc.split)
      return launch_tiles(dev, A, lda, B, ldb, Cm, ldc, m, k, n, accumulate, tile_edge, variant, stream, tc.slot,
                          tc.dp);
    int bcfg, rcfg;
    strip_cfgs(m, n, bcfg, rcfg);
    const int64_t m1 = bcfg != kStripNone ? m - m % 128 : m, n1 = rcfg != kStripNone ? n - n % 128 : n;
    // Main part on whole 128 x 128 tiles, then the right strip (all rows)
    // and the bottom strip (the main part's columns); disjoint parts of C.
    // The strips go on a side stream forked after the main launch, so their
    // CTAs take SMs as the main launch's CTAs retire (its ~0.2 ms end-time
    // spread) instead of waiting for the last one; the caller's stream then
    // waits for them (TB_STRIP_CONCURRENT=0: all on the caller's stream).
    DeviceState& st = g_dev[dev];
    const char* sce = std::getenv("TB_STRIP_CONCURRENT");
    const bool side_ok = !g_plan && !(sce && std::strcmp(sce, "0") == 0);
    std::unique_lock<std::mutex> side_lk(st.side_mu, std::defer_lock);
    DeviceState::SideStream* ss = nullptr;
    if (side_ok) {
      side_lk.lock();
      DeviceState::SideStream& e = st.side[stream];
      if (!e.s) {
        if (cudaStreamCreateWithFlags(&e.s, cudaStreamNonBlocking) != cudaSuccess ||
            cudaEventCreateWithFlags(&e.fork, cudaEventDisableTiming) != cudaSuccess ||
            cudaEventCreateWithFlags(&e.join, cudaEventDisableTiming) != cudaSuccess) {
          cudaGetLastError();
          if (e.s) cudaStreamDestroy(e.s);
          if (e.fork) cudaEventDestroy(e.fork);
          e = DeviceState::SideStream{};
        }
      }
      if (e.s) ss = &e;
    }
    if (ss) {
      TB_CUDA(cudaEventRecord(ss->fork, stream), "strip fork");
      TB_CUDA(cudaStreamWaitEvent(ss->s, ss->fork, 0), "strip fork");
    }
    if ((s = launch_tiles(dev, A, lda, B, ldb, Cm, ldc, m1, k, n1, accumulate, tile_edge, variant, stream, -1)))
      return s;
    const cudaStream_t strip_stream = ss ? ss->s : stream;
    if (rcfg != kStripNone &&
        (s = launch_tiles(dev, A, lda, B + n1, ldb, Cm + n1, ldc, m, k, n - n1, accumulate, tile_edge, variant,
                          strip_stream, rcfg)))
      return s;
    if (bcfg != kStripNone &&
        (s = launch_tiles(dev, A + m1 * lda, lda, B, ldb, Cm + m1 * ldc, ldc, m - m1, k, n1, accumulate, tile_edge,
                          variant, strip_stream, bcfg)))
      return s;
    if (ss) {
      TB_CUDA(cudaEventRecord(ss->join, ss->s), "strip join");
      TB_CUDA(cudaStreamWaitEvent(stream, ss->join, 0), "strip join");
    }
    return TB_STATUS_OK;
  }
  return launch_tiles(dev, A, lda, B, ldb, Cm, ldc, m, k, n, accumulate, tile_edge, variant, stream, kStripNone);
}

// One launch on resolved operands. strip: kStripNone = choose_bm's tile
// height, -1 = 128 x 128 forced, else an edge-strip shape.
int launch_tiles(int dev, const double* A, int64_t lda, const double* B, int64_t ldb, double* Cm, int64_t ldc,
                 int64_t m, int64_t k, int64_t n, int accumulate, int tile_edge, int variant, cudaStream_t stream,
                 int strip, bool dp_only) {
  int s = TB_STATUS_OK;
  if (variant == TB_VARIANT_PAPER) {
    const int K = tile_edge;
    dim3 block(K, K);
    dim3 grid((unsigned)((n + K - 1) / K), (unsigned)((m + K - 1) / K));
    if (g_plan) {
      char b[256];
      std::snprintf(b, sizeof(b), "{\"kernel\":\"paper\",\"m\":%lld,\"n\":%lld,\"k\":%lld,\"block\":[%d,%d],"
                    "\"grid\":[%u,%u]},", (long long)m, (long long)n, (long long)k, K, K, grid.x, grid.y);
      g_plan->json += b;
      return TB_STATUS_OK;
    }
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
    const StripInfo si = strip > 0 ? strip_info(strip) : StripInfo{0, 0, 1, nullptr, 0};
    const bool narrow = si.fn != nullptr;  // an edge-strip shape (TMA only)
    const int bm = narrow ? si.bm : strip == kStrip64x128 ? 64 : strip < 0 ? 128 : choose_bm(m, n, dev_sms(dev), dfma);
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
    const int64_t kstage = narrow ? (int64_t)Cfg::BK * si.sub : bm == 64 ? (int64_t)Cfg::BK
                                                                       : (int64_t)Cfg::BK * kCfgs[cfg].sub;
    p.num_k = (int)((k + kstage - 1) / kstage);
    const Schedule sc = plan_schedule(tiles, p.num_k, dev_sms(dev), dp_only);
    p.num_k = sc.num_k;  // split-K pads the k-slab count (extra slabs read as zeros)
    p.dp_tiles = sc.dp;
    p.sk_tiles = sc.sk;
    p.sk_ipc = sc.ipc;
    p.max_seg = sc.max_seg;
    p.partials = nullptr;
    p.counters = nullptr;
    if (g_plan) {
      const bool tma = variant == TB_VARIANT_DMMA_TMA || (dfma && tma_ok(A, lda, B, ldb));
      const char* shape = sc.sk == 0 ? "data-parallel" : sc.dp == 0 && sc.grid != dev_sms(dev) ? "split-k"
                                                                                                 : "stream-k";
      char b[512];
      std::snprintf(b, sizeof(b),
                    "{\"kernel\":\"%s\",\"loader\":\"%s\",\"tile\":[%d,%d,%d],\"m\":%lld,\"n\":%lld,"
                    "\"k\":%lld,\"grid\":%d,\"schedule\":\"%s\",\"dp_tiles\":%d,\"sk_tiles\":%d,"
                    "\"sk_iters_per_cta\":%d,\"max_segments\":%d,\"k_stages\":%d,\"strip\":%s},",
                    dfma ? "dfma" : "dmma", tma ? "tma" : "cp.async", bm, bn, (int)kstage, (long long)m,
                    (long long)n, (long long)k, sc.grid, shape, sc.dp, sc.sk, sc.ipc, sc.max_seg, sc.num_k,
                    narrow ? "true" : "false");
      g_plan->json += b;
      return TB_STATUS_OK;
    }
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
        units += (double)(r[4] & 0xffffffffull);
        endmax = std::max(endmax, (double)(r[3] - t0));
        endmin = std::min(endmin, (double)(r[3] - t0));
      }
      const double g = sc.grid;
      if (std::strcmp(std::getenv("TB_TIMELINE"), "2") == 0)  // per-CTA lines: SM, units, end, main loop
        for (int c = 0; c < sc.grid; ++c) {
          const unsigned long long* r = &h[(size_t)c * 8];
          std::fprintf(stderr, "TBCTA cta=%d smid=%llu units=%llu end_us=%.2f mainloop_us=%.2f fixup_us=%.2f\n", c,
                       r[4] >> 32, r[4] & 0xffffffffull, (r[3] - t0) / 1e3, r[7] / 1e3, r[5] / 1e3);
        }
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
#ifdef TB_TIMELINE
struct PipeTimeline {
  unsigned long long* buf = nullptr;
  int grid = 0;
};
PipeTimeline g_pipe_tl;  // tooling build: the last PIPE launch's stamps

// Summarise and free the last PIPE launch's stamps (after it completed).
void pipe_timeline_report() {
  if (!g_pipe_tl.buf) return;
  const int g = g_pipe_tl.grid;
  std::vector<unsigned long long> h((size_t)g * 12);
  if (cudaMemcpy(h.data(), g_pipe_tl.buf, h.size() * sizeof(unsigned long long), cudaMemcpyDeviceToHost) ==
      cudaSuccess) {
    unsigned long long t0 = ~0ull, tend = 0;
    double wait = 0, wmax = 0, w0 = 0, nw = 0, ml = 0, epi = 0, units = 0, endmin = 1e30, lastw = 0;
    for (int c = 0; c < g; ++c) t0 = std::min(t0, h[(size_t)c * 8]);
    for (int c = 0; c < g; ++c) {
      const unsigned long long* r = &h[(size_t)c * 8];
      const unsigned long long* w = &h[(size_t)g * 8 + (size_t)c * 4];
      tend = std::max(tend, r[3]);
      endmin = std::min(endmin, (double)(r[3] - t0));
      wait += (double)w[0];
      wmax = std::max(wmax, (double)w[0]);
      w0 += (double)w[2];
      nw += (double)w[1];
      lastw = std::max(lastw, w[3] ? (double)(w[3] - t0) : 0.0);
      ml += (double)r[7];
      epi += (double)r[6];
      units += (double)(r[4] & 0xffffffffull);
    }
    std::fprintf(stderr,
                 "TBPIPE grid=%d span_us=%.1f end_min_us=%.1f flag_wait_mean_us=%.1f flag_wait_max_us=%.1f "
                 "panel0_wait_mean_us=%.1f waits_per_cta=%.2f last_wait_end_us=%.1f mainloop_mean_us=%.1f "
                 "epilogue_mean_us=%.1f units=%.2f\n",
                 g, (double)(tend - t0) * 1e-3, endmin * 1e-3, wait / g * 1e-3, wmax * 1e-3, w0 / g * 1e-3, nw / g,
                 lastw * 1e-3, ml / g * 1e-3, epi / g * 1e-3, units / g);
  }
  cudaFree(g_pipe_tl.buf);
  g_pipe_tl.buf = nullptr;
}
#endif

// Flag-wait timeout of the fused phase-1 launch (ms; after it the launch
// aborts, dgemm_dmma.cuh kPipeAbortWord). TB_PIPE_TIMEOUT_MS overrides
// (read per call: the abort test shortens it in-process).
int pipe_timeout_ms() {
  const char* e = std::getenv("TB_PIPE_TIMEOUT_MS");
  const long v = e ? std::atol(e) : 0;
  return v > 0 && v < 3600000 ? (int)v : 10000;
}

int launch_pipe(int dev, const double* A, int64_t lda, const double* B, int64_t ldb, double* Cm, int64_t ldc,
                int64_t m, int64_t k, int64_t n, const int* panel_it_d, int* flags_d, int Q, int timeout_ms,
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
  p.sk_ipc = timeout_ms;                                 // PIPE: flag-wait timeout (ms)
  p.max_seg = 1;
  p.counters = const_cast<int*>(panel_it_d);             // PIPE: panel k-stage bounds
  p.partials = reinterpret_cast<double*>(flags_d);       // PIPE: panel flags + abort word
  if ((s = get_encoder())) return s;
  CUtensorMap mA, mB;
  if ((s = encode_map(&mA, A, m, k, lda, Cfg::BM))) return s;
  if ((s = encode_map(&mB, B, k, n, ldb, Cfg::BK))) return s;
  void* args[] = {&mA, &mB, &p};
  const int grid = (int)std::min<int64_t>(tiles, dev_sms(dev));
#ifdef TB_TIMELINE
  p.timeline = nullptr;
  if (std::getenv("TB_TIMELINE")) {  // read back by the host-buffer entry after the call
    const size_t words = (size_t)grid * 12;
    TB_CUDA(cudaMalloc(&g_pipe_tl.buf, words * sizeof(unsigned long long)), "timeline alloc");
    TB_CUDA(cudaMemsetAsync(g_pipe_tl.buf, 0, words * sizeof(unsigned long long), stream), "timeline");
    g_pipe_tl.grid = grid;
    p.timeline = g_pipe_tl.buf;
  }
#endif
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
    if ((s = ensure_cublas(dev))) return s;
    // The handle is shared per device: its stream binding and the DGEMM
    // enqueue happen under one lock, so concurrent callers with different
    // streams each get their GEMM on their own stream.
    std::lock_guard<std::mutex> lk(st.cublas_mu);
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
