// dgemm_dmma.cuh — sm_100a FP64 GEMM on the DMMA pipe (mma.sync m8n8k4 f64).
//
// The paper's K = 32 tiled kernel (reference kernel.ts:50-78)
// "revisited for Blackwell": instead of one output per thread fed by two
// shared-memory loads per FMA, a 128 x 128 CTA tile is computed by 8 consumer
// warps (64 x 32 warp tiles, 32 DMMA accumulators each) while a producer
// warpgroup streams 128 x 16 / 16 x 128 k-slabs of A and B into a STAGES-deep
// shared-memory ring (TMA with SWIZZLE_128B, or 8-byte cp.async with zero fill
// when the TMA 16-byte alignment rule does not hold). Full/empty mbarriers hand
// stages between producer and consumers; there is no __syncthreads in the main
// loop.
//
// Persistent schedule. One CTA per SM walks a static work list: first the
// data-parallel tiles (a multiple of gridDim.x, round-robin in grouped raster
// order), then a stream-K region — the last (T mod P) + P tiles' k-iterations
// split evenly across all CTAs, so the final partial wave does not leave SMs
// idle. The producer runs ahead across work units, so a tile's epilogue
// overlaps the next tile's loads. A tile split into segments is reduced
// deterministically: every segment writes its partial to a workspace slot,
// the CTA that completes the tile's segment count last sums the slots in
// segment order (fixed, independent of timing) and writes C, then resets the
// tile's counter for the next launch.
//
// Bank-conflict-free fragment loads. With the swizzled layout, the natural
// DMMA k order (lane q feeds k = 4s + q) gives 2-way conflicts. The k index
// inside a 16-deep slab is therefore permuted (legal: it only reorders the
// sum): lane q feeds k-pair PA(q) = {0,2,5,7}[q] to DMMA steps 0 and 1 and
// PB(q) = PA(q) ^ 1 = {1,3,4,6}[q] to steps 2 and 3. A fragments then come in
// as one conflict-free 128-bit load per two steps, B fragments as
// conflict-free 64-bit loads (derivation in DESIGN.md §4).
#pragma once

// Barrier-discipline mutants (tests/test_gpu_mutations.py, in the style of
// the reference's barriers.test.ts:37-82): test-only builds with
// -DTB_MUTATE=<n> break one ordering rule of the consumer's stage protocol
// so the suite can show it catches the break. Never set in the product
// build (0: the production kernel; SASS identical with the hooks compiled out).
//   1  fragment loads of a stage's first half-step issued BEFORE its
//      full-barrier wait (the "missing load barrier")
//   2  the stage released to the producer (empty arrive) right after its
//      full-barrier wait, before its fragments are read (the "missing reuse
//      barrier")
//   3  no fence.proxy.async before the empty arrive (the round-1 race)
#ifndef TB_MUTATE
#define TB_MUTATE 0
#endif

// Software-pipelined fragment loads on every DMMA tile shape (1) or only on
// 128 x 128 tiles with the plain loop elsewhere (0; A/B builds).
#ifndef TB_XPF_ALL
#define TB_XPF_ALL 1
#endif

// L2 prefetch of the old C tile ahead of an accumulating epilogue (1) or not (0; A/B builds).
#ifndef TB_C_PREFETCH
#define TB_C_PREFETCH 1
#endif

#ifndef TB_EARLY_RELEASE
#define TB_EARLY_RELEASE -1
#endif

#ifndef TB_GROUP_M
#define TB_GROUP_M 16  // tile-raster band height (A/B builds: tools/build_variant.py NAME -DTB_GROUP_M=16)
#endif
#include <cstdint>
#include <type_traits>
#include <cuda.h>
#include "ptx.cuh"

namespace tb {

enum class Loader : int { TMA = 0, CPASYNC = 1 };
// Consumer arithmetic: DMMA (mma.sync m8n8k4 f64, warp-cooperative 8x8x4) or
// DFMA (scalar fused multiply-add, 8x8 register tile per thread).
enum class Math : int { DMMA = 0, DFMA = 1 };

// BM (tile rows) is a template parameter: 128 is the production tile; 64
// halves the row padding and doubles the tile count for small problems
// (warp tile 32 x 32). Everything else is shared.
template <int BM_, int BN_ = 128, int WARPS_M_ = 2>
struct DmmaCfgT {
  static constexpr int BM = BM_, BN = BN_, BK = 16;
  static constexpr int WARPS_M = WARPS_M_, WARPS_N = 8 / WARPS_M_;
  static constexpr int WM = BM / WARPS_M;  // 64
  static constexpr int WN = BN / WARPS_N;  // 32
  static constexpr int MI = WM / 8;        // 8 DMMA rows per warp
  static constexpr int NI = WN / 8;        // 4 DMMA cols per warp
  static constexpr int CONSUMER_WARPS = WARPS_M * WARPS_N;
  static constexpr int CONSUMER_THREADS = CONSUMER_WARPS * 32;
  // Warpgroup specialisation: warpgroup 0 = producer (one TMA-issuing lane, or
  // all 4 warps issuing cp.async), warpgroups 1-2 = the 8 consumer warps.
  // setmaxnreg moves registers from the producer to the consumers
  // (4*32*PRODUCER_REGS + 8*32*CONSUMER_REGS <= 64K).
  static constexpr int THREADS = (CONSUMER_WARPS + 4) * 32;
  static constexpr int PRODUCER_REGS = 40;
  static constexpr int CONSUMER_REGS = 232;
  static constexpr int A_STAGE = BM * BK * 8;  // 16 KB: [128 rows][16 k] swizzled
  static constexpr int B_STAGE = BK * BN * 8;  // 16 KB: 8 boxes of [16 k][16 n] swizzled
  static constexpr int STAGE = A_STAGE + B_STAGE;
  static constexpr int B_BOX = BK * 16 * 8;  // 2 KB
  static constexpr int GROUP_M = TB_GROUP_M; // tile raster: GROUP_M tile-rows per band
  static constexpr int TILE_ELEMS = BM * BN;
};
using DmmaCfg = DmmaCfgT<128>;

// A pipeline stage holds SUB consecutive 16-deep k sub-slabs (SUB * STAGE bytes).
template <int SUB, int STAGES, int BM = 128, int BN = 128>
constexpr int dmma_smem_bytes() {
  return STAGES * SUB * DmmaCfgT<BM, BN>::STAGE + 2 * STAGES * 8 + 16 + 1024;  // + barriers + flag + alignment slack
}

struct GemmParams {
  const double* A;
  const double* B;
  double* C;
  int64_t lda, ldb, ldc;
  int m, n, k;
  int tiles_m, tiles_n;
  int num_k;       // pipeline stages (SUB x 16-deep k sub-slabs) per tile
  int accumulate;  // C += A·B instead of C = A·B
  int vec_store;   // C rows 16-byte aligned: store double2
  // persistent schedule
  int dp_tiles;    // data-parallel tiles, processed round-robin (multiple of gridDim.x)
  int sk_tiles;    // stream-K tiles after them
  int sk_ipc;      // stream-K k-iterations per CTA
  int max_seg;     // workspace slots per stream-K tile
  double* partials;  // [sk_tiles][max_seg][TILE_ELEMS] in fragment order
  int* counters;     // [sk_tiles], zero between launches (self-resetting)
#ifdef TB_TIMELINE
  unsigned long long* timeline;  // tooling build only: [grid][8] per-CTA %globaltimer stamps
#endif
};
// Pipelined host-buffer mode (PIPE instantiation only) has no stream-K
// region, so it reuses the stream-K fields (keeping GemmParams' layout, which
// ptxas's allocation for the production kernel turned out to depend on):
//   sk_tiles  -> number of K-panels Q
//   counters  -> panel_it[Q + 1]: panel q covers k-stages [panel_it[q], panel_it[q+1])
//   partials  -> panel_flags[kPipeFlagWords] (int): panel q is usable once
//                flags[q] != 0 (written by the copy stream after the panel's
//                copies); flags[kPipeAbortWord] is the launch's abort word
//   sk_ipc    -> flag-wait timeout in milliseconds
// Each CTA owns tiles blockIdx.x, +gridDim.x, ... and walks them
// panel-major, accumulating into C for panels after the first.
//
// Abort instead of trap: a producer that waits longer than the timeout for a
// panel flag (a host pipeline that stopped enqueueing, e.g. blocked behind
// another thread's device-synchronising call) sets the abort word and, like
// every producer that then sees the word, stops loading: it completes each
// remaining stage's full barrier with a plain arrive (no bytes), so the
// consumers run out their units on stale shared memory and the launch ends
// normally. The host reads the word after the call and returns
// TB_STATUS_RUNTIME; the CUDA context stays usable (a __trap would poison it
// for the whole process). The host can also set the word to cut a launch short.
constexpr int kPipeMaxPanels = 120;
constexpr int kPipeAbortWord = 127;
constexpr int kPipeFlagWords = 128;
__device__ __forceinline__ int pipe_panels(const GemmParams& p) { return p.sk_tiles; }
__device__ __forceinline__ const int* pipe_panel_it(const GemmParams& p) { return p.counters; }
__device__ __forceinline__ int* pipe_flags(const GemmParams& p) { return reinterpret_cast<int*>(p.partials); }

#ifdef TB_TIMELINE
__device__ __forceinline__ unsigned long long tl_now() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
#define TB_TL(stmt) stmt
#else
#define TB_TL(stmt)
#endif

// Grouped raster over the (tile_m, tile_n) grid so concurrently resident CTAs
// share A row-panels and B column-panels in L2.
__device__ __forceinline__ void tile_coords(int tile, int tiles_m, int tiles_n, int& tm, int& tn) {
  const int group = DmmaCfg::GROUP_M * tiles_n;
  const int first_m = (tile / group) * DmmaCfg::GROUP_M;
  const int gm = min(tiles_m - first_m, DmmaCfg::GROUP_M);
  const int r = tile % group;
  tm = first_m + r % gm;
  tn = r / gm;
}

// The CTA's static work list: (tile, [kb, ke)) units. Producer and consumers
// each walk their own copy, so they agree without communicating.
struct WorkIter {
  int t;
  int64_t it, end;  // stream-K iteration range (64-bit: sk_tiles * num_k may exceed 2^31)
  __device__ __forceinline__ explicit WorkIter(const GemmParams& p) {
    t = blockIdx.x;
    it = (int64_t)blockIdx.x * p.sk_ipc;
    end = min(it + p.sk_ipc, (int64_t)p.sk_tiles * p.num_k);
  }
  __device__ __forceinline__ bool next(const GemmParams& p, int& tile, int& kb, int& ke) {
    if (t < p.dp_tiles) {
      tile = t;
      kb = 0;
      ke = p.num_k;
      t += gridDim.x;
      return true;
    }
    if (it >= end) return false;
    const int st = (int)(it / p.num_k);
    kb = (int)(it - (int64_t)st * p.num_k);
    ke = (int)min((int64_t)p.num_k, kb + (end - it));
    tile = p.dp_tiles + st;
    it += ke - kb;
    return true;
  }
};

// PIPE mode work list: (tile, panel) units, panel-major over this CTA's tiles.
struct PipeIter {
  int t, q;
  __device__ __forceinline__ explicit PipeIter(const GemmParams&) : t(blockIdx.x), q(0) {}
  __device__ __forceinline__ bool next(const GemmParams& p, int& tile, int& kb, int& ke) {
    const int tiles = p.tiles_m * p.tiles_n;
    if (t >= tiles) {
      t = blockIdx.x;
      ++q;
    }
    if (q >= pipe_panels(p) || t >= tiles) return false;
    tile = t;
    kb = pipe_panel_it(p)[q];
    ke = pipe_panel_it(p)[q + 1];
    t += gridDim.x;
    return true;
  }
};

__device__ __forceinline__ void consumer_bar() { asm volatile("bar.sync 1, %0;\n" ::"n"(DmmaCfg::CONSUMER_THREADS)); }

template <int SUB, int STAGES, Loader LD, Math MT = Math::DMMA, int BM = 128, bool PIPE = false, int BN = 128,
          int WARPS_M = 2>
__global__ void __launch_bounds__(DmmaCfg::THREADS, 1)
    dgemm_dmma_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                      const GemmParams p) {
  using C = DmmaCfgT<BM, BN, WARPS_M>;
  static_assert(C::WARPS_M * C::WARPS_N == 8 && C::MI >= 2 && C::WN % 16 == 0, "8 consumer warps, >= 16 x 16 each");
  static_assert(MT == Math::DMMA || (BN == 128 && WARPS_M == 2), "the DFMA comparison path is laid out for 128 x 128");
  using Iter = typename std::conditional<PIPE, PipeIter, WorkIter>::type;
  static_assert(!PIPE || (LD == Loader::TMA && MT == Math::DMMA), "PIPE mode: TMA + DMMA only");
  static_assert(MT == Math::DMMA || BM == 128, "the DFMA comparison path is laid out for 128-row tiles");
  extern __shared__ uint8_t smem_raw[];
  // SWIZZLE_128B's XOR pattern is a function of absolute smem address bits
  // [4:6] ^ [7:9]: stage buffers must start on 1024-byte boundaries.
  // (Offset the __shared__ array itself so the compiler keeps the shared
  // address space and emits LDS rather than generic loads.)
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  constexpr int STAGE_BYTES = SUB * C::STAGE;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * STAGE_BYTES);
  uint64_t* empty = full + STAGES;
  int* flag = reinterpret_cast<int*>(empty + STAGES);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  TB_TL(unsigned long long* tl = p.timeline ? p.timeline + 8 * blockIdx.x : nullptr;)
  TB_TL(if (tl && threadIdx.x == 0) {
    unsigned smid;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
    tl[0] = tl_now();
    tl[4] = (unsigned long long)smid << 32;  // [4]: smid << 32 | units
  })

  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(smem_u32(&full[s]), LD == Loader::TMA ? 1 : 128);
      mbar_init(smem_u32(&empty[s]), C::CONSUMER_WARPS);
    }
    fence_barrier_init();
  }
  __syncthreads();

  if (warp < 4) {
    // ------------------------------------------------------------ producer
    setmaxnreg_dec<C::PRODUCER_REGS>();
    if (LD == Loader::TMA && threadIdx.x != 0) return;
    if (LD == Loader::TMA) {
      tma_prefetch_desc(&tmA);
      tma_prefetch_desc(&tmB);
    }
    int s = 0;
    uint32_t ph = 0;
    // cp.async loader: stage g's copies are committed as one group and its
    // full barrier is arrived on (release) once cp.async.wait_group shows the
    // group complete, CP_LAG stages later, so CP_LAG + 1 stages stay in
    // flight. CP_LAG <= STAGES - 1 keeps every arrive ahead of the empty-slot
    // wait that could depend on it (no deadlock).
    constexpr int CP_LAG = STAGES - 1 < 4 ? STAGES - 1 : 4;
    int g = 0;
    Iter w(p);
    int tile, kb, ke;
    int ready_upto = 0;  // PIPE: panel flags observed set so far
    bool aborted = false;  // PIPE: stop loading, complete the remaining stages empty
    while (w.next(p, tile, kb, ke)) {
      if constexpr (PIPE) {
        // Wait for the panel holding k-stages [kb, ke) (panels land in order).
        while (!aborted && ready_upto < pipe_panels(p) && pipe_panel_it(p)[ready_upto] <= kb) {
          if (ld_acquire_gpu(&pipe_flags(p)[ready_upto]) == 0) {
            // Bounded: a panel that does not land within the timeout aborts
            // the launch (see kPipeAbortWord) instead of hanging the device.
            const unsigned long long t_start = globaltimer_ns();
            const unsigned long long t_max = 1000000ull * (unsigned)p.sk_ipc;
            int* abort_word = pipe_flags(p) + kPipeAbortWord;
            while (ld_acquire_gpu(&pipe_flags(p)[ready_upto]) == 0) {
              if (ld_acquire_gpu(abort_word) != 0) {
                aborted = true;
                break;
              }
              if (globaltimer_ns() - t_start > t_max) {
                st_release_gpu(abort_word, 1 + ready_upto);  // 1 + the panel that never landed
                aborted = true;
                break;
              }
            }
            // tooling build: [grid][8] stamps, then [grid][4] producer flag waits
            // (total ns, count, panel-0 ns, last wait end)
            TB_TL(if (p.timeline) {
              unsigned long long* w = p.timeline + 8 * gridDim.x + 4 * blockIdx.x;
              const unsigned long long t_end = globaltimer_ns();
              w[0] += t_end - t_start;
              w[1] += 1;
              if (ready_upto == 0) w[2] = t_end - t_start;
              w[3] = t_end;
            })
          }
          ++ready_upto;
        }
      }
      int tm, tn;
      tile_coords(tile, p.tiles_m, p.tiles_n, tm, tn);
      const int m0 = tm * C::BM, n0 = tn * C::BN;
      for (int kt = kb; kt < ke; ++kt) {
        mbar_wait(smem_u32(&empty[s]), ph ^ 1);  // fresh barrier: parity 1 reads as complete
        const uint32_t stage = smem_u32(smem + s * STAGE_BYTES);
        if (PIPE && aborted) {
          mbar_arrive(smem_u32(&full[s]));  // aborted launch: release the stage with no bytes
        } else if constexpr (LD == Loader::TMA) {
          const uint32_t fb = smem_u32(&full[s]);
          mbar_arrive_expect_tx(fb, STAGE_BYTES);  // OOB-filled boxes still count full bytes
#pragma unroll
          for (int u = 0; u < SUB; ++u) {
            const uint32_t sa = stage + u * C::STAGE, sb = sa + C::A_STAGE;
            const int k0 = (kt * SUB + u) * C::BK;
            tma_load_2d(sa, &tmA, fb, k0, m0);
#pragma unroll
            for (int j = 0; j < C::BN / 16; ++j) tma_load_2d(sb + j * C::B_BOX, &tmB, fb, n0 + 16 * j, k0);
          }
        } else {
          // 8-byte cp.async into the same swizzled layout; src-size 0
          // zero-fills out-of-range cells (the paper's "load zero" edge rule,
          // PAPER.md:124).
          const int pt = threadIdx.x;  // 0..127
#pragma unroll
          for (int u = 0; u < SUB; ++u) {
            const uint32_t sa = stage + u * C::STAGE, sb = sa + C::A_STAGE;
            const int k0 = (kt * SUB + u) * C::BK;
#pragma unroll 4
            for (int i = 0; i < (C::BM * C::BK) / 128; ++i) {
              const int e = i * 128 + pt, r = e >> 4, kk = e & 15;
              const int gm = m0 + r, gk = k0 + kk;
              const bool ok = gm < p.m && gk < p.k;
              const double* src = ok ? p.A + (int64_t)gm * p.lda + gk : p.A;
              cp_async_8(sa + r * 128 + (((kk >> 1) ^ (r & 7)) << 4) + (kk & 1) * 8, src, ok);
            }
#pragma unroll 4
            for (int i = 0; i < (C::BK * C::BN) / 128; ++i) {
              const int e = i * 128 + pt, kr = e / C::BN, nn = e % C::BN;
              const int gk = k0 + kr, gn = n0 + nn;
              const bool ok = gk < p.k && gn < p.n;
              const double* src = ok ? p.B + (int64_t)gk * p.ldb + gn : p.B;
              cp_async_8(sb + (nn >> 4) * C::B_BOX + kr * 128 + ((((nn & 15) >> 1) ^ (kr & 7)) << 4) + (nn & 1) * 8,
                         src, ok);
            }
          }
          cp_async_commit();
          if (g >= CP_LAG) {
            cp_async_wait<CP_LAG>();
            mbar_arrive(smem_u32(&full[(g - CP_LAG) % STAGES]));
          }
          ++g;
        }
        if (++s == STAGES) {
          s = 0;
          ph ^= 1;
        }
      }
      // The unit's loads are all issued (the consumers are ~STAGES stages
      // behind): if its epilogue will add the old C tile (C += A·B, or a
      // PIPE panel after the first), pull that tile into L2 now so the
      // epilogue's loads hit L2 instead of DRAM.
      if constexpr (LD == Loader::TMA && TB_C_PREFETCH) {
        if ((PIPE ? (p.accumulate || kb != 0) : p.accumulate) && p.vec_store && !(PIPE && aborted)) {
          const int r_end = min(m0 + C::BM, p.m);
          const uint32_t bytes = (uint32_t)((min(n0 + C::BN, p.n) - n0) * 8) & ~15u;  // never past the row
          if (bytes)
            for (int r = m0; r < r_end; ++r) bulk_prefetch_l2(p.C + (int64_t)r * p.ldc + n0, bytes);
        }
      }
    }
    if constexpr (LD == Loader::CPASYNC) {
      cp_async_wait<0>();
      for (int x = g > CP_LAG ? g - CP_LAG : 0; x < g; ++x) mbar_arrive(smem_u32(&full[x % STAGES]));
    }
    return;
  }

  // -------------------------------------------------------------- consumers
  setmaxnreg_inc<C::CONSUMER_REGS>();
  const int ct = threadIdx.x - 128;  // consumer thread 0..255
  const int cw = warp - 4;
  const int wm = cw / C::WARPS_N, wn = cw % C::WARPS_N;
  const int q = lane & 3, g = lane >> 2;
  // Output coordinates of acc[i][j][e] inside the CTA tile:
  //   row = row_base + i * row_step, col = col_base + j * col_step + e.
  // DMMA: 2 x 4 warps of 64 x 32 (C fragment rows g, cols 2q).
  // DFMA: 4 x 2 warps of 32 x 64; lane (lr, lc) = (lane >> 3, lane & 7) owns
  //       rows lr + 4i and column pairs 2lc + 16j, so a quarter-warp shares
  //       one A row (broadcast) and covers 8 distinct 16-byte B chunks.
  const int lr = lane >> 3, lc = lane & 7;
  const int row_base = MT == Math::DMMA ? wm * C::WM + g : (cw >> 1) * 32 + lr;
  const int row_step = MT == Math::DMMA ? 8 : 4;
  const int col_base = MT == Math::DMMA ? wn * C::WN + 2 * q : (cw & 1) * 64 + 2 * lc;
  const int col_step = MT == Math::DMMA ? 8 : 16;
  // DFMA A offsets: row ra = row_base + 4i, 16-byte chunk kp -> kp ^ (ra & 7),
  // so byte = dfma_a[i] ^ (kp << 4) with dfma_a[i] = ra*128 + ((ra & 7) << 4).
  uint32_t dfma_a[C::MI];
#pragma unroll
  for (int i = 0; i < C::MI; ++i) {
    const int ra = row_base + 4 * i;
    dfma_a[i] = ra * 128 + ((ra & 7) << 4);
  }
  const int pa = 2 * q + (q >> 1);  // {0,2,5,7}
  const int pb = pa ^ 1;            // {1,3,4,6}

  // A: row r = wm*64 + mi*8 + g (so r & 7 == g), 16-byte chunk c -> c ^ g.
  const uint32_t a_off0 = (wm * C::WM + g) * 128 + ((pa ^ g) << 4);
  const uint32_t a_off1 = (wm * C::WM + g) * 128 + ((pb ^ g) << 4);
  // B: column nn = (ni&1)*8 + g inside box wn*2 + (ni>>1); k row kv:
  // byte = box*2048 + kv*128 + (((nn>>1) ^ (kv&7)) << 4) + (nn&1)*8, and
  // (ni&1) flips chunk bit 2, i.e. byte bit 6.
  uint32_t b_off[4];
  {
    const int kv[4] = {2 * pa, 2 * pa + 1, 2 * pb, 2 * pb + 1};
#pragma unroll
    for (int e = 0; e < 4; ++e)
      b_off[e] = wn * (C::WN / 16) * C::B_BOX + kv[e] * 128 + ((((g >> 1) ^ (kv[e] & 7))) << 4) + (g & 1) * 8;
  }

  int s = 0;
  uint32_t ph = 0;
  Iter w(p);
  int tile, kb, ke;
  while (w.next(p, tile, kb, ke)) {
    double acc[C::MI][C::NI][2];
#pragma unroll
    for (int i = 0; i < C::MI; ++i)
#pragma unroll
      for (int j = 0; j < C::NI; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

    TB_TL(unsigned long long tl_u = 0;)
    if constexpr (MT == Math::DMMA && (TB_XPF_ALL || (SUB == 1 && BM == 128 && BN == 128))) {
      // Software-pipelined fragment loads: the fragments of half-step h + 1
      // (a half-step = 8 of a 16-deep sub-slab's k) are loaded before the
      // DMMAs of half-step h issue, across sub-slabs and across stages (the
      // next stage's full barrier is waited on, and its first half-step
      // loaded, before this stage's last DMMAs), so the tensor pipe does not
      // drain at stage boundaries and the schedule does not depend on how
      // ptxas interleaves a plain loop (+0.3-0.45 % at N = 5000-10000 on
      // 128 x 128 tiles, profiles/r01_xpf_ab.txt; a few address registers
      // spill there, per stage, outside the DMMA stream).
      constexpr int HS = 2 * SUB;
      // Early stage release on every shape but 128 x 128 (same-box A/B,
      // profiles/r02_early_release_ab.jsonl: 64 x 96 / 128 x 96 / 96 x 96
      // +0.3-1.3 %, 128 x 64 neutral, 128 x 128 -0.6 %). TB_EARLY_RELEASE=0|1
      // forces it off / on everywhere (A/B builds).
      constexpr bool kEarlyRelease = TB_EARLY_RELEASE < 0 ? !(BM == 128 && BN == 128) : TB_EARLY_RELEASE != 0;
      double2 fa[2][C::MI];
      double fb[2][2][C::NI];
      auto ld = [&](int stage, int hs, int buf) {
        const int half = hs & 1;
        const uint8_t* sa = smem + stage * STAGE_BYTES + (hs >> 1) * C::STAGE;
        const uint8_t* sb = sa + C::A_STAGE;
#pragma unroll
        for (int i = 0; i < C::MI; ++i)
          fa[buf][i] = *reinterpret_cast<const double2*>(sa + (half ? a_off1 : a_off0) + i * 8 * 128);
#pragma unroll
        for (int j = 0; j < C::NI; ++j) {
          const uint32_t box = (j >> 1) * C::B_BOX, flip = (j & 1) ? 64u : 0u;
          fb[buf][0][j] = *reinterpret_cast<const double*>(sb + box + (b_off[2 * half] ^ flip));
          fb[buf][1][j] = *reinterpret_cast<const double*>(sb + box + (b_off[2 * half + 1] ^ flip));
        }
      };
      auto mma = [&](int buf) {
#pragma unroll
        for (int i = 0; i < C::MI; ++i)
#pragma unroll
          for (int j = 0; j < C::NI; ++j) dmma_8x8x4(acc[i][j][0], acc[i][j][1], fa[buf][i].x, fb[buf][0][j]);
#pragma unroll
        for (int i = 0; i < C::MI; ++i)
#pragma unroll
          for (int j = 0; j < C::NI; ++j) dmma_8x8x4(acc[i][j][0], acc[i][j][1], fa[buf][i].y, fb[buf][1][j]);
      };
#if TB_MUTATE == 1
      ld(s, 0, 0);
      mbar_wait(smem_u32(&full[s]), ph);
#else
      mbar_wait(smem_u32(&full[s]), ph);
#if TB_MUTATE == 2
      __syncwarp();
      if (lane == 0) mbar_arrive(smem_u32(&empty[s]));
#endif
      ld(s, 0, 0);
#endif
      TB_TL(if (tl && ct == 0) { tl_u = tl_now(); if (tl[1] == 0) tl[1] = tl_u; })
      for (int kt = kb; kt < ke; ++kt) {
#pragma unroll
        for (int hs = 0; hs + 1 < HS; ++hs) {
          ld(s, hs + 1, (hs + 1) & 1);
          mma(hs & 1);
        }
        const int s1 = s + 1 == STAGES ? 0 : s + 1;
        const uint32_t ph1 = s + 1 == STAGES ? ph ^ 1 : ph;
        if constexpr (kEarlyRelease) {
          // Every fragment of stage s is now loaded (the last half-step's
          // went out before the mma above): release the stage before waiting
          // on the next one, so the proxy fence waits only on those loads,
          // not on the next stage's freshly issued ones, and the producer
          // refills a half-step earlier.
#if TB_MUTATE != 3
          fence_proxy_async();
#endif
          __syncwarp();
#if TB_MUTATE != 2
          if (lane == 0) mbar_arrive(smem_u32(&empty[s]));
#endif
        }
        if (kt + 1 < ke) {
#if TB_MUTATE == 1
          ld(s1, 0, 0);
          mbar_wait(smem_u32(&full[s1]), ph1);
#else
          mbar_wait(smem_u32(&full[s1]), ph1);
#if TB_MUTATE == 2
          __syncwarp();
          if (lane == 0) mbar_arrive(smem_u32(&empty[s1]));
#endif
          ld(s1, 0, 0);
#endif
        }
        mma(1);
        if constexpr (!kEarlyRelease) {
#if TB_MUTATE != 3
          fence_proxy_async();
#endif
          __syncwarp();
#if TB_MUTATE != 2
          if (lane == 0) mbar_arrive(smem_u32(&empty[s]));
#endif
        }
        s = s1;
        ph = ph1;
      }
    } else
    for (int kt = kb; kt < ke; ++kt) {
#if TB_MUTATE != 1
      mbar_wait(smem_u32(&full[s]), ph);
#else
      if constexpr (MT == Math::DFMA) mbar_wait(smem_u32(&full[s]), ph);  // mutant 1 covers the DMMA loops
#endif
#if TB_MUTATE == 2
      __syncwarp();
      if (lane == 0) mbar_arrive(smem_u32(&empty[s]));
#endif
      TB_TL(if (tl && ct == 0 && kt == kb) { tl_u = tl_now(); if (tl[1] == 0) tl[1] = tl_u; })
      if constexpr (MT == Math::DFMA) {
#pragma unroll
        for (int u = 0; u < SUB; ++u) {
          const uint8_t* sa = smem + s * STAGE_BYTES + u * C::STAGE;
          const uint8_t* sb = sa + C::A_STAGE + (cw & 1) * 4 * C::B_BOX;
#pragma unroll
          for (int kp = 0; kp < C::BK / 2; ++kp) {
            double2 a[C::MI], b0[C::NI], b1[C::NI];
#pragma unroll
            for (int i = 0; i < C::MI; ++i) a[i] = *reinterpret_cast<const double2*>(sa + (dfma_a[i] ^ (kp << 4)));
            const uint32_t o0 = (2 * kp) * 128 + ((lc ^ ((2 * kp) & 7)) << 4);
            const uint32_t o1 = (2 * kp + 1) * 128 + ((lc ^ ((2 * kp + 1) & 7)) << 4);
#pragma unroll
            for (int j = 0; j < C::NI; ++j) {
              b0[j] = *reinterpret_cast<const double2*>(sb + j * C::B_BOX + o0);
              b1[j] = *reinterpret_cast<const double2*>(sb + j * C::B_BOX + o1);
            }
#pragma unroll
            for (int i = 0; i < C::MI; ++i)
#pragma unroll
              for (int j = 0; j < C::NI; ++j) {
                acc[i][j][0] = fma(a[i].x, b0[j].x, acc[i][j][0]);
                acc[i][j][1] = fma(a[i].x, b0[j].y, acc[i][j][1]);
              }
#pragma unroll
            for (int i = 0; i < C::MI; ++i)
#pragma unroll
              for (int j = 0; j < C::NI; ++j) {
                acc[i][j][0] = fma(a[i].y, b1[j].x, acc[i][j][0]);
                acc[i][j][1] = fma(a[i].y, b1[j].y, acc[i][j][1]);
              }
          }
        }
      } else {
#pragma unroll
      for (int hs = 0; hs < 2 * SUB; ++hs) {
        const int half = hs & 1;
        const uint8_t* sa = smem + s * STAGE_BYTES + (hs >> 1) * C::STAGE;
        const uint8_t* sb = sa + C::A_STAGE;
        double2 af[C::MI];
        double bf[2][C::NI];
#pragma unroll
        for (int i = 0; i < C::MI; ++i)
          af[i] = *reinterpret_cast<const double2*>(sa + (half ? a_off1 : a_off0) + i * 8 * 128);
#pragma unroll
        for (int j = 0; j < C::NI; ++j) {
          const uint32_t box = (j >> 1) * C::B_BOX, flip = (j & 1) ? 64u : 0u;
          bf[0][j] = *reinterpret_cast<const double*>(sb + box + (b_off[2 * half] ^ flip));
          bf[1][j] = *reinterpret_cast<const double*>(sb + box + (b_off[2 * half + 1] ^ flip));
        }
#if TB_MUTATE == 1
        if (hs == 0) mbar_wait(smem_u32(&full[s]), ph);
#endif
#pragma unroll
        for (int i = 0; i < C::MI; ++i)
#pragma unroll
          for (int j = 0; j < C::NI; ++j) dmma_8x8x4(acc[i][j][0], acc[i][j][1], af[i].x, bf[0][j]);
#pragma unroll
        for (int i = 0; i < C::MI; ++i)
#pragma unroll
          for (int j = 0; j < C::NI; ++j) dmma_8x8x4(acc[i][j][0], acc[i][j][1], af[i].y, bf[1][j]);
      }
      }
      // Release the stage to the producer. The fragment loads above are
      // generic-proxy reads that the next TMA (async proxy) into this stage
      // must not overtake: without the proxy fence ptxas issues the arrive
      // while the last LDS are still outstanding, and a TMA landing before
      // they are serviced corrupts those fragments (observed on B200 when the
      // accumulate epilogue's global loads back up the LSU queue).
#if TB_MUTATE != 3
      fence_proxy_async();
#endif
      __syncwarp();
#if TB_MUTATE != 2
      if (lane == 0) mbar_arrive(smem_u32(&empty[s]));
#endif
      if (++s == STAGES) {
        s = 0;
        ph ^= 1;
      }
    }

    TB_TL(const unsigned long long tl_m = tl && ct == 0 ? tl_now() : 0;)
    TB_TL(if (tl && ct == 0) { tl[2] = tl_m; tl[4] += 1; tl[7] += tl_m - tl_u; })
    // ------------------------------------------------- stream-K segment fixup
    if (!PIPE && (kb != 0 || ke != p.num_k)) {
      const int st = tile - p.dp_tiles;
      const int64_t first = (int64_t)st * p.num_k;
      const int seg = (int)((first + kb) / p.sk_ipc - first / p.sk_ipc);
      const int nseg = (int)((first + p.num_k - 1) / p.sk_ipc - first / p.sk_ipc + 1);
      double2* slots = reinterpret_cast<double2*>(p.partials) + (size_t)st * p.max_seg * (C::TILE_ELEMS / 2);
      double2* mine = slots + (size_t)seg * (C::TILE_ELEMS / 2);
      // A segment that finds every other segment already published is the
      // tile's last: it keeps its partial in registers (no store, no fence,
      // no atomic) — typically the CTA that ran the tile's first k-range at
      // the end of its work list, i.e. the launch's critical path. Others
      // publish (store, fence, count) and the one whose count completes the
      // tile reduces.
      if (ct == 0) *flag = ld_acquire_gpu(&p.counters[st]);
      consumer_bar();
      bool last = (*flag == nseg - 1);
      consumer_bar();  // flag is rewritten below / by the next unit
      if (!last) {
#pragma unroll
        for (int i = 0; i < C::MI; ++i)
#pragma unroll
          for (int j = 0; j < C::NI; ++j)
            __stcg(mine + (i * C::NI + j) * C::CONSUMER_THREADS + ct, make_double2(acc[i][j][0], acc[i][j][1]));
        __threadfence();
        consumer_bar();
        if (ct == 0) *flag = atomicAdd(&p.counters[st], 1);
        consumer_bar();
        last = (*flag == nseg - 1);
        consumer_bar();  // flag is reused by the next unit
        if (!last) {
          TB_TL(if (tl && ct == 0) { const unsigned long long t = tl_now(); tl[5] += t - tl_m; tl[3] = t; })
          continue;
        }
      }
      __threadfence();
      // Deterministic reduction: all segments summed in index order
      // 0..nseg-1, whichever CTA finishes last. This CTA's own partial enters
      // from registers: for seg <= 1 the running sum starts as own + p_other
      // (the first addition commutes, so this is bitwise p0 + p1) and the
      // rest are added in order; for seg >= 2 (split-K) it is stored to its
      // slot (if not already published) and all slots are summed from memory.
      if (seg <= 1) {
        for (int sg = 0; sg < nseg; ++sg) {
          if (sg == seg) continue;
          const double2* src = slots + (size_t)sg * (C::TILE_ELEMS / 2) + ct;
#pragma unroll
          for (int i = 0; i < C::MI; ++i)
#pragma unroll
            for (int j = 0; j < C::NI; ++j) {
              const double2 v = __ldcg(src + (i * C::NI + j) * C::CONSUMER_THREADS);
              acc[i][j][0] += v.x;
              acc[i][j][1] += v.y;
            }
        }
      } else {
#pragma unroll
        for (int i = 0; i < C::MI; ++i)
#pragma unroll
          for (int j = 0; j < C::NI; ++j)
            __stcg(mine + (i * C::NI + j) * C::CONSUMER_THREADS + ct, make_double2(acc[i][j][0], acc[i][j][1]));
#pragma unroll
        for (int i = 0; i < C::MI; ++i)
#pragma unroll
          for (int j = 0; j < C::NI; ++j) {
            const double2* src = slots + (i * C::NI + j) * C::CONSUMER_THREADS + ct;
            double2 sum = __ldcg(src);
            for (int sg = 1; sg < nseg; ++sg) {
              const double2 v = __ldcg(src + (size_t)sg * (C::TILE_ELEMS / 2));
              sum.x += v.x;
              sum.y += v.y;
            }
            acc[i][j][0] = sum.x;
            acc[i][j][1] = sum.y;
          }
      }
      if (ct == 0) p.counters[st] = 0;  // self-reset for the next launch
    }

    // --------------------------------------------------------------- epilogue
    TB_TL(const unsigned long long tl_e = tl && ct == 0 ? tl_now() : 0;)
    TB_TL(if (tl && ct == 0) tl[5] += tl_e - tl_m;)
    int tm, tn;
    tile_coords(tile, p.tiles_m, p.tiles_n, tm, tn);
    const int m0 = tm * C::BM, n0 = tn * C::BN;
    // C += A·B when asked; in PIPE mode also for every panel after the first.
#define TB_ACCUM (PIPE ? (p.accumulate || kb != 0) : p.accumulate)
    if (TB_ACCUM && p.vec_store && m0 + C::BM <= p.m && n0 + C::BN <= p.n) {
      // C += A·B on an interior tile: the old C values are fetched in two
      // batches of 16 independent 16-byte loads (no branches, no stores in
      // between), so the epilogue pays two memory round trips, not one per
      // element.
      constexpr int HALF = (C::MI + 1) / 2;  // odd MI (96-row tiles: 3): the second batch is one row shorter
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        double2 old[HALF][C::NI];
#pragma unroll
        for (int ii = 0; ii < HALF; ++ii) {
          if (h * HALF + ii >= C::MI) break;
          const double* crow = p.C + (int64_t)(m0 + row_base + (h * HALF + ii) * row_step) * p.ldc;
#pragma unroll
          for (int j = 0; j < C::NI; ++j)
            old[ii][j] = __ldcg(reinterpret_cast<const double2*>(crow + n0 + col_base + j * col_step));
        }
#pragma unroll
        for (int ii = 0; ii < HALF; ++ii) {
          if (h * HALF + ii >= C::MI) break;
#pragma unroll
          for (int j = 0; j < C::NI; ++j) {
            acc[h * HALF + ii][j][0] += old[ii][j].x;
            acc[h * HALF + ii][j][1] += old[ii][j].y;
          }
        }
      }
    } else if (TB_ACCUM) {
#undef TB_ACCUM
      // Edge tiles / unaligned rows: element-wise, bounds-checked.
#pragma unroll
      for (int i = 0; i < C::MI; ++i) {
        const int r = m0 + row_base + i * row_step;
        if (r >= p.m) continue;
        const double* crow = p.C + (int64_t)r * p.ldc;
#pragma unroll
        for (int j = 0; j < C::NI; ++j) {
          const int c = n0 + col_base + j * col_step;
          if (c + 1 < p.n) {
            if (p.vec_store) {
              const double2 o = __ldcg(reinterpret_cast<const double2*>(crow + c));
              acc[i][j][0] += o.x;
              acc[i][j][1] += o.y;
            } else {
              acc[i][j][0] += __ldcg(crow + c);
              acc[i][j][1] += __ldcg(crow + c + 1);
            }
          } else if (c < p.n) {
            acc[i][j][0] += __ldcg(crow + c);
          }
        }
      }
    }
#pragma unroll
    for (int i = 0; i < C::MI; ++i) {
      const int r = m0 + row_base + i * row_step;
      if (r >= p.m) continue;
      double* crow = p.C + (int64_t)r * p.ldc;
#pragma unroll
      for (int j = 0; j < C::NI; ++j) {
        const int c = n0 + col_base + j * col_step;
        const double v0 = acc[i][j][0], v1 = acc[i][j][1];
        if (c + 1 < p.n) {
          if (p.vec_store) {
            *reinterpret_cast<double2*>(crow + c) = make_double2(v0, v1);
          } else {
            crow[c] = v0;
            crow[c + 1] = v1;
          }
        } else if (c < p.n) {
          crow[c] = v0;
        }
      }
    }
    TB_TL(if (tl && ct == 0) { const unsigned long long t = tl_now(); tl[6] += t - tl_e; tl[3] = t; })
  }
}

}  // namespace tb
