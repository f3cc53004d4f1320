// tb_pipeline.cuh — the host-buffer pipeline's shape (pure host code,
// included by tb_capi.cu only; exported as tb_pipeline_plan for tests):
// phase-1 rows and K-panels, phase-2 row blocks.
#pragma once

// The host pipeline's shape (pure; exported as tb_pipeline_plan for tests).
struct PipePlan {
  int64_t Mq = 0;
  bool fused = false;          // phase 1 as one PIPE-mode launch
  std::vector<int64_t> pk;     // phase-1 K-panel bounds
  std::vector<int64_t> gb;     // phase-1 row groups (one per compute stream)
  std::vector<int64_t> rb;     // phase-2 row-block bounds, rb[0] = Mq
};

// staged_inputs: A or B is pageable and goes through the pinned staging ring,
// whose host copies share host DRAM bandwidth with the DMA: the effective
// H2D rate is ~42 GB/s instead of 55, so phase 1 needs more rows to outlast
// its transfers (N = 10000 numpy operands: Mq 5248 -> 7168 rows, 64.6 ->
// 59.0 ms; profiles/r01_pipe_staged_mq.txt).
// staged_output: C is pageable and drains through the same ring; the drain
// (DMA into a slot, then the pool's copy out) runs at ~28 GB/s, so phase 1
// must leave more rows to phase 2 (N = 10000 all-numpy: Mq 6144, 59.2 ms;
// with the pinned-C cap 7168, 64.2 ms).
PipePlan plan_pipeline(int64_t m, int64_t k, int64_t n, int sms, bool fused_ok, bool staged_inputs = false,
                       bool staged_output = false) {
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
  // Pipelined from 1e9 flops (N ~ 800): N = 1000 / 2000 / 3000 pinned
  // 0.58 / 2.26 / 5.52 (one copy / GEMM / copy sequence) -> 0.50 / 1.59 /
  // 3.49 ms (profiles/r01_pipe_min_flops.txt, r01_pipe_fused_threshold.txt,
  // r01_pipe_small_blocks.txt).
  static const double min_flops = [] {  // TB_PIPE_MIN_FLOPS: tuning override
    const char* e = std::getenv("TB_PIPE_MIN_FLOPS");
    return e ? std::atof(e) : 1e9;
  }();
  if (flops >= min_flops) {
    constexpr double kRate = 36e12;                       // flop/s (FP64 DMMA)
    const double kH2D = staged_inputs ? 42e9 : 55e9;       // B/s (PCIe gen5 x16 / through staging, measured)
    const double den = (double)n * kH2D - 4.0 * kRate;
    int64_t mq = den > 0 ? (int64_t)(1.2 * 4.0 * kRate * (double)n / den) : m;
    // Phase-2 row blocks of ~m/4 rows (512..1536, on tile bounds): smaller
    // problems need finer blocks for their D2H to overlap (N = 2000: 1536-row
    // blocks 1.85 ms, 512-row 1.66; profiles/r01_pipe_small_blocks.txt).
    int64_t kp0 = 256, kp_max = 2048, groups = 2;
    if (const char* e = std::getenv("TB_PIPE_KP0")) kp0 = std::max<long long>(16, std::atoll(e));        // tuning
    if (const char* e = std::getenv("TB_PIPE_KPMAX")) kp_max = std::max<long long>(16, std::atoll(e));   // tuning
    int64_t blk = std::min<int64_t>(1536, std::max<int64_t>(512, (m / 4 + 64) / 128 * 128));
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
    // ... but leave phase 2 enough work to hide phase 1's C on its way back:
    // Mq·n·8 bytes at the D2H rate <= (m - Mq)·n·2k flops at kRate, i.e.
    // Mq <= m·c / (c + 1.2·8/D2H) with c = 2k/kRate and a x1.2 margin. Before
    // the cap, N = 4000 / 6000 ran all rows in phase 1 and copied the whole
    // C after the last GEMM: 7.66 / 18.4 ms pinned, now 6.59 / 15.2
    // (profiles/r01_pipe_staged_mq.txt).
    const double c2k = 2.0 * (double)k / kRate, kD2H = staged_output ? 28e9 : 53e9;
    const int64_t mq_cap =
        std::max<int64_t>(128, (int64_t)((double)m * c2k / (c2k + 1.2 * 8.0 / kD2H)) / 128 * 128);
    if (!std::getenv("TB_PIPE")) mq = std::min(mq, mq_cap);
    // D2H-bound sizes: every row of C leaves after B has fully landed (phase-1 rows need all K-panels),
    // so all of C's D2H (8mn/D) must fit under phase 2's compute, (m - Mq)·2kn/F: Mq <= m(1 - 4F/(D·k)).
    // Where that binds (N ~ 3000-7000 pinned), phase-2 blocks shrink to ~0.3 ms of compute each (>= 256
    // rows) so C streams back while A still streams in (pinned e2e N = 4000 / 5000 / 6000: 6.38 / 11.38 /
    // 16.19 -> 6.08 / 10.75 / 14.71 ms before the first-panel change below, profiles/r02_pipe_d2h_cap.txt).
    // TB_PIPE_D2HCAP=0 disables (A/B).
    const char* dce = std::getenv("TB_PIPE_D2HCAP");
    if (!std::getenv("TB_PIPE") && !(dce && std::strcmp(dce, "0") == 0)) {
      const double f = 1.0 - 4.0 * kRate / (kD2H * (double)k);
      const int64_t cap2 = f > 0 ? std::max<int64_t>(128, (int64_t)((double)m * f) / 128 * 128) : 128;
      if (cap2 < mq) {
        mq = cap2;
        const int64_t b3 = (int64_t)(0.3e-3 * kRate / (2.0 * (double)k * (double)n)) / 128 * 128;
        blk = std::max<int64_t>(256, std::min(blk, b3));
        // With the smaller phase 1, a 512-deep first panel (fewer, larger panel GEMMs) wins:
        // N = 3000 / 4000 / 5000 / 6000 -1.8 / -1.1 / -4.6 / -1.2 % (profiles/r02_pipe_d2h_cap.txt).
        if (!std::getenv("TB_PIPE_KP0")) kp0 = std::max<int64_t>(kp0, 512);
      }
    }
    if (const char* e = std::getenv("TB_PIPE_BLK")) blk = std::max<long long>(128, std::atoll(e));  // tuning
    // Phase 1 as one persistent launch that waits on per-panel flags (PIPE
    // mode) rather than a launch per panel and row group, from 2e11 flops:
    // below that (N <= ~4600) the launch-per-panel form is as fast or faster
    // (pinned N = 1200 / 2000 / 3000 / 4000: 0.95 / 1.85 / 3.52 / 6.31 ms vs
    // fused 1.06 / 1.93 / 3.67 / 6.49), above it the fused launch wins
    // (N = 5000 / 10000: 10.53 / 57.2 vs 10.75 / 59.9;
    // profiles/r01_pipe_fused_threshold.txt). TB_PIPE_FUSED=0 / 1 forces
    // either form (A/B).
    const char* fe = std::getenv("TB_PIPE_FUSED");
    fused = fused_ok && (fe ? std::strcmp(fe, "0") != 0 : flops >= 2e11);
    if (fused && !std::getenv("TB_PIPE")) {
      // The fused launch gives CTA c the phase-1 tiles c, c + P, ...: pick
      // the tile-row count (>= the compute-cover minimum, up to 8 more) whose
      // tile count leaves the least imbalance, ceil(T/P) - T/P (N = 10000:
      // 34 rows -> 18.15 tiles per CTA, 59.1 ms; 41 rows -> 21.89, 58.0 ms;
      // profiles/r01_pipe_trace_mq_sweep.txt).
      const int64_t tn = (n + 127) / 128, P_sm = sms;
      int64_t best_r = mq / 128;
      double best_imb = 2.0;
      for (int64_t rr = mq / 128; rr <= mq / 128 + 8 && rr * 128 < m - blk / 2 && rr * 128 <= mq_cap; ++rr) {
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
    // Later panels are at least k / max_panels deep: when the transfers only
    // just keep up (staged operands) the slack rule alone leaves every panel
    // at kp0, and each panel costs the phase-1 launch an accumulating
    // epilogue per tile (TB_PIPE_MAXP, 0 = no floor).
    static const int64_t max_panels = [] {
      const char* e = std::getenv("TB_PIPE_MAXP");
      return e ? (int64_t)std::atoll(e) : (int64_t)0;
    }();
    const int64_t kp_floor = max_panels > 0 ? std::max<int64_t>(kp0, k / max_panels) : kp0;
    for (int64_t at = 0, step = kp0; at < k;) {
      int64_t nx = at + step >= k - step / 2 ? k : ((at + step) / kal * kal);
      if (nx <= at) nx = std::min<int64_t>(k, at + kal);
      arrive += tr_per_k * (double)(nx - at);
      finish = std::max(finish, arrive) + c_per_k * (double)(nx - at);
      pk.push_back(nx);
      at = nx;
      step = std::min<int64_t>(kp_max, std::max<int64_t>(kp_floor, (int64_t)((finish - arrive) / tr_per_k)));
    }
    // Below 2e10 flops (N <~ 2150) there is no phase 1: B lands first (one
    // copy) and every row of C comes from full-K row blocks whose copies and
    // GEMMs overlap (pinned N = 1000 / 1500 / 2000: 0.58 / 0.96 / 1.66 ->
    // 0.50 / 0.92 / 1.59 ms; from N = 3000 up the panel phase wins;
    // profiles/r01_pipe_small_blocks.txt). TB_PIPE_MQ0=0 / 1 forces (A/B).
    const char* m0e = std::getenv("TB_PIPE_MQ0");
    const bool mq0 = m0e ? std::strcmp(m0e, "1") == 0 : flops < 2e10;
    if (mq0 && !fused) {
      Mq = 0;
      pk = {0, k};
      // ~256-row blocks here (N = 1000 / 1500 / 2000: 0.64 / 0.98 / 1.58 ->
      // 0.60 / 0.95 / 1.53 ms against ~m/4; profiles/r01_pipe_small_blocks.txt)
      if (!std::getenv("TB_PIPE")) blk = 256;
    }
    gb = (groups >= 2 && Mq >= 2048) ? std::vector<int64_t>{0, (Mq / 2 + 127) / 128 * 128, Mq}
                                     : std::vector<int64_t>{0, Mq};
    int64_t r = m - Mq;
    std::vector<int64_t> tail, tsz{std::min<int64_t>(128, blk / 4), blk / 6, blk / 3};
    // TB_TAIL=t0,t1,... (last block first) overrides the tail sizes (tuning).
    if (const char* e = std::getenv("TB_TAIL")) {
      tsz.clear();
      for (const char* q = e; *q;) {
        char* end = nullptr;
        const long long v = std::strtoll(q, &end, 10);
        if (end == q) break;
        if (v > 0) tsz.push_back(v);
        q = *end == ',' ? end + 1 : end;
      }
    }
    // Shrinking tail (N = 10000: ..., 512, 256, 144 rows): each block's D2H
    // ends about when the next block's GEMM does, so the copies after the
    // last GEMM are ~20 MB (57.4 -> 57.1 ms, profiles/r01_pipe_tail_sweep.txt).
    for (int64_t t : tsz)
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
  if (pl.pk.size() - 1 < 2 || pl.pk.size() - 1 > (size_t)tb::kPipeMaxPanels) pl.fused = false;  // flag table size
  return pl;
}
