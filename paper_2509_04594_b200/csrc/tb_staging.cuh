// tb_staging.cuh — pageable host buffers at pinned speed (included by
// tb_capi.cu only). cudaMemcpyAsync from pageable memory runs through the
// driver's own single-threaded bounce buffer (N = 10000 host-buffer call:
// 239 ms vs 57 ms pinned) and registering the caller's buffers costs ~140 ms
// per GB. Instead the host pipeline stages pageable operands through a ring
// of pinned slots, filling and draining them with a small pool of copy
// threads (69 GB/s host-to-host on the GPU box's 16 cores).
#pragma once

#include <atomic>
#include <condition_variable>
#include <functional>
#include <memory>
#include <thread>

namespace {

// A fixed pool: run(parts, fn) calls fn(i) for every i in [0, parts) on the
// workers and the calling thread and returns when all are done. One run at
// a time (callers hold the device's host mutex). Inside a session
// (set_active(true) for the duration of a host-buffer call) idle workers
// spin on the run counter instead of sleeping, so the many small staging
// copies of a call do not each pay a futex wake-up (N = 4000: 16 panels ->
// ~1 ms per panel with sleeping workers).
class CopyPool {
 public:
  explicit CopyPool(int workers) {
    for (int i = 0; i < workers; ++i) th_.emplace_back([this] { worker(); });
  }
  ~CopyPool() {
    {
      std::lock_guard<std::mutex> lk(mu_);
      stop_.store(true);
      active_.store(false);
    }
    cv_.notify_all();
    for (auto& t : th_) t.join();
  }
  int threads() const { return (int)th_.size() + 1; }

  void set_active(bool on) {
    {
      std::lock_guard<std::mutex> lk(mu_);
      active_.store(on);
    }
    if (on) cv_.notify_all();
  }

  void run(int parts, const std::function<void(int)>& fn) {
    // Close the previous generation first: a worker still inside it fails
    // its CAS (or sees no parts left) before job_ / parts_ change.
    ctr_.store((gen_ << 32) | 0xffffffffu, std::memory_order_release);
    job_ = &fn;
    parts_ = parts;
    pending_.store(parts, std::memory_order_relaxed);
    {
      std::lock_guard<std::mutex> lk(mu_);
      ++gen_;
      // (generation << 32 | next part): a part is taken by a CAS that also
      // checks the generation, so a worker still looking at the previous
      // run can never take (or double-take) a part of this one.
      ctr_.store(gen_ << 32, std::memory_order_release);
    }
    if (!active_.load()) cv_.notify_all();
    drain_parts(gen_);
    while (pending_.load(std::memory_order_acquire) > 0) std::this_thread::yield();
  }

 private:
  void drain_parts(uint64_t g) {
    uint64_t v = ctr_.load(std::memory_order_acquire);
    for (;;) {
      if ((v >> 32) != g) return;
      const uint32_t i = (uint32_t)(v & 0xffffffffu);
      if (i >= (uint32_t)parts_) return;
      if (!ctr_.compare_exchange_weak(v, v + 1, std::memory_order_acq_rel, std::memory_order_acquire)) continue;
      (*job_)((int)i);
      pending_.fetch_sub(1, std::memory_order_acq_rel);
      v = ctr_.load(std::memory_order_acquire);
    }
  }
  void worker() {
    uint64_t seen = 0;
    for (;;) {
      uint64_t v;
      while (((v = ctr_.load(std::memory_order_acquire)) >> 32) == seen) {
        if (stop_.load()) return;
        if (active_.load()) {
          std::this_thread::yield();
          continue;
        }
        std::unique_lock<std::mutex> lk(mu_);
        cv_.wait(lk, [&] { return stop_.load() || active_.load() || (ctr_.load() >> 32) != seen; });
      }
      seen = v >> 32;
      drain_parts(seen);
    }
  }

  std::vector<std::thread> th_;
  std::mutex mu_;
  std::condition_variable cv_;
  const std::function<void(int)>* job_ = nullptr;
  int parts_ = 0;
  uint64_t gen_ = 0;  // written by run() only (under mu_)
  std::atomic<uint64_t> ctr_{0};
  std::atomic<int> pending_{0};
  std::atomic<bool> active_{false}, stop_{false};
};

// rows x width bytes from src (pitch spitch) to dst (pitch dpitch), split by
// rows over the pool.
void pool_copy_rows(CopyPool& pool, char* dst, size_t dpitch, const char* src, size_t spitch, size_t width,
                    size_t rows) {
  // 256 KB per part: one host thread copies ~4 GB/s, so a 5 MB panel slice
  // split by MB kept only 5 of the 16 threads busy (staged panels at 14-25
  // GB/s at N = 4000, below the 55 GB/s link).
  const size_t bytes = width * rows;
  const int parts = (int)std::max<size_t>(1, std::min<size_t>(std::min<size_t>((size_t)pool.threads(), bytes >> 18), rows));
  pool.run(parts, [&](int i) {
    const size_t r0 = rows * i / parts, r1 = rows * (i + 1) / parts;
    if (dpitch == width && spitch == width) {
      std::memcpy(dst + r0 * width, src + r0 * width, (r1 - r0) * width);
    } else {
      for (size_t r = r0; r < r1; ++r) std::memcpy(dst + r * dpitch, src + r * spitch, width);
    }
  });
}

// True when the host pointer is page-locked (cudaHostAlloc'd or registered).
bool is_pinned(const void* p) {
  cudaPointerAttributes at;
  if (cudaPointerGetAttributes(&at, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return at.type == cudaMemoryTypeHost;
}

// Pinned slots plus one event each marking the slot's last device copy.
struct StageRing {
  static constexpr int kSlots = 8;
  static constexpr size_t kSlotBytes = size_t(32) << 20;
  static constexpr int64_t kSlotCols = (int64_t)(kSlotBytes / sizeof(double));  // widest row chunk per slot
  char* slot[kSlots] = {};
  cudaEvent_t ev[kSlots] = {};
  int next = 0;
  std::unique_ptr<CopyPool> pool;

  int ensure() {
    if (pool) return TB_STATUS_OK;
    for (int i = 0; i < kSlots; ++i) {
      TB_CUDA(cudaHostAlloc(reinterpret_cast<void**>(&slot[i]), kSlotBytes, cudaHostAllocDefault),
              "pinned staging allocation");
      TB_CUDA(cudaEventCreateWithFlags(&ev[i], cudaEventDisableTiming), "event create");
    }
    const unsigned hw = std::thread::hardware_concurrency();
    pool.reset(new CopyPool((int)std::min<unsigned>(16, hw ? hw : 4) - 1));
    return TB_STATUS_OK;
  }
  void release() {
    pool.reset();
    for (int i = 0; i < kSlots; ++i) {
      if (slot[i]) cudaFreeHost(slot[i]);
      if (ev[i]) cudaEventDestroy(ev[i]);
      slot[i] = nullptr;
      ev[i] = nullptr;
    }
    next = 0;
  }
};

StageRing g_ring[kMaxDevices];  // per device; used under the device's host mutex

}  // namespace
