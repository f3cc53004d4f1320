// tb_staging.cuh — pageable host buffers at pinned speed (included by
// tb_capi.cu only). cudaMemcpyAsync from pageable memory runs through the
// driver's own single-threaded bounce buffer (N = 10000 host-buffer call:
// 239 ms vs 57 ms pinned) and registering the caller's buffers costs ~140 ms
// per GB. Instead the host pipeline stages pageable operands through a ring
// of pinned slots, filling and draining them with a small pool of copy
// threads (69 GB/s host-to-host on the GPU box's 16 cores).
#pragma once

#include <condition_variable>
#include <functional>
#include <memory>
#include <thread>

namespace {

// A fixed pool: run(parts, fn) calls fn(i) for every i in [0, parts) on the
// workers and the calling thread and returns when all are done. One run at
// a time (callers hold the device's host mutex).
class CopyPool {
 public:
  explicit CopyPool(int workers) {
    for (int i = 0; i < workers; ++i) th_.emplace_back([this] { worker(); });
  }
  ~CopyPool() {
    {
      std::lock_guard<std::mutex> lk(mu_);
      stop_ = true;
    }
    cv_.notify_all();
    for (auto& t : th_) t.join();
  }
  int threads() const { return (int)th_.size() + 1; }

  void run(int parts, const std::function<void(int)>& fn) {
    {
      std::lock_guard<std::mutex> lk(mu_);
      job_ = &fn;
      parts_ = parts;
      next_ = 0;
      pending_ = parts;
      ++gen_;
    }
    cv_.notify_all();
    drain_parts();
    std::unique_lock<std::mutex> lk(mu_);
    done_cv_.wait(lk, [this] { return pending_ == 0; });
    job_ = nullptr;
  }

 private:
  void drain_parts() {
    for (;;) {
      int i;
      const std::function<void(int)>* fn;
      {
        std::lock_guard<std::mutex> lk(mu_);
        if (!job_ || next_ >= parts_) return;
        i = next_++;
        fn = job_;
      }
      (*fn)(i);
      std::lock_guard<std::mutex> lk(mu_);
      if (--pending_ == 0) done_cv_.notify_all();
    }
  }
  void worker() {
    uint64_t seen = 0;
    for (;;) {
      {
        std::unique_lock<std::mutex> lk(mu_);
        cv_.wait(lk, [&] { return stop_ || gen_ != seen; });
        if (stop_) return;
        seen = gen_;
      }
      drain_parts();
    }
  }

  std::vector<std::thread> th_;
  std::mutex mu_;
  std::condition_variable cv_, done_cv_;
  const std::function<void(int)>* job_ = nullptr;
  int parts_ = 0, next_ = 0, pending_ = 0;
  uint64_t gen_ = 0;
  bool stop_ = false;
};

// rows x width bytes from src (pitch spitch) to dst (pitch dpitch), split by
// rows over the pool.
void pool_copy_rows(CopyPool& pool, char* dst, size_t dpitch, const char* src, size_t spitch, size_t width,
                    size_t rows) {
  const size_t bytes = width * rows;
  const int parts = (int)std::max<size_t>(1, std::min<size_t>((size_t)pool.threads(), bytes >> 20));
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
