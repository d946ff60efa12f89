// host_staging.h — host side of the end-to-end path: pinned staging of
// PAGEABLE buffers, and the host half of the two-sided domain check.
//
// cudaMemcpyAsync from pageable memory goes through the driver's bounce
// buffer at ~14 GB/s here (measured: 1.7 G queries/s end to end on cfg3
// versus 6.9 with pinned arrays).  A numpy array handed to batch_search is
// pageable, so the library stages it itself: a small ring of pinned slots
// (cached process-wide, reused across calls) filled / drained by a pool of
// host threads doing parallel memcpy, overlapped with the DMA of the
// previous slot on the copy engine.
#pragma once

#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <memory>
#include <condition_variable>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <thread>
#include <vector>

namespace fsg {

// Parallel memcpy by n threads (the caller is thread 0); workers live for
// the lifetime of the pool.
class CopyPool {
 public:
  explicit CopyPool(int n) : n_(std::max(1, n)) {
    for (int i = 1; i < n_; ++i) threads_.emplace_back([this, i] { worker(i); });
  }
  ~CopyPool() {
    {
      std::lock_guard<std::mutex> lk(mu_);
      stop_ = true;
      ++gen_;
    }
    cv_.notify_all();
    for (auto& t : threads_) t.join();
  }
  CopyPool(const CopyPool&) = delete;
  CopyPool& operator=(const CopyPool&) = delete;

  void copy(void* dst, const void* src, size_t bytes) {
    if (n_ == 1 || bytes < (1u << 20)) {
      std::memcpy(dst, src, bytes);
      return;
    }
    {
      std::lock_guard<std::mutex> lk(mu_);
      dst_ = static_cast<char*>(dst);
      src_ = static_cast<const char*>(src);
      bytes_ = bytes;
      pending_ = n_ - 1;
      ++gen_;
    }
    cv_.notify_all();
    slice(0, dst_, src_, bytes_);
    std::unique_lock<std::mutex> lk(mu_);
    done_.wait(lk, [this] { return pending_ == 0; });
  }

 private:
  void slice(int i, char* dst, const char* src, size_t bytes) const {
    const size_t per = ((bytes + n_ - 1) / n_ + 63) & ~size_t(63);
    const size_t a = std::min(bytes, per * i), b = std::min(bytes, a + per);
    if (b > a) std::memcpy(dst + a, src + a, b - a);
  }
  void worker(int i) {
    unsigned long long seen = 0;
    std::unique_lock<std::mutex> lk(mu_);
    for (;;) {
      cv_.wait(lk, [&] { return gen_ != seen; });
      seen = gen_;
      if (stop_) return;
      char* d = dst_;
      const char* s = src_;
      const size_t b = bytes_;
      lk.unlock();
      slice(i, d, s, b);
      lk.lock();
      if (--pending_ == 0) done_.notify_one();
    }
  }

  int n_;
  std::vector<std::thread> threads_;
  std::mutex mu_;
  std::condition_variable cv_, done_;
  unsigned long long gen_ = 0;
  bool stop_ = false;
  char* dst_ = nullptr;
  const char* src_ = nullptr;
  size_t bytes_ = 0;
  int pending_ = 0;
};

// Process-wide cache of pinned staging slots (allocation pins pages and is
// slow; a slot is reused by later calls once released).
class PinnedSlots {
 public:
  static void* acquire(size_t bytes) {
    std::lock_guard<std::mutex> lk(mu());
    auto& fl = free_list();
    for (size_t i = 0; i < fl.size(); ++i)
      if (fl[i].second >= bytes) {
        void* p = fl[i].first;
        fl.erase(fl.begin() + i);
        return p;
      }
    void* p = nullptr;
    if (cudaHostAlloc(&p, bytes, cudaHostAllocDefault) != cudaSuccess) return nullptr;
    sizes().push_back({p, bytes});
    return p;
  }
  static void release(void* p) {
    std::lock_guard<std::mutex> lk(mu());
    for (auto& e : sizes())
      if (e.first == p) free_list().push_back(e);
  }

 private:
  static std::mutex& mu() {
    static std::mutex m;
    return m;
  }
  static std::vector<std::pair<void*, size_t>>& free_list() {
    static std::vector<std::pair<void*, size_t>> v;
    return v;
  }
  static std::vector<std::pair<void*, size_t>>& sizes() {
    static std::vector<std::pair<void*, size_t>> v;
    return v;
  }
};

inline bool is_pinned(const void* p) {
  cudaPointerAttributes a;
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();  // clear the sticky-free error of an unknown pointer
    return false;
  }
  return a.type == cudaMemoryTypeHost;
}

// ---------------------------------------------------------------------------
// Host-side domain check of the queries (the compare of batch.py:411-413,
// NaN included), run while the uploads and searches of the same call are in
// flight.  It lets the default (atomic) end-to-end path start writing results
// back before the last chunk has been uploaded: "nothing is written on
// OutOfDomain" only needs to know that no query is bad, and host threads
// (AVX2, ~100 GB/s with 16 threads) scanning from the end meet the device's
// own fused check, which advances from the start at the PCIe upload rate.
// The device still reports the position.
// ---------------------------------------------------------------------------
template <typename T>
__attribute__((always_inline)) inline uint64_t scan_span_body(const T* z, uint64_t a, uint64_t b, T x0, T xn) {
  constexpr uint64_t kBlock = 4096;  // branch-free (vectorised) test per block, exact scan only if it fails
  for (uint64_t i = a; i < b; i += kBlock) {
    const uint64_t e = std::min(b, i + kBlock);
    int bad = 0;
    for (uint64_t k = i; k < e; ++k) bad |= (int)!(z[k] >= x0) | (int)!(z[k] < xn);
    if (bad)
      for (uint64_t k = i; k < e; ++k)
        if (!(z[k] >= x0 && z[k] < xn)) return k;
  }
  return ~0ull;
}
template <typename T>
uint64_t scan_span_generic(const T* z, uint64_t a, uint64_t b, T x0, T xn) {
  return scan_span_body<T>(z, a, b, x0, xn);
}
template <typename T>
__attribute__((target("avx2"), optimize("O3"))) uint64_t scan_span_avx2(const T* z, uint64_t a, uint64_t b, T x0,
                                                                          T xn) {
  return scan_span_body<T>(z, a, b, x0, xn);
}

// Two-sided domain check of the atomic host path.  The device checks every
// chunk as it arrives: prefix_bad[c] (copied to pinned memory before done[c]
// fires) is the first bad position in chunks 0..c, so the device covers a
// prefix that grows at the PCIe upload rate.  Host threads scan chunks from
// the END at host-memory speed.  Returns true once the two meet with no bad
// query; false as soon as either side sees one (the caller then reports the
// device's position and writes nothing).
template <typename T>
bool domain_clean_two_sided(const T* z, uint64_t m, uint64_t chunk, T x0, T xn, int nthreads,
                            const cudaEvent_t* done, const volatile unsigned long long* prefix_bad, int64_t nch) {
  static const bool avx2 = __builtin_cpu_supports("avx2");
  constexpr uint64_t kSlice = 1u << 20;  // elements between stop checks
  std::atomic<int64_t> next{nch - 1}, gpu_upto{-1};
  std::atomic<bool> stop{false}, bad{false};
  std::unique_ptr<std::atomic<char>[]> clean(new std::atomic<char>[nch]);
  for (int64_t c = 0; c < nch; ++c) clean[c].store(0, std::memory_order_relaxed);
  auto worker = [&] {
    for (;;) {
      const int64_t c = next.fetch_sub(1);
      if (c < 0 || c <= gpu_upto.load()) return;
      const uint64_t e = std::min(m, (uint64_t)(c + 1) * chunk);
      for (uint64_t a = (uint64_t)c * chunk; a < e; a += kSlice) {
        if (stop.load(std::memory_order_relaxed)) return;
        const uint64_t b = std::min(e, a + kSlice);
        if ((avx2 ? scan_span_avx2<T>(z, a, b, x0, xn) : scan_span_generic<T>(z, a, b, x0, xn)) != ~0ull) {
          bad.store(true);
          stop.store(true);
          return;
        }
      }
      clean[c].store(1);
    }
  };
  std::vector<std::thread> th;
  for (int i = 0; i < std::max(1, nthreads); ++i) th.emplace_back(worker);
  int64_t g = -1;  // chunks [0, g] verified by the device
  while (!bad.load()) {
    while (g + 1 < nch && cudaEventQuery(done[g + 1]) == cudaSuccess) {
      if (prefix_bad[g + 1] != ~0ull) {
        bad.store(true);
        break;
      }
      gpu_upto.store(++g);
    }
    bool covered = true;
    for (int64_t c = g + 1; c < nch && covered; ++c) covered = clean[c].load() != 0;
    if (covered) break;
    std::this_thread::sleep_for(std::chrono::microseconds(20));
  }
  stop.store(true);
  for (auto& t : th) t.join();
  return !bad.load();
}

// Processes sharing this host's cores: one per GPU under torchrun
// (LOCAL_WORLD_SIZE), so N ranks do not oversubscribe the host N times over.
inline unsigned host_procs() {
  if (const char* e = std::getenv("LOCAL_WORLD_SIZE")) {
    const int n = std::atoi(e);
    if (n > 1) return (unsigned)n;
  }
  return 1u;
}

inline int host_scan_threads() {
  if (const char* e = std::getenv("FSG_SCAN_THREADS")) {  // tuning override
    const int n = std::atoi(e);
    if (n > 0) return std::min(n, 64);
  }
  const unsigned hc = std::thread::hardware_concurrency();
  return (int)std::max(1u, std::min(32u, (hc ? hc : 4u) / host_procs()));
}

inline int host_copy_threads() {
  if (const char* e = std::getenv("FSG_COPY_THREADS")) {  // tuning override
    const int n = std::atoi(e);
    if (n > 0) return std::min(n, 64);
  }
  // every hardware thread (this process's share of them): staging is host-
  // memory-bandwidth bound (tools/pageable_threads.py on the 16-core GPU
  // host: 8 -> 4.7, 16 -> 5.2 G queries/s)
  const unsigned hc = std::thread::hardware_concurrency();
  return (int)std::max(2u, std::min(32u, (hc ? hc : 4u) / host_procs()));
}

}  // namespace fsg
