// host_staging.h — host side of the end-to-end path for PAGEABLE buffers.
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
// OutOfDomain" only needs to know that no query is bad, and the host can
// establish that at ~100 GB/s (16 threads, AVX2), faster than PCIe uploads
// the queries.  The device kernels still perform their own fused check and
// report the position.
// ---------------------------------------------------------------------------
template <typename T>
inline uint64_t scan_span_generic(const T* z, uint64_t a, uint64_t b, T x0, T xn) {
  constexpr uint64_t kBlock = 4096;
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
__attribute__((target("avx2"), optimize("O3"))) uint64_t scan_span_avx2(const T* z, uint64_t a, uint64_t b, T x0,
                                                                          T xn) {
  constexpr uint64_t kBlock = 4096;
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

// First position in z[0, m) outside [x0, xn), ~0 if none; n threads over
// contiguous spans (the smallest bad position wins).
template <typename T>
uint64_t host_first_bad(const T* z, uint64_t m, T x0, T xn, int n) {
  static const bool avx2 = __builtin_cpu_supports("avx2");
  auto scan = [&](uint64_t a, uint64_t b) {
    return avx2 ? scan_span_avx2<T>(z, a, b, x0, xn) : scan_span_generic<T>(z, a, b, x0, xn);
  };
  if (n <= 1 || m < (1u << 20)) return scan(0, m);
  std::vector<uint64_t> res(n, ~0ull);
  std::vector<std::thread> th;
  const uint64_t per = (m + n - 1) / n;
  for (int i = 1; i < n; ++i)
    th.emplace_back([&, i] { res[i] = scan(std::min(m, per * i), std::min(m, per * (i + 1))); });
  res[0] = scan(0, std::min(m, per));
  for (auto& t : th) t.join();
  return *std::min_element(res.begin(), res.end());
}

inline int host_scan_threads() {
  if (const char* e = std::getenv("FSG_SCAN_THREADS")) {  // tuning override
    const int n = std::atoi(e);
    if (n > 0) return std::min(n, 64);
  }
  const unsigned hc = std::thread::hardware_concurrency();
  return (int)std::max(1u, std::min(32u, hc ? hc : 4u));
}

inline int host_copy_threads() {
  if (const char* e = std::getenv("FSG_COPY_THREADS")) {  // tuning override
    const int n = std::atoi(e);
    if (n > 0) return std::min(n, 64);
  }
  const unsigned hc = std::thread::hardware_concurrency();
  return (int)std::max(2u, std::min(16u, hc ? hc / 2 : 4u));
}

}  // namespace fsg
