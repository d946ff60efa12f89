// host_staging.h — host side of the end-to-end path: pinned staging of
// PAGEABLE buffers, and the host half of the two-sided domain check.
//
// cudaMemcpyAsync from pageable memory goes through the driver's bounce
// buffer at ~14 GB/s here (measured: 1.7 G queries/s end to end on cfg3
// versus 6.9 with pinned arrays).  A numpy array handed to batch_search is
// pageable, so the library stages it itself: a small ring of pinned slots
// (cached process-wide, reused across calls) filled / drained by the
// process-wide host pool doing parallel memcpy, overlapped with the DMA of the
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
#include <deque>
#include <functional>
#include <unistd.h>
#include <mutex>
#include <thread>
#include <vector>

namespace fsg {

// Process-wide pool of host worker threads, created once per process on first
// use and kept for its lifetime (re-created in a forked child, whose copy of
// the parent's pool has no threads).  Every host-side parallel step of the
// end-to-end path -- the parallel memcpy of pageable staging and the host
// half of the two-sided domain check -- runs as a job on it, so no call
// spawns or joins threads (that cost hundreds of microseconds per call,
// against ~0.1 ms of PCIe for a 4 MB batch).  Jobs from concurrent callers
// queue and run in order; a caller may help run its own job's tasks.
class HostPool {
 public:
  struct Job {
    std::function<void(int)> fn;
    int n = 0;
    int next = 0, finished = 0;  // guarded by the pool mutex
    std::condition_variable cv;
  };

  static HostPool& get();
  int size() const { return (int)threads_.size(); }

  std::shared_ptr<Job> submit(int n, std::function<void(int)> fn) {
    auto job = std::make_shared<Job>();
    job->fn = std::move(fn);
    job->n = n;
    if (n <= 0) return job;
    {
      std::lock_guard<std::mutex> lk(mu_);
      q_.push_back(job);
    }
    cv_.notify_all();
    return job;
  }
  // Wait for every task of `job`; with `help` the caller runs unclaimed tasks itself.
  void wait(const std::shared_ptr<Job>& job, bool help) {
    std::unique_lock<std::mutex> lk(mu_);
    while (help && job->next < job->n) {
      const int i = job->next++;
      lk.unlock();
      job->fn(i);
      lk.lock();
      ++job->finished;
    }
    job->cv.wait(lk, [&] { return job->finished == job->n; });
    // a fully claimed job may still sit in the queue; workers drop it lazily
  }
  void run(int n, std::function<void(int)> fn) { wait(submit(n, std::move(fn)), true); }

 private:
  explicit HostPool(int n) {
    for (int i = 0; i < n; ++i) threads_.emplace_back([this] { worker(); });
  }
  void worker() {
    std::unique_lock<std::mutex> lk(mu_);
    for (;;) {
      cv_.wait(lk, [&] { return !q_.empty(); });
      std::shared_ptr<Job> job = q_.front();
      if (job->next >= job->n) {
        q_.pop_front();
        continue;
      }
      const int i = job->next++;
      if (job->next >= job->n) q_.pop_front();
      lk.unlock();
      job->fn(i);
      lk.lock();
      if (++job->finished == job->n) job->cv.notify_all();
    }
  }
  std::vector<std::thread> threads_;  // detached at exit: the pool lives as long as the process
  std::mutex mu_;
  std::condition_variable cv_;
  std::deque<std::shared_ptr<Job>> q_;
};

// Processes sharing this host's cores: one per GPU under torchrun
// (LOCAL_WORLD_SIZE), so N ranks do not oversubscribe the host N times over.
inline unsigned host_procs() {
  if (const char* e = std::getenv("LOCAL_WORLD_SIZE")) {
    const int n = std::atoi(e);
    if (n > 1) return (unsigned)n;
  }
  return 1u;
}

inline int env_threads(const char* name) {
  if (const char* e = std::getenv(name)) {  // tuning override
    const int n = std::atoi(e);
    if (n > 0) return std::min(n, 64);
  }
  return 0;
}

inline int host_share() {
  const unsigned hc = std::thread::hardware_concurrency();
  return (int)std::max(1u, std::min(32u, (hc ? hc : 4u) / host_procs()));
}

inline int host_scan_threads() {
  const int n = env_threads("FSG_SCAN_THREADS");
  return n ? n : host_share();
}

inline int host_copy_threads() {
  // every hardware thread (this process's share of them): staging is host-
  // memory-bandwidth bound (tools/pageable_threads.py on the 16-core GPU
  // host: 8 -> 4.7, 16 -> 5.2 G queries/s)
  const int n = env_threads("FSG_COPY_THREADS");
  return n ? n : std::max(2, host_share());
}

inline HostPool& HostPool::get() {
  static std::mutex mu;
  static HostPool* pool = nullptr;
  static pid_t owner = 0;
  std::lock_guard<std::mutex> lk(mu);
  if (!pool || owner != getpid()) {  // first use, or a forked child
    pool = new HostPool(std::max(host_copy_threads(), host_scan_threads()));
    for (auto& t : pool->threads_) t.detach();
    owner = getpid();
  }
  return *pool;
}

// Parallel memcpy over `n` slices on the host pool (the caller runs slices too).
inline void host_copy(void* dst, const void* src, size_t bytes, int n) {
  n = std::max(1, std::min(n, HostPool::get().size() + 1));
  if (n == 1 || bytes < (1u << 20)) {
    std::memcpy(dst, src, bytes);
    return;
  }
  char* d = static_cast<char*>(dst);
  const char* s = static_cast<const char*>(src);
  const size_t per = ((bytes + n - 1) / n + 63) & ~size_t(63);
  HostPool::get().run(n, [=](int i) {
    const size_t a = std::min(bytes, per * i), b = std::min(bytes, a + per);
    if (b > a) std::memcpy(d + a, s + a, b - a);
  });
}

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
  auto job = HostPool::get().submit(std::max(1, std::min(nthreads, HostPool::get().size())),
                                    [&](int) { worker(); });
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
  HostPool::get().wait(job, false);  // tasks not yet started return at once
  return !bad.load();
}

}  // namespace fsg
