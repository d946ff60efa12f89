// Tuning aid (not product): cost of page-locking a caller buffer in place
// (cudaHostRegister) vs staging it through the pinned slot ring.
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <cuda_runtime.h>
int main() {
  cudaFree(0);
  for (size_t gb : {1, 4}) {
    size_t bytes = gb << 30;
    char* p = (char*)aligned_alloc(4096, bytes);
    memset(p, 1, bytes);
    for (int rep = 0; rep < 2; ++rep) {
      auto t0 = std::chrono::steady_clock::now();
      cudaError_t e = cudaHostRegister(p, bytes, cudaHostRegisterDefault);
      auto t1 = std::chrono::steady_clock::now();
      void* d; cudaMalloc(&d, bytes);
      auto t2 = std::chrono::steady_clock::now();
      cudaMemcpy(d, p, bytes, cudaMemcpyHostToDevice);
      auto t3 = std::chrono::steady_clock::now();
      cudaError_t e2 = cudaHostUnregister(p);
      auto t4 = std::chrono::steady_clock::now();
      cudaFree(d);
      auto ms = [](auto a, auto b) { return std::chrono::duration<double, std::milli>(b - a).count(); };
      printf("%zu GB rep %d: register %.1f ms (%s), H2D %.1f ms (%.1f GB/s), unregister %.1f ms (%s)\n", gb, rep,
             ms(t0, t1), cudaGetErrorString(e), ms(t2, t3), bytes / ms(t2, t3) / 1e6, ms(t3, t4), cudaGetErrorString(e2));
    }
    free(p);
  }
}
