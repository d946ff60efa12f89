// Micro-benchmark (tuning aid, not product): random 8-B per-lane gathers from
// an L2-resident table (the rank directory's access pattern: cfg5 N+1 = 2^20+1
// reads one 8-B word of a 2.5 MB directory per query) under each global load
// cache operator, to see whether bypassing or not allocating in L1 changes
// the L1TEX cost of a gather (node_probe.cu measures ~31 SM-cycles per warp
// instruction with ld.global.nc).
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o gather_ops_probe gather_ops_probe.cu && ./gather_ops_probe
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e)); return 1; } } while (0)

__device__ __forceinline__ uint32_t hash(uint32_t x) {
  x ^= x >> 16; x *= 0x7feb352dU; x ^= x >> 15; x *= 0x846ca68bU; x ^= x >> 16;
  return x;
}

template <int OP>
__device__ __forceinline__ unsigned long long ld8(const unsigned long long* p) {
  unsigned long long v;
  if constexpr (OP == 0) asm volatile("ld.global.nc.u64 %0, [%1];" : "=l"(v) : "l"(p));
  else if constexpr (OP == 1) asm volatile("ld.global.nc.L1::no_allocate.u64 %0, [%1];" : "=l"(v) : "l"(p));
  else if constexpr (OP == 2) asm volatile("ld.global.cg.u64 %0, [%1];" : "=l"(v) : "l"(p));
  else if constexpr (OP == 3) asm volatile("ld.global.ca.u64 %0, [%1];" : "=l"(v) : "l"(p));
  else if constexpr (OP == 4) asm volatile("ld.global.cs.u64 %0, [%1];" : "=l"(v) : "l"(p));
  else if constexpr (OP == 5) asm volatile("ld.global.nc.L1::evict_last.u64 %0, [%1];" : "=l"(v) : "l"(p));
  else asm volatile("ld.global.lu.u64 %0, [%1];" : "=l"(v) : "l"(p));
  return v;
}

static const char* kOpName[] = {"ld.global.nc", "ld.global.nc.L1::no_allocate", "ld.global.cg", "ld.global.ca",
                                "ld.global.cs", "ld.global.nc.L1::evict_last", "ld.global.lu"};

template <int OP>
__global__ void probe(const unsigned long long* __restrict__ tab, uint32_t nrows, int iters,
                      unsigned long long* sink) {
  constexpr int U = 8;
  uint32_t st = hash((blockIdx.x * blockDim.x + threadIdx.x) * 7919u + 77u);
  unsigned long long acc = 0;
  for (int it = 0; it < iters; ++it) {
    unsigned long long v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      st = hash(st + u);
      v[u] = ld8<OP>(tab + st % nrows);
    }
#pragma unroll
    for (int u = 0; u < U; ++u) acc ^= v[u];
  }
  if (acc == 0x1234567890ull) sink[0] = acc;
}

template <int OP>
int run(const unsigned long long* tab, size_t tb, int sms, unsigned long long* sink) {
  const uint32_t nrows = (uint32_t)(tb / 8);
  const int iters = 64;
  for (int threads : {256, 512}) {
    int per_sm = 0;
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, probe<OP>, threads, 0));
    const int grid = sms * per_sm * 4;
    probe<OP><<<grid, threads>>>(tab, nrows, iters, sink);
    CK(cudaDeviceSynchronize());
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaEventRecord(a);
    const int reps = 5;
    for (int r = 0; r < reps; ++r) probe<OP><<<grid, threads>>>(tab, nrows, iters, sink);
    cudaEventRecord(b);
    CK(cudaEventSynchronize(b));
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    const double rows = (double)reps * grid * threads * iters * 8;
    printf("%-30s table %6zu KB  threads %3d x %d/SM: %7.1f G rows/s  %6.2f SM-cycles per warp instr\n",
           kOpName[OP], tb >> 10, threads, per_sm, rows / (ms * 1e-3) / 1e9,
           (double)sms * 1.92e9 * (ms * 1e-3) / (rows / 32.0));
  }
  return 0;
}

int main() {
  int sms = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  unsigned long long* sink;
  CK(cudaMalloc(&sink, 8));
  for (size_t tb : {(size_t)2560 << 10, (size_t)16 << 20, (size_t)64 << 10}) {
    unsigned long long* tab;
    CK(cudaMalloc(&tab, tb));
    CK(cudaMemset(tab, 1, tb));
    int rc = run<0>(tab, tb, sms, sink) | run<1>(tab, tb, sms, sink) | run<2>(tab, tb, sms, sink) |
             run<3>(tab, tb, sms, sink) | run<4>(tab, tb, sms, sink) | run<5>(tab, tb, sms, sink) |
             run<6>(tab, tb, sms, sink);
    if (rc) return rc;
    CK(cudaFree(tab));
  }
  return 0;
}
