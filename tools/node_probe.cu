// Micro-benchmark (tuning aid, not product): random node gathers from an
// L2-resident table (bitset2's padded array below the shared-memory levels:
// 2^21 f64 = 16 MB at cfg5 N+1 = 2^20 + 1), node = G lanes x B bytes:
//   G = 1   each lane gathers its own B-byte row (B = 8 .. 128; B >= 32 as
//           ld.global.nc.v4.u64 pieces of one line)
//   G > 1   G lanes cooperate on one G*B-byte node (consecutive B-byte
//           pieces), so one warp instruction touches 32 / G nodes
// Nodes/s and node bytes/s over the whole GPU, CUDA events.  This is the
// L1TEX cost model behind the bitset2 deep-level layout (profiles/r02/).
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o node_probe node_probe.cu && ./node_probe
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e)); return 1; } } while (0)

__device__ __forceinline__ uint32_t hash(uint32_t x) {
  x ^= x >> 16; x *= 0x7feb352dU; x ^= x >> 15; x *= 0x846ca68bU; x ^= x >> 16;
  return x;
}

template <int B>
struct Piece { unsigned long long v[B / 8]; };

template <int B>
__device__ __forceinline__ Piece<B> ld(const char* p) {
  Piece<B> r;
  if constexpr (B == 8) {
    asm volatile("ld.global.nc.u64 %0, [%1];" : "=l"(r.v[0]) : "l"(p));
  } else if constexpr (B == 16) {
    asm volatile("ld.global.nc.v2.u64 {%0, %1}, [%2];" : "=l"(r.v[0]), "=l"(r.v[1]) : "l"(p));
  } else {
#pragma unroll
    for (int k = 0; k < B / 32; ++k)
      asm volatile("ld.global.nc.v4.u64 {%0, %1, %2, %3}, [%4];"
                   : "=l"(r.v[4 * k]), "=l"(r.v[4 * k + 1]), "=l"(r.v[4 * k + 2]), "=l"(r.v[4 * k + 3])
                   : "l"(p + 32 * k));
  }
  return r;
}

template <int B, int G>
__global__ void probe(const char* __restrict__ tab, uint32_t nnodes, int iters, unsigned long long* sink) {
  constexpr int U = B >= 64 ? 4 : 8;  // loads in flight per lane
  const uint32_t lane = threadIdx.x & 31;
  const uint32_t grp = (blockIdx.x * blockDim.x + threadIdx.x) / G;  // lanes of a group share the node
  uint32_t st = hash(grp * 7919u + 77u);
  unsigned long long acc = 0;
  for (int it = 0; it < iters; ++it) {
    Piece<B> v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      st = hash(st + u);
      const uint64_t node = st % nnodes;
      v[u] = ld<B>(tab + node * (uint64_t)(G * B) + (lane % G) * B);
    }
#pragma unroll
    for (int u = 0; u < U; ++u)
#pragma unroll
      for (int k = 0; k < B / 8; ++k) acc ^= v[u].v[k];
  }
  if (acc == 0x1234567890ull) sink[0] = acc;
}

template <int B, int G>
int run(const char* tab, size_t tb, int sms, unsigned long long* sink) {
  constexpr int U = B >= 64 ? 4 : 8;
  const uint32_t nnodes = (uint32_t)(tb / (G * B));
  const int iters = 64 * 8 / U;
  for (int threads : {256, 512}) {
    int per_sm = 0;
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, probe<B, G>, threads, 0));
    const int grid = sms * per_sm * 4;
    probe<B, G><<<grid, threads>>>(tab, nnodes, iters, sink);
    CK(cudaDeviceSynchronize());
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaEventRecord(a);
    const int reps = 5;
    for (int r = 0; r < reps; ++r) probe<B, G><<<grid, threads>>>(tab, nnodes, iters, sink);
    cudaEventRecord(b);
    CK(cudaEventSynchronize(b));
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    const double lane_loads = (double)reps * grid * threads * iters * U;
    const double nodes = lane_loads / G;
    printf("B=%3d G=%2d node=%4d B  table %5zu KB  threads %3d x %d/SM: %7.1f Gnodes/s  %7.1f GB/s  "
           "%6.2f SM-cycles per warp instr\n",
           B, G, B * G, tb >> 10, threads, per_sm, nodes / (ms * 1e-3) / 1e9, nodes * G * B / (ms * 1e-3) / 1e9,
           (double)sms * 1.92e9 * (ms * 1e-3) / (lane_loads / 32.0 * (B >= 32 ? B / 32 : 1)));
  }
  return 0;
}

int main() {
  int sms = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  unsigned long long* sink;
  CK(cudaMalloc(&sink, 8));
  for (size_t tb : {(size_t)16 << 20, (size_t)2 << 20}) {
    char* tab;
    CK(cudaMalloc(&tab, tb));
    CK(cudaMemset(tab, 1, tb));
    int rc = run<8, 1>(tab, tb, sms, sink) | run<16, 1>(tab, tb, sms, sink) | run<32, 1>(tab, tb, sms, sink) |
             run<64, 1>(tab, tb, sms, sink) | run<128, 1>(tab, tb, sms, sink) | run<8, 4>(tab, tb, sms, sink) |
             run<8, 8>(tab, tb, sms, sink) | run<8, 16>(tab, tb, sms, sink) | run<16, 8>(tab, tb, sms, sink) |
             run<32, 4>(tab, tb, sms, sink) | run<16, 4>(tab, tb, sms, sink) | run<32, 2>(tab, tb, sms, sink);
    if (rc) return rc;
    CK(cudaFree(tab));
  }
  return 0;
}
