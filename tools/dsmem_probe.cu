// Micro-benchmark (tuning aid, not product): random 8-byte gathers from a
// table distributed over a thread-block cluster's shared memory (DSMEM,
// mapa + ld.shared::cluster) vs the same gathers from global memory (L2),
// at the table sizes of cfg4 / cfg5's rank directories.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o dsmem_probe dsmem_probe.cu
//   ./dsmem_probe
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e)); return 1; } } while (0)

__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;\n" ::: "memory");
}
__device__ __forceinline__ uint2 ld_dsmem(const void* local_generic, uint32_t cta) {
  uint32_t a = (uint32_t)__cvta_generic_to_shared(local_generic), ra;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(a), "r"(cta));
  uint2 v;
  asm volatile("ld.shared::cluster.v2.u32 {%0, %1}, [%2];" : "=r"(v.x), "=r"(v.y) : "r"(ra));
  return v;
}

__device__ __forceinline__ uint32_t hash(uint32_t x) {
  x ^= x >> 16; x *= 0x7feb352dU; x ^= x >> 15; x *= 0x846ca68bU; x ^= x >> 16;
  return x;
}

// Each CTA owns words [rank*wpc, (rank+1)*wpc); every thread issues `iters`
// rounds of UNR independent random gathers over the whole cluster table.
template <int UNR>
__global__ void dsmem_gather(uint32_t words_per_cta, uint32_t csize, int iters, unsigned long long* sink) {
  extern __shared__ uint2 tab[];
  const uint32_t me = cluster_rank();
  for (uint32_t i = threadIdx.x; i < words_per_cta; i += blockDim.x) tab[i] = make_uint2(me * words_per_cta + i, i);
  cluster_sync();
  const uint32_t total = words_per_cta * csize;
  uint32_t s = hash(blockIdx.x * blockDim.x + threadIdx.x + 12345);
  uint32_t acc = 0;
  for (int it = 0; it < iters; ++it) {
    uint2 v[UNR];
#pragma unroll
    for (int u = 0; u < UNR; ++u) {
      s = hash(s + u);
      const uint32_t w = s % total;
      const uint32_t cta = w / words_per_cta, off = w - cta * words_per_cta;
      v[u] = ld_dsmem(tab + off, cta);
    }
#pragma unroll
    for (int u = 0; u < UNR; ++u) acc += v[u].x ^ v[u].y;
  }
  cluster_sync();  // peers must not exit while their smem is read
  if (acc == 0x12345678u) sink[0] = acc;
}

template <int UNR>
__global__ void global_gather(const uint2* __restrict__ tab, uint32_t total, int iters, unsigned long long* sink) {
  uint32_t s = hash(blockIdx.x * blockDim.x + threadIdx.x + 12345);
  uint32_t acc = 0;
  for (int it = 0; it < iters; ++it) {
    uint2 v[UNR];
#pragma unroll
    for (int u = 0; u < UNR; ++u) {
      s = hash(s + u);
      v[u] = __ldg(tab + s % total);
    }
#pragma unroll
    for (int u = 0; u < UNR; ++u) acc += v[u].x ^ v[u].y;
  }
  if (acc == 0x12345678u) sink[0] = acc;
}

int main() {
  int sms = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  unsigned long long* sink;
  CK(cudaMalloc(&sink, 8));
  cudaEvent_t a, b;
  CK(cudaEventCreate(&a));
  CK(cudaEventCreate(&b));
  const int iters = 64, UNR = 8;
  const uint32_t table_bytes[] = {1u << 20, 1792u << 10};
  for (uint32_t tb : table_bytes) {
    for (int csize : {2, 4, 8, 16}) {
      for (int threads : {512, 1024}) {
        const uint32_t wpc = (tb / 8 + csize - 1) / csize;
        const size_t smem = (size_t)wpc * 8;
        if (smem > 227 * 1024) continue;
        auto k = dsmem_gather<UNR>;
        CK(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        if (csize > 8) CK(cudaFuncSetAttribute(k, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
        cudaLaunchConfig_t cfg = {};
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeClusterDimension;
        attr[0].val.clusterDim.x = csize;
        attr[0].val.clusterDim.y = 1;
        attr[0].val.clusterDim.z = 1;
        cfg.blockDim = dim3(threads);
        cfg.dynamicSmemBytes = smem;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
        int nclusters = 0;
        cfg.gridDim = dim3(csize);
        if (cudaOccupancyMaxActiveClusters(&nclusters, k, &cfg) != cudaSuccess || nclusters == 0) {
          cudaGetLastError();
          printf("dsmem table %u KB cluster %d threads %d: no fit\n", tb >> 10, csize, threads);
          continue;
        }
        cfg.gridDim = dim3(nclusters * csize);
        for (int rep = 0; rep < 2; ++rep) {
          CK(cudaEventRecord(a));
          CK(cudaLaunchKernelEx(&cfg, k, wpc, (uint32_t)csize, iters, sink));
          CK(cudaEventRecord(b));
          CK(cudaEventSynchronize(b));
        }
        float ms;
        CK(cudaEventElapsedTime(&ms, a, b));
        const double g = (double)nclusters * csize * threads * iters * UNR;
        printf("dsmem  table %5u KB cluster %2d threads %4d ctas %3d: %.1f Ggather/s\n", tb >> 10, csize, threads,
               nclusters * csize, g / (ms * 1e6));
      }
    }
    uint2* gt;
    CK(cudaMalloc(&gt, tb));
    CK(cudaMemset(gt, 1, tb));
    for (int threads : {512, 1024}) {
      const int ctas = sms * (2048 / threads);
      for (int rep = 0; rep < 2; ++rep) {
        CK(cudaEventRecord(a));
        global_gather<UNR><<<ctas, threads>>>(gt, tb / 8, iters, sink);
        CK(cudaEventRecord(b));
        CK(cudaEventSynchronize(b));
      }
      float ms;
      CK(cudaEventElapsedTime(&ms, a, b));
      const double g = (double)ctas * threads * iters * UNR;
      printf("global table %5u KB            threads %4d ctas %3d: %.1f Ggather/s\n", tb >> 10, threads, ctas,
             g / (ms * 1e6));
    }
    CK(cudaFree(gt));
  }
  return 0;
}
