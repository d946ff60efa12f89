// Micro-benchmark (tuning aid, not product): query exchange over a thread-
// block cluster's shared memory.  The rank directory of a table too large
// for one SM's shared memory (cfg5 N+1 = 2^20+1: 2.5 MB) is split over the
// C CTAs of a cluster; every CTA routes each of its queries to the CTA that
// owns the query's slice (bulk copies shared::cta -> shared::cluster, the
// receiver's mbarrier counting the bytes), the owner resolves it with one
// shared-memory gather and bulk-copies the answers back.  This measures the
// exchange engine alone (queries generated in registers, no HBM stream) to
// see whether it beats ~290 G random L2 gathers/s.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o cluster_exchange_probe cluster_exchange_probe.cu
//   ./cluster_exchange_probe
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

#define CK(x)                                                                              \
  do {                                                                                     \
    cudaError_t e = (x);                                                                   \
    if (e != cudaSuccess) {                                                                \
      printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e));                     \
      return 1;                                                                            \
    }                                                                                      \
  } while (0)

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;\n" ::: "memory");
}
__device__ __forceinline__ uint32_t mapa(uint32_t a, uint32_t cta) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(cta));
  return r;
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_remote_arrive_tx(uint32_t rbar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.release.cluster.shared::cluster.b64 _, [%0], %1;" ::"r"(rbar), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "W:\n\t"
      "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra W;\n\t}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void bulk_s2c(uint32_t rdst, uint32_t src, uint32_t bytes, uint32_t rbar) {
  asm volatile("cp.async.bulk.shared::cluster.shared::cta.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   rdst),
               "r"(src), "r"(bytes), "r"(rbar)
               : "memory");
}
__device__ __forceinline__ uint32_t hash(uint32_t x) {
  x ^= x >> 16;
  x *= 0x7feb352dU;
  x ^= x >> 15;
  x *= 0x846ca68bU;
  x ^= x >> 16;
  return x;
}

// smem: table slice [tab_words uint2] | per stage: send[T] u32, inbox[T] u32 | barriers
// Each CTA sends T/C entries to every peer per round (equal segments: the
// probe measures the engine; real segments vary).  Software-pipelined over S
// stages: iteration r sends round r, serves round r - 1 and collects the
// answers of round r - 2, so each exchange latency has a whole iteration.
template <int Q, int S>
__global__ void exchange(uint32_t C, uint32_t T, uint32_t tab_words, int rounds, unsigned long long* sink) {
  extern __shared__ __align__(128) unsigned char smem[];
  uint2* tab = reinterpret_cast<uint2*>(smem);
  uint32_t* send = reinterpret_cast<uint32_t*>(smem + (size_t)tab_words * 8);  // [S][T]
  uint32_t* inbox = send + S * T;                                               // [S][T]
  uint64_t* bars = reinterpret_cast<uint64_t*>(inbox + S * T);                  // full[S], back[S]
  const uint32_t me = cluster_rank();
  const uint32_t seg = T / C, segb = seg * 4;
  for (uint32_t i = threadIdx.x; i < tab_words; i += blockDim.x) tab[i] = make_uint2(hash(i), me * tab_words + i);
  if (threadIdx.x == 0) {
    for (int b = 0; b < 2 * S; ++b) mbar_init(bars + b, C);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  cluster_sync();
  uint32_t s0 = hash(blockIdx.x * blockDim.x + threadIdx.x);
  uint32_t acc = 0;
  for (int r = 0; r < rounds + 2; ++r) {
    if (r < rounds) {
      const uint32_t st = r % S;
      uint32_t* sb = send + st * T;
#pragma unroll
      for (int q = 0; q < Q; ++q) {
        const uint32_t pos = q * blockDim.x + threadIdx.x;
        s0 = hash(s0 + q);
        sb[pos] = s0 % tab_words;
      }
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      __syncthreads();
      if (threadIdx.x < C) {
        const uint32_t d = threadIdx.x;
        const uint32_t rbar = mapa(smem_u32(bars + st), d);
        mbar_remote_arrive_tx(rbar, segb);
        bulk_s2c(mapa(smem_u32(inbox + st * T + me * seg), d), smem_u32(sb + d * seg), segb, rbar);
      }
    }
    if (r >= 1 && r - 1 < rounds) {  // serve round r - 1 and reply in place
      const int rr = r - 1;
      const uint32_t st = rr % S;
      mbar_wait(bars + st, (rr / S) & 1);
      uint32_t* ib = inbox + st * T;
      for (uint32_t i = threadIdx.x; i < T; i += blockDim.x) {
        const uint32_t w = ib[i];
        const uint2 d = tab[w];
        ib[i] = d.y + __popc(d.x & w);
      }
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      __syncthreads();
      if (threadIdx.x < C) {
        const uint32_t c = threadIdx.x;
        const uint32_t rbar = mapa(smem_u32(bars + S + st), c);
        mbar_remote_arrive_tx(rbar, segb);
        bulk_s2c(mapa(smem_u32(send + st * T + me * seg), c), smem_u32(ib + c * seg), segb, rbar);
      }
    }
    if (r >= 2) {  // answers of round r - 2
      const int rr = r - 2;
      const uint32_t ps = rr % S;
      mbar_wait(bars + S + ps, (rr / S) & 1);
      const uint32_t* sb = send + ps * T;
#pragma unroll
      for (int q = 0; q < Q; ++q) acc += sb[q * blockDim.x + threadIdx.x];
    }
  }
  cluster_sync();
  if (acc == 0x12345678u) sink[0] = acc;
}

template <int Q, int S>
int run(uint32_t C, uint32_t threads, uint32_t tab_bytes, int rounds, unsigned long long* sink, cudaEvent_t a,
        cudaEvent_t b) {
  const uint32_t T = threads * Q;
  const size_t smem = tab_bytes + (size_t)8 * S * T + 16 * S;
  if (smem > 227 * 1024) return 0;
  auto k = exchange<Q, S>;
  CK(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  if (C > 8) CK(cudaFuncSetAttribute(k, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
  cudaLaunchConfig_t cfg = {};
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = C;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.blockDim = dim3(threads);
  cfg.dynamicSmemBytes = smem;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cfg.gridDim = dim3(C);
  int ncl = 0;
  if (cudaOccupancyMaxActiveClusters(&ncl, k, &cfg) != cudaSuccess || ncl == 0) {
    cudaGetLastError();
    printf("C=%u threads=%u Q=%d S=%d: no fit\n", C, threads, Q, S);
    return 0;
  }
  cfg.gridDim = dim3(ncl * C);
  float ms = 0;
  for (int rep = 0; rep < 2; ++rep) {
    CK(cudaEventRecord(a));
    CK(cudaLaunchKernelEx(&cfg, k, C, T, tab_bytes / 8, rounds, sink));
    CK(cudaEventRecord(b));
    CK(cudaEventSynchronize(b));
    CK(cudaGetLastError());
    CK(cudaEventElapsedTime(&ms, a, b));
  }
  const double qs = (double)ncl * C * T * rounds / (ms * 1e-3);
  const double cyc = ms * 1e-3 * 1.965e9 / rounds;
  printf("C=%2u S=%d table=%3u KB SMs=%3u threads=%4u T=%5u: %7.1f G queries/s  (%.0f cycles/round, %.3f cycles/query/SM)\n",
         C, S, tab_bytes >> 10, ncl * C, threads, T, qs / 1e9, cyc, cyc / T);
  return 0;
}

int main() {
  unsigned long long* sink;
  CK(cudaMalloc(&sink, 8));
  cudaEvent_t a, b;
  CK(cudaEventCreate(&a));
  CK(cudaEventCreate(&b));
  const int rounds = 2000;
  for (uint32_t C : {4u, 8u, 16u}) {
    for (uint32_t tab_kb : {96u, 160u}) {
      for (uint32_t threads : {512u, 1024u}) {
        run<2, 3>(C, threads, tab_kb << 10, rounds, sink, a, b);
        run<4, 3>(C, threads, tab_kb << 10, rounds, sink, a, b);
        run<2, 4>(C, threads, tab_kb << 10, rounds, sink, a, b);
        run<4, 4>(C, threads, tab_kb << 10, rounds, sink, a, b);
        run<8, 3>(C, threads, tab_kb << 10, rounds, sink, a, b);
      }
    }
  }
  return 0;
}
