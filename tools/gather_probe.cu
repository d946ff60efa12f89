// Micro-benchmark (tuning aid, not product): random row gathers from an
// L2-resident table (the rank directories of cfg4 / cfg5 N+1 = 2^20+1) by
// the three engines sm_100a offers:
//   ldg8 / ldg16  ld.global.nc of an 8-B / 16-B row per lane (LSU, L1TEX)
//   bulk16        cp.async.bulk (UBLKCP) of one 16-B row per lane into smem,
//                 completion on an mbarrier (async proxy, no L1TEX t-stage)
//   gather4       cp.async.bulk.tensor.2d ... tile::gather4 (UTMALDG): four
//                 16-B rows per instruction, one instruction per lane
//   mix           half the warps ldg8, half gather4 (do the engines add?)
// Rows/s over the whole GPU, CUDA events.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o gather_probe gather_probe.cu
//   ./gather_probe
#include <cstdio>
#include <cstdint>
#include <cuda.h>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e)); return 1; } } while (0)

__device__ __forceinline__ uint32_t hash(uint32_t x) {
  x ^= x >> 16; x *= 0x7feb352dU; x ^= x >> 15; x *= 0x846ca68bU; x ^= x >> 16;
  return x;
}

__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t n) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"((uint32_t)__cvta_generic_to_shared(b)), "r"(n));
}
__device__ __forceinline__ void mbar_expect(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"((uint32_t)__cvta_generic_to_shared(b)),
               "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tW: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t@!p bra W;\n\t}" ::"r"(
          (uint32_t)__cvta_generic_to_shared(b)),
      "r"(parity) : "memory");
}
__device__ __forceinline__ void bulk16(void* dst, const void* src, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], 16, [%2];" ::"r"(
                   (uint32_t)__cvta_generic_to_shared(dst)),
               "l"(src), "r"((uint32_t)__cvta_generic_to_shared(bar)) : "memory");
}
__device__ __forceinline__ void gather4(void* dst, const CUtensorMap* tm, uint32_t r0, uint32_t r1, uint32_t r2,
                                        uint32_t r3, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, "
      "%5, %6, %7}], [%2];" ::"r"((uint32_t)__cvta_generic_to_shared(dst)),
      "l"(tm), "r"((uint32_t)__cvta_generic_to_shared(bar)), "r"(0), "r"(r0), "r"(r1), "r"(r2), "r"(r3)
      : "memory");
}

constexpr int STAGES = 3;
constexpr int ROWS_PER_LANE = 4;  // rows per lane per stage
constexpr int WARP_STAGE_BYTES = 32 * 128;  // gather4 destinations 128-B aligned: one 128-B slot per lane

// mode 0 ldg8, 1 ldg16, 2 bulk16, 3 gather4, 4 mix (even warps ldg8, odd gather4)
template <int MODE>
__global__ void probe(const uint4* __restrict__ tab, uint32_t nrows, int iters, const __grid_constant__ CUtensorMap tm,
                      unsigned long long* sink) {
  extern __shared__ __align__(128) unsigned char smem[];
  const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t nwarps = blockDim.x >> 5;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem);  // [nwarps][STAGES]
  unsigned char* buf = smem + ((nwarps * STAGES * 8 + 127) & ~127u) + warp * STAGES * WARP_STAGE_BYTES;
  uint64_t* mb = bars + warp * STAGES;
  if (lane == 0)
    for (int s = 0; s < STAGES; ++s) mbar_init(mb + s, 1);
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  __syncthreads();
  uint32_t st = hash(blockIdx.x * blockDim.x + threadIdx.x + 77);
  uint32_t acc = 0;
  const bool use_ldg = MODE == 0 || MODE == 1 || (MODE == 4 && (warp & 1) == 0);
  if (use_ldg) {
    for (int it = 0; it < iters; ++it) {
      if (MODE == 1) {
        uint4 v[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) { st = hash(st + u); v[u] = __ldg(tab + st % nrows); }
#pragma unroll
        for (int u = 0; u < 8; ++u) acc += v[u].x ^ v[u].w;
      } else {
        const uint2* t2 = reinterpret_cast<const uint2*>(tab);
        uint2 v[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) { st = hash(st + u); v[u] = __ldg(t2 + st % (2 * nrows)); }
#pragma unroll
        for (int u = 0; u < 8; ++u) acc += v[u].x ^ v[u].y;
      }
    }
    // same number of rows as the async modes: iters * 8 per lane; caller accounts
  } else {
    // async: a ring of STAGES stages per warp, each 32 lanes x 4 rows x 16 B
    const int nst = iters * 8 / ROWS_PER_LANE;  // same rows per lane as the ldg modes
    auto issue = [&](int s) {
      unsigned char* dst = buf + (s % STAGES) * WARP_STAGE_BYTES;
      if (lane == 0) mbar_expect(mb + (s % STAGES), 32 * ROWS_PER_LANE * 16);
      __syncwarp();
      uint32_t r[ROWS_PER_LANE];
#pragma unroll
      for (int u = 0; u < ROWS_PER_LANE; ++u) { st = hash(st + u); r[u] = st % nrows; }
      if (MODE == 2) {
#pragma unroll
        for (int u = 0; u < ROWS_PER_LANE; ++u) bulk16(dst + lane * 128 + u * 16, tab + r[u], mb + (s % STAGES));
      } else {
        gather4(dst + lane * 128, &tm, r[0], r[1], r[2], r[3], mb + (s % STAGES));
      }
    };
    for (int s = 0; s < STAGES - 1 && s < nst; ++s) issue(s);
    for (int s = 0; s < nst; ++s) {
      if (s + STAGES - 1 < nst) issue(s + STAGES - 1);
      mbar_wait(mb + (s % STAGES), (s / STAGES) & 1);
      const uint4* p = reinterpret_cast<const uint4*>(buf + (s % STAGES) * WARP_STAGE_BYTES + lane * 128);
#pragma unroll
      for (int u = 0; u < ROWS_PER_LANE; ++u) { uint4 v = p[u]; acc += v.x ^ v.w; }
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      __syncwarp();
    }
  }
  if (acc == 0x12345678u) sink[0] = acc;
}

typedef CUresult (*EncodeTiled)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int main() {
  int sms = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q));
  EncodeTiled enc = (EncodeTiled)fn;
  unsigned long long* sink;
  CK(cudaMalloc(&sink, 8));
  const size_t table_bytes[] = {1792u << 10, 2560u << 10, 5u << 20};
  for (size_t tb : table_bytes) {
    const uint32_t nrows = (uint32_t)(tb / 16);
    uint4* tab;
    CK(cudaMalloc(&tab, tb));
    CK(cudaMemset(tab, 1, tb));
    CUtensorMap tm;
    cuuint64_t dims[2] = {4, nrows};
    cuuint64_t strides[1] = {16};
    cuuint32_t box[2] = {4, 1};
    cuuint32_t es[2] = {1, 1};
    CUresult cr = enc(&tm, CU_TENSOR_MAP_DATA_TYPE_UINT32, 2, tab, dims, strides, box, es,
                      CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                      CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (cr != CUDA_SUCCESS) { printf("encode failed %d\n", (int)cr); return 1; }
    const char* names[] = {"ldg8", "ldg16", "bulk16", "gather4", "mix"};
    for (int threads : {256, 512}) {
      for (int mode = 0; mode < 5; ++mode) {
        const int iters = 64;
        const int nwarps = threads / 32;
        const size_t smem = ((nwarps * STAGES * 8 + 127) & ~127) + (size_t)nwarps * STAGES * WARP_STAGE_BYTES;
        int ctas_per_sm = 1;
        void (*k)(const uint4*, uint32_t, int, const CUtensorMap, unsigned long long*) =
            mode == 0 ? probe<0> : mode == 1 ? probe<1> : mode == 2 ? probe<2> : mode == 3 ? probe<3> : probe<4>;
        CK(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&ctas_per_sm, k, threads, smem));
        const int grid = sms * ctas_per_sm * 8;
        for (int w = 0; w < 2; ++w) k<<<grid, threads, smem>>>(tab, nrows, iters, tm, sink);
        CK(cudaDeviceSynchronize());
        cudaEvent_t a, b;
        cudaEventCreate(&a);
        cudaEventCreate(&b);
        cudaEventRecord(a);
        const int reps = 5;
        for (int rr = 0; rr < reps; ++rr) k<<<grid, threads, smem>>>(tab, nrows, iters, tm, sink);
        cudaEventRecord(b);
        CK(cudaEventSynchronize(b));
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        const double rows = (double)reps * grid * threads * iters * 8;
        printf("%-8s table %5zu KB threads %4d ctas/sm %d: %7.1f Grows/s  (%.1f GB/s of row bytes)\n", names[mode],
               tb >> 10, threads, ctas_per_sm, rows / (ms * 1e-3) / 1e9,
               rows * (mode == 0 ? 8 : mode == 4 ? 12 : 16) / (ms * 1e-3) / 1e9);
      }
    }
    CK(cudaFree(tab));
  }
  return 0;
}
