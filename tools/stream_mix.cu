// Tuning aid (not product): HBM throughput of a pure stream kernel with the
// read:write byte mix of each search-kernel shape -- 4->4 (f32 queries,
// int32 out), 4->8, 8->4, 8->8 -- using the search kernel's access pattern
// (grid-stride, 16-B nc loads, 16-B streaming stores, 3 groups in flight).
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o stream_mix stream_mix.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

template <typename In, typename Out, int U>
__global__ void stream(const In* __restrict__ z, Out* __restrict__ o, uint64_t n4) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t g0 = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; g0 < n4; g0 += U * stride) {
    In v[U][4];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const uint64_t g = g0 + u * stride;
      if (g < n4) {
        if constexpr (sizeof(In) == 4) {
          const float4 t = __ldg(reinterpret_cast<const float4*>(z) + g);
          v[u][0] = t.x, v[u][1] = t.y, v[u][2] = t.z, v[u][3] = t.w;
        } else {
          const double2 a = __ldg(reinterpret_cast<const double2*>(z) + 2 * g);
          const double2 b = __ldg(reinterpret_cast<const double2*>(z) + 2 * g + 1);
          v[u][0] = a.x, v[u][1] = a.y, v[u][2] = b.x, v[u][3] = b.y;
        }
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const uint64_t g = g0 + u * stride;
      if (g < n4) {
        if constexpr (sizeof(Out) == 4) {
          __stcs(reinterpret_cast<int4*>(o) + g, make_int4((int)v[u][0], (int)v[u][1], (int)v[u][2], (int)v[u][3]));
        } else {
          __stcs(reinterpret_cast<longlong2*>(o) + 2 * g, make_longlong2((long long)v[u][0], (long long)v[u][1]));
          __stcs(reinterpret_cast<longlong2*>(o) + 2 * g + 1, make_longlong2((long long)v[u][2], (long long)v[u][3]));
        }
      }
    }
  }
}


// Persistent CTAs over contiguous tiles: tile = blockDim * U groups; CTA b
// takes tiles b, b + grid, ... (TILES_PER_CTA = 0) or one contiguous span of
// tiles (TILES_PER_CTA = 1).
template <typename In, typename Out, int U, int CONTIG>
__global__ void stream_tiles(const In* __restrict__ z, Out* __restrict__ o, uint64_t n4) {
  const uint64_t tile = (uint64_t)blockDim.x * U;
  const uint64_t ntiles = (n4 + tile - 1) / tile;
  uint64_t t0, t1, step;
  if (CONTIG) {
    const uint64_t per = (ntiles + gridDim.x - 1) / gridDim.x;
    t0 = blockIdx.x * per;
    t1 = t0 + per < ntiles ? t0 + per : ntiles;
    step = 1;
  } else {
    t0 = blockIdx.x;
    t1 = ntiles;
    step = gridDim.x;
  }
  for (uint64_t t = t0; t < t1; t += step) {
    const uint64_t g0 = t * tile + threadIdx.x;
    float4 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const uint64_t g = g0 + (uint64_t)u * blockDim.x;
      if (g < n4) v[u] = __ldg(reinterpret_cast<const float4*>(z) + g);
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const uint64_t g = g0 + (uint64_t)u * blockDim.x;
      if (g < n4) __stcs(reinterpret_cast<int4*>(o) + g, make_int4((int)v[u].x, (int)v[u].y, (int)v[u].z, (int)v[u].w));
    }
  }
}

template <int U, int CONTIG>
void run_tiles(uint64_t n, int threads, int ctas_per_sm) {
  float* z;
  int32_t* o;
  cudaMalloc(&z, n * 4);
  cudaMalloc(&o, n * 4);
  cudaMemset(z, 0, n * 4);
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (int i = 0; i < 3; ++i) stream_tiles<float, int32_t, U, CONTIG><<<sms * ctas_per_sm, threads>>>(z, o, n / 4);
  cudaEventRecord(a);
  for (int i = 0; i < 10; ++i) stream_tiles<float, int32_t, U, CONTIG><<<sms * ctas_per_sm, threads>>>(z, o, n / 4);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  printf("f32->i32 tiles U=%d threads=%d ctas/SM=%d %s: %.1f GB/s (%.1f G elements/s)\n", U, threads, ctas_per_sm,
         CONTIG ? "contiguous span" : "round-robin tiles", 8.0 * n / (ms / 10 * 1e-3) / 1e9, n / (ms / 10 * 1e-3) / 1e9);
  cudaFree(z);
  cudaFree(o);
}


// Persistent CTAs streaming through a shared-memory ring with the bulk-copy
// engine: thread 0 issues cp.async.bulk loads of CHUNK-byte query chunks
// (mbarrier complete_tx), all threads convert smem -> smem, thread 0 issues
// cp.async.bulk stores of the result chunk (bulk_group), STAGES deep.
__device__ __forceinline__ uint32_t sa(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
template <int STAGES, int CHUNK, int STORE_TMA>
__global__ void stream_tma(const float* __restrict__ z, int32_t* __restrict__ o, uint64_t n) {
  extern __shared__ __align__(128) unsigned char sm[];
  float* in = reinterpret_cast<float*>(sm);
  int32_t* ob = reinterpret_cast<int32_t*>(sm + STAGES * CHUNK);
  __shared__ __align__(8) uint64_t full[STAGES];
  constexpr uint32_t E = CHUNK / 4;  // elements per chunk
  const uint64_t nch = n / E;        // whole chunks only (n multiple of E here)
  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa(&full[s])));
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  auto issue = [&](uint64_t c, int s) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(&full[s])), "r"((uint32_t)CHUNK) : "memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(sa(in + s * E)),
                 "l"(z + c * E), "r"((uint32_t)CHUNK), "r"(sa(&full[s])) : "memory");
  };
  uint64_t c = blockIdx.x;
  if (threadIdx.x == 0)
    for (int s = 0; s < STAGES; ++s)
      if (c + (uint64_t)s * gridDim.x < nch) issue(c + (uint64_t)s * gridDim.x, s);
  uint32_t phase = 0;
  for (uint64_t it = 0; c < nch; ++it, c += gridDim.x) {
    const int s = (int)(it % STAGES);
    // wait for chunk c in stage s
    asm volatile("{\n\t.reg .pred p;\nW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t@!p bra W_%=;\n}" ::"r"(sa(&full[s])), "r"(phase) : "memory");
    const float4* src = reinterpret_cast<const float4*>(in + s * E);
    if (STORE_TMA) {
      // the result buffer of stage s must have been read out by its previous store
      if (threadIdx.x == 0) asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(STAGES - 1) : "memory");
      __syncthreads();
      int4* dst = reinterpret_cast<int4*>(ob + s * E);
      for (uint32_t i = threadIdx.x; i < E / 4; i += blockDim.x) {
        const float4 v = src[i];
        dst[i] = make_int4((int)v.x, (int)v.y, (int)v.z, (int)v.w);
      }
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      __syncthreads();
      if (threadIdx.x == 0) {
        asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(o + c * E), "r"(sa(dst)), "r"((uint32_t)CHUNK) : "memory");
        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
      }
    } else {
      int4* dst = reinterpret_cast<int4*>(o + c * E);
      for (uint32_t i = threadIdx.x; i < E / 4; i += blockDim.x) {
        const float4 v = src[i];
        __stcs(dst + i, make_int4((int)v.x, (int)v.y, (int)v.z, (int)v.w));
      }
      __syncthreads();  // every thread is done reading stage s
    }
    if (threadIdx.x == 0) {
      const uint64_t nx = c + (uint64_t)STAGES * gridDim.x;
      if (nx < nch) issue(nx, s);
    }
    if (s == STAGES - 1) phase ^= 1;
  }
  if (threadIdx.x == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

template <int STAGES, int CHUNK, int STORE_TMA>
void run_tma(uint64_t n, int threads, int ctas_per_sm = 1) {
  float* z;
  int32_t* o;
  cudaMalloc(&z, n * 4);
  cudaMalloc(&o, n * 4);
  cudaMemset(z, 0, n * 4);
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const size_t smem = (STORE_TMA ? 2ull : 1ull) * STAGES * CHUNK;
  auto k = stream_tma<STAGES, CHUNK, STORE_TMA>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (int i = 0; i < 3; ++i) k<<<sms * ctas_per_sm, threads, smem>>>(z, o, n);
  cudaEventRecord(a);
  for (int i = 0; i < 10; ++i) k<<<sms * ctas_per_sm, threads, smem>>>(z, o, n);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  // correctness spot check: o[i] == (int)z[i] == 0
  int32_t h[4] = {1, 1, 1, 1};
  cudaMemcpy(h, o + n - 4, 16, cudaMemcpyDeviceToHost);
  printf("f32->i32 TMA ring stages=%d chunk=%dKB threads=%d ctas/SM=%d store=%s: %.1f GB/s (%.1f G elements/s) %s tail=%d\n", STAGES,
         CHUNK / 1024, threads, ctas_per_sm, STORE_TMA ? "bulk" : "st.cs", 8.0 * n / (ms / 10 * 1e-3) / 1e9, n / (ms / 10 * 1e-3) / 1e9,
         cudaGetErrorString(cudaGetLastError()), h[3]);
  cudaFree(z);
  cudaFree(o);
}

template <typename In, typename Out, int U>
void run(const char* name, uint64_t n, int ctas_per_sm, int threads, bool persistent) {
  In* z;
  Out* o;
  cudaMalloc(&z, n * sizeof(In));
  cudaMalloc(&o, n * sizeof(Out));
  cudaMemset(z, 0, n * sizeof(In));
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const uint64_t grid = persistent ? (uint64_t)sms * ctas_per_sm : (n / 4 + (uint64_t)threads * U - 1) / ((uint64_t)threads * U);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (int i = 0; i < 3; ++i) stream<In, Out, U><<<(unsigned)grid, threads>>>(z, o, n / 4);
  cudaEventRecord(a);
  for (int i = 0; i < 10; ++i) stream<In, Out, U><<<(unsigned)grid, threads>>>(z, o, n / 4);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  const double bytes = (double)n * (sizeof(In) + sizeof(Out));
  printf("%s U=%d threads=%d %s: %.1f GB/s (%.1f G elements/s) %s\n", name, U, threads,
         persistent ? (ctas_per_sm == 1 ? "persistent x1" : "persistent x2") : "full grid",
         bytes / (ms / 10 * 1e-3) / 1e9, n / (ms / 10 * 1e-3) / 1e9, cudaGetErrorString(cudaGetLastError()));
  cudaFree(z);
  cudaFree(o);
}

int main() {
  const uint64_t n = 1ull << 30;
  run<float, int32_t, 3>("f32->i32", n, 1, 1024, true);  // the search kernel's shape (grid-stride)
  run<float, int32_t, 2>("f32->i32", n, 1, 256, false);  // full grid
  run_tma<4, 16384, 1>(n, 256);
  run_tma<3, 16384, 1>(n, 256);
  run_tma<5, 16384, 1>(n, 256);
  run_tma<4, 16384, 1>(n, 512);
  run_tma<4, 16384, 1>(n, 1024);
  run_tma<4, 16384, 0>(n, 256);
  run_tma<6, 16384, 0>(n, 256);
  run_tma<8, 16384, 0>(n, 512);
  run_tma<4, 16384, 0>(n, 1024);
  run_tma<8, 16384, 0>(n, 1024);
  run_tma<2, 16384, 1>(n, 256, 2);
  run_tma<4, 8192, 1>(n, 256, 2);
  return 0;
}
