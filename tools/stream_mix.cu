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
  run_tiles<3, 1>(n, 1024, 4);
  run_tiles<3, 1>(n, 1024, 16);
  run_tiles<3, 1>(n, 1024, 64);
  run_tiles<2, 1>(n, 1024, 16);
  run_tiles<2, 1>(n, 1024, 64);
  run_tiles<3, 0>(n, 1024, 16);
  run_tiles<2, 1>(n, 512, 32);
  run_tiles<2, 1>(n, 512, 128);
  run_tiles<2, 1>(n, 256, 64);
  run_tiles<2, 1>(n, 256, 256);
  return 0;
}
