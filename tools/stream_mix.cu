// Tuning aid (not product): HBM throughput of a pure stream kernel with the
// read:write byte mix of each search-kernel shape -- 4->4 (f32 queries,
// int32 out), 4->8, 8->4, 8->8 -- using the search kernel's access pattern
// (grid-stride, 16-B nc loads, 16-B streaming stores, 3 groups in flight).
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o stream_mix stream_mix.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

template <typename In, typename Out>
__global__ void __launch_bounds__(1024, 1) stream(const In* __restrict__ z, Out* __restrict__ o, uint64_t n4) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t g0 = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; g0 < n4; g0 += 3 * stride) {
    In v[3][4];
#pragma unroll
    for (int u = 0; u < 3; ++u) {
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
    for (int u = 0; u < 3; ++u) {
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

template <typename In, typename Out>
void run(const char* name, uint64_t n) {
  In* z;
  Out* o;
  cudaMalloc(&z, n * sizeof(In));
  cudaMalloc(&o, n * sizeof(Out));
  cudaMemset(z, 0, n * sizeof(In));
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (int i = 0; i < 3; ++i) stream<In, Out><<<sms, 1024>>>(z, o, n / 4);
  cudaEventRecord(a);
  for (int i = 0; i < 10; ++i) stream<In, Out><<<sms, 1024>>>(z, o, n / 4);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  const double bytes = (double)n * (sizeof(In) + sizeof(Out));
  printf("%s: %.1f GB/s (%.1f G elements/s) %s\n", name, bytes / (ms / 10 * 1e-3) / 1e9, n / (ms / 10 * 1e-3) / 1e9,
         cudaGetErrorString(cudaGetLastError()));
  cudaFree(z);
  cudaFree(o);
}

int main() {
  run<float, int32_t>("f32 -> int32 (1:1)", 1ull << 30);
  run<float, int64_t>("f32 -> int64 (1:2)", 1ull << 30);
  run<double, int32_t>("f64 -> int32 (2:1)", 1ull << 29);
  run<double, int64_t>("f64 -> int64 (1:1)", 1ull << 29);
  return 0;
}
