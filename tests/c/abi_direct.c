/*
 * Standalone C client of libfsgpu.so (include/fsgpu.h): no Python, no torch.
 * Certifies H, builds K, the rank directory and fused records, runs the
 * direct and bitset2 searches on device-resident queries and the end-to-end
 * host path, and checks every answer against a CPU linear scan
 * (max{i : X_i <= z}).  Also checks OutOfDomain positions.  Exit 0 = pass.
 *
 *   gcc -std=c11 -O2 -I include tests/c/abi_direct.c -L paper_1506_08620_b200 -lfsgpu \
 *       -L /usr/local/cuda/lib64 -lcudart -Wl,-rpath,... -o abi_direct
 */
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <cuda_runtime_api.h>

#include "fsgpu.h"

#define CHECK(x)                                                                            \
  do {                                                                                      \
    int rc_ = (x);                                                                          \
    if (rc_) {                                                                              \
      fprintf(stderr, "%s:%d: %s -> %d (%s)\n", __FILE__, __LINE__, #x, rc_, fs_last_error()); \
      return 1;                                                                             \
    }                                                                                       \
  } while (0)
#define CUDA(x)                                                                             \
  do {                                                                                      \
    cudaError_t e_ = (x);                                                                   \
    if (e_ != cudaSuccess) {                                                                \
      fprintf(stderr, "%s:%d: %s -> %s\n", __FILE__, __LINE__, #x, cudaGetErrorString(e_)); \
      return 1;                                                                             \
    }                                                                                       \
  } while (0)

static uint64_t rng = 88172645463325252ull;
static double urand(void) {  /* xorshift64* in [0, 1) */
  rng ^= rng >> 12;
  rng ^= rng << 25;
  rng ^= rng >> 27;
  return (double)((rng * 2685821657736338717ull) >> 11) / 9007199254740992.0;
}

/* max{i <= N-1 : X_i <= z} (partition.py:180-192), by bisection on the host */
static int32_t scan(const float* x, uint64_t n1, float z) {
  uint64_t lo = 0, hi = n1 - 1; /* answer in [lo, hi) */
  while (hi - lo > 1) {
    const uint64_t mid = (lo + hi) / 2;
    if (x[mid] <= z) lo = mid;
    else hi = mid;
  }
  return (int32_t)lo;
}

int main(void) {
  const uint64_t n1 = 4097, m = 1000003;
  float* x = malloc(n1 * sizeof(float));
  double acc = 0.0;
  for (uint64_t i = 0; i < n1; ++i) {
    x[i] = (float)acc;
    acc += 0.5 + urand();
  }
  float* z = malloc(m * sizeof(float));
  for (uint64_t j = 0; j < m; ++j) {
    float v = (float)(urand() * (double)x[n1 - 1]);
    if (v >= x[n1 - 1]) v = nextafterf(x[n1 - 1], 0.0f);
    z[j] = v;
  }
  /* exact knots and their neighbours */
  for (uint64_t i = 0; i + 1 < n1 && i < 1000; ++i) z[i] = x[i];
  for (uint64_t i = 1; i + 1 < n1 && i < 1000; ++i) z[1000 + i] = nextafterf(x[i], 0.0f);

  void *dx, *dws, *dk, *df, *ddir, *drec, *dpad, *dz, *dout, *dst;
  CUDA(cudaMalloc(&dx, n1 * sizeof(float)));
  CUDA(cudaMemcpy(dx, x, n1 * sizeof(float), cudaMemcpyHostToDevice));
  CUDA(cudaMalloc(&dws, fs_workspace_bytes()));

  float h = 0, h0 = 0;
  uint64_t r = 0;
  uint32_t inc = 0;
  int64_t pos = -1;
  CHECK(fs_certify(FS_F32, dx, n1, 32, 1, dws, &h, &h0, &r, &inc, &pos, NULL));
  CUDA(cudaMalloc(&dk, (r + 1) * 4));
  CUDA(cudaMalloc(&df, n1 * 8));
  CHECK(fs_build_table(FS_F32, dx, n1, (double)h, r, 1, dk, df, dws, NULL));
  CUDA(cudaMalloc(&ddir, ((r >> 5) + 1) * 8));
  CHECK(fs_build_rank(FS_F32, dx, n1, (double)h, r, df, ddir, NULL));
  CUDA(cudaMalloc(&drec, (r + 1) * 8));
  CHECK(fs_build_fused(FS_F32, dx, n1, dk, r, drec, NULL));
  int pbits = 0;
  while ((1ull << pbits) <= n1 - 1) ++pbits;
  CUDA(cudaMalloc(&dpad, (1ull << pbits) * sizeof(float)));
  CHECK(fs_build_padded(FS_F32, dx, n1, pbits, dpad, NULL));

  CUDA(cudaMalloc(&dz, m * sizeof(float)));
  CUDA(cudaMalloc(&dout, m * sizeof(int32_t)));
  CUDA(cudaMalloc(&dst, fs_search_ws_words() * 8));
  CUDA(cudaMemset(dst, 0, fs_search_ws_words() * 8));
  CUDA(cudaMemcpy(dz, z, m * sizeof(float), cudaMemcpyHostToDevice));

  int32_t* want = malloc(m * sizeof(int32_t));
  for (uint64_t j = 0; j < m; ++j) want[j] = scan(x, n1, z[j]);
  int32_t* got = malloc(m * sizeof(int32_t));

  fs_plan plan;
  memset(&plan, 0, sizeof(plan));
  plan.dtype = FS_F32;
  plan.n1 = n1;
  plan.x = dx;
  plan.x0 = x[0];
  plan.xn = x[n1 - 1];
  plan.h = h;
  plan.r = r;
  plan.q = 1;
  plan.pbits = pbits;

  const char* names[4] = {"direct/K", "direct/rank+records", "direct-cache", "bitset2"};
  for (int v = 0; v < 4; ++v) {
    plan.algorithm = v <= 1 ? FS_ALGO_DIRECT : (v == 2 ? FS_ALGO_DIRECT_CACHE : FS_ALGO_BITSET2);
    plan.table = v <= 1 ? dk : (v == 2 ? drec : dpad);
    plan.rank = v == 1 ? ddir : NULL;
    plan.records = v == 1 ? drec : NULL;
    CHECK(fs_search_device(&plan, dz, m, dout, 4, (unsigned long long*)dst, NULL));
    unsigned long long bad = 0;
    CUDA(cudaMemcpy(&bad, dst, 8, cudaMemcpyDeviceToHost));
    CUDA(cudaMemcpy(got, dout, m * 4, cudaMemcpyDeviceToHost));
    uint64_t wrong = 0;
    for (uint64_t j = 0; j < m; ++j) wrong += got[j] != want[j];
    if (wrong || bad != ~0ull) {
      fprintf(stderr, "%s: %llu wrong answers, first_bad %llu\n", names[v], (unsigned long long)wrong, bad);
      return 1;
    }
    printf("%s: %llu queries exact\n", names[v], (unsigned long long)m);
  }

  /* end-to-end host path, and the OutOfDomain contract */
  memset(got, 0xAB, m * 4);
  CHECK(fs_search_host(&plan, z, m, got, 4, dz, dout, (unsigned long long*)dst, 65536, &pos, NULL, NULL, 0));
  for (uint64_t j = 0; j < m; ++j)
    if (got[j] != want[j]) {
      fprintf(stderr, "host path wrong at %llu\n", (unsigned long long)j);
      return 1;
    }
  z[777777] = x[n1 - 1];    /* right endpoint: out of domain */
  z[900000] = NAN;
  memset(got, 0x5A, m * 4);
  int rc = fs_search_host(&plan, z, m, got, 4, dz, dout, (unsigned long long*)dst, 65536, &pos, NULL, NULL, 0);
  if (rc != FS_OUT_OF_DOMAIN || pos != 777777) {
    fprintf(stderr, "expected FS_OUT_OF_DOMAIN at 777777, got rc=%d pos=%lld\n", rc, (long long)pos);
    return 1;
  }
  for (uint64_t j = 0; j < m; ++j)
    if (((uint32_t*)got)[j] != 0x5A5A5A5Au) {
      fprintf(stderr, "out written despite OutOfDomain\n");
      return 1;
    }
  printf("host path exact; OutOfDomain(777777) with out untouched\n");
  printf("PASS %s h=%.9g r=%llu\n", fs_version(), (double)h, (unsigned long long)r);
  return 0;
}
