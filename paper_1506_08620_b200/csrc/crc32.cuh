// crc32.cuh — zlib-compatible CRC-32 of a device buffer (index-file
// checksum, bench/persist.py:63,91), computed in parallel on the GPU.
//
// The payload is cut into fixed CHUNK-byte chunks.  Each thread computes the
// standard CRC-32 (reflected polynomial 0xEDB88320, pre/post inverted) of
// one chunk with slice-by-4 tables in shared memory; a log-depth tree then
// merges neighbours with the GF(2) identity
//     crc(A || B) = (crc(A) * x^(8|B|) mod P) xor crc(B)
// (the conditioning of the standard CRC cancels in this identity), where
// x^(8n) mod P comes from repeated squaring of x^(2^k) mod P.
#pragma once

#include <cstdint>

namespace fsg {

constexpr uint32_t kCrcPoly = 0xedb88320u;
constexpr uint32_t kCrcChunk = 4096;

// a(x) * b(x) mod P in the reflected representation (bit 31 = x^0).
__host__ __device__ __forceinline__ uint32_t crc_multmodp(uint32_t a, uint32_t b) {
  uint32_t m = 1u << 31, p = 0;
  for (;;) {
    if (a & m) {
      p ^= b;
      if ((a & (m - 1)) == 0) break;
    }
    m >>= 1;
    b = (b & 1) ? (b >> 1) ^ kCrcPoly : b >> 1;
  }
  return p;
}

// x^(8n) mod P.
__device__ __forceinline__ uint32_t crc_x8n(uint64_t n) {
  uint32_t x2k = 1u << 23;  // x^8 in reflected form (x^k is bit 31 - k)
  uint32_t p = 1u << 31;    // x^0
  while (n) {
    if (n & 1) p = crc_multmodp(x2k, p);
    x2k = crc_multmodp(x2k, x2k);
    n >>= 1;
  }
  return p;
}

__device__ __forceinline__ uint32_t crc_combine(uint32_t crc_a, uint32_t crc_b, uint64_t len_b) {
  return crc_multmodp(crc_x8n(len_b), crc_a) ^ crc_b;
}

// CRC of each CHUNK-byte chunk (the last may be shorter).
__global__ void crc32_chunks_kernel(const unsigned char* __restrict__ data, uint64_t bytes, uint32_t* __restrict__ out,
                                    uint64_t nchunks) {
  __shared__ uint32_t T[4][256];
  for (uint32_t i = threadIdx.x; i < 256; i += blockDim.x) {
    uint32_t c = i;
    for (int k = 0; k < 8; ++k) c = (c & 1) ? (c >> 1) ^ kCrcPoly : c >> 1;
    T[0][i] = c;
  }
  __syncthreads();
  for (uint32_t i = threadIdx.x; i < 256; i += blockDim.x) {
    uint32_t c = T[0][i];
    for (int t = 1; t < 4; ++t) {
      c = (c >> 8) ^ T[0][c & 0xff];
      T[t][i] = c;
    }
  }
  __syncthreads();
  for (uint64_t ch = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; ch < nchunks;
       ch += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t a = ch * kCrcChunk;
    const uint64_t b = a + kCrcChunk < bytes ? a + kCrcChunk : bytes;
    const unsigned char* p = data + a;
    uint64_t n = b - a;
    uint32_t crc = 0xffffffffu;
    // bytes until 4-B alignment, then words, then the tail
    while (n && (reinterpret_cast<uintptr_t>(p) & 3)) {
      crc = T[0][(crc ^ *p++) & 0xff] ^ (crc >> 8);
      --n;
    }
    const uint32_t* w = reinterpret_cast<const uint32_t*>(p);
    for (; n >= 4; n -= 4) {
      crc ^= __ldg(w++);
      crc = T[3][crc & 0xff] ^ T[2][(crc >> 8) & 0xff] ^ T[1][(crc >> 16) & 0xff] ^ T[0][crc >> 24];
    }
    p = reinterpret_cast<const unsigned char*>(w);
    while (n--) crc = T[0][(crc ^ *p++) & 0xff] ^ (crc >> 8);
    out[ch] = ~crc;
  }
}

// One tree level: c[i] = combine(c[i], c[i + step]) for i % (2 step) == 0.
__global__ void crc32_combine_kernel(uint32_t* __restrict__ c, uint64_t nchunks, uint64_t step, uint64_t bytes) {
  for (uint64_t t = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; t * 2 * step + step < nchunks;
       t += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t i = t * 2 * step, j = i + step;
    const uint64_t end_chunk = j + step < nchunks ? j + step : nchunks;
    const uint64_t b0 = j * kCrcChunk;
    const uint64_t b1 = end_chunk * (uint64_t)kCrcChunk < bytes ? end_chunk * (uint64_t)kCrcChunk : bytes;
    c[i] = crc_combine(c[i], c[j], b1 - b0);
  }
}

}  // namespace fsg
