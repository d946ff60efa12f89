// common.cuh — sm_100a device helpers shared by the search and build kernels.
//
// Numeric helpers pin the reference's numpy semantics exactly
// (SURVEY.md Appendix A): every float op is an explicit _rn intrinsic so
// nvcc can neither contract nor reassociate, and the bucket index is a
// round-toward-zero conversion (numpy .astype(np.int64) on a non-negative
// value, batch.py:316).  The library is compiled without --use_fast_math and
// with -ftz=false -prec-div=true so subnormals survive, as in numpy.
#pragma once

#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

namespace fsg {

// Sparse two-level table: bit 31 of a super-bucket rank C[J] marks a dense
// (bitmask) super-bucket (knot indices stay below 2^31).
constexpr uint32_t kDenseFlag = 0x80000000u;
// Super-buckets holding more knots than this are stored densely.
constexpr uint32_t kDenseOcc = 64;
// Group records (fs_build_sparse_rec): knot offsets per record (16-B
// records hold six, 8-B records two), the value of an unused offset slot, and
// the largest super-bucket shift (its offsets stay below the sentinel and the
// 15-bit SWAR compare of the probe).
template <int SLOTS> struct RecWord;
template <> struct RecWord<6> { using type = uint4; };
template <> struct RecWord<2> { using type = uint2; };
template <> struct RecWord<8> { using type = uint4; };
template <> struct RecWord<3> { using type = uint2; };
constexpr uint32_t kRecSentinel = 0x7FFFu;
constexpr int kRecMaxShift = 14;
// 16-B records with eight 12-bit offset fields (FS_SPARSE_RECORDS12): each
// field stored as 0x800 | offset (guard bit preset, offsets < 2^10), unused
// fields 0xFFF; shifts up to 10.
constexpr int kRec12MaxShift = 10;
// 8-B records with three 13-bit offset fields (FS_SPARSE_RECORDS8X3): the
// 64-bit word is base (bits 0..23, N + 1 <= 2^24) | overflow (bit 24) | fields
// 0x1000 | offset at bits 25 + 13k (offsets < 2^11, unused 0x1FFF); shifts up
// to 11.
constexpr int kRec3MaxShift = 11;
// Zoned records (FS_SPARSE_ZONED, 8 B each): at most this many zones, so a
// warp's zone-descriptor loads touch at most two words per bank; slot records
// are the three-offset 8-B records (24-bit base, 13-bit fields) at shifts
// kZonedMinShift..kZonedMaxShift; a zone no slot shift fits takes 32-bucket
// rank records {mask, base} (the same 8 B per 32 buckets as a slot record at
// shift 5, with a cheaper decode).
constexpr uint32_t kZonedMaxZones = 64;
constexpr int kZonedSlots = 3;
constexpr int kZonedMinShift = 6;
constexpr int kZonedMaxShift = kRec3MaxShift;
constexpr int kZonedMinZoneShift = kRec3MaxShift;
constexpr int kZonedRankShift = 5;
constexpr uint32_t kZonedRankFlag = 16u;
constexpr int kZonedMaxStripe = 10;  // striped rank words: a mask bit per 2^k buckets, k <= 10
// Count words (FS_SPARSE_COUNT): one stripe shift k for the whole table, 16
// stripes of 2^k buckets per 8-B word {2-bit knot counts, first knot index},
// bit 31 of the index flags a word with a stripe of four or more knots
constexpr int kCountWordShift = 4;
constexpr int kCountMaxShift = 27;
constexpr uint32_t kCountFlag = 0x80000000u;
constexpr int kCountMaxOffsetShift = 8;  // knot offsets beside the words are bytes: stripes of at most 2^8 buckets

// Bounds-checked builds (FSG_BOUNDS_CHECK=1, tools/bounds_check.sh): every
// table gather of the search probes checks its index against the table's
// extent, and every shared-memory gather its offset against the CTA's dynamic
// shared memory, and traps on a violation.  compute-sanitizer is closed on
// this GPU pool; the GPU test suite runs against this build instead.
#ifndef FSG_BOUNDS_CHECK
#define FSG_BOUNDS_CHECK 0
#endif
#if FSG_BOUNDS_CHECK
#define FSG_BOUND(c)                                                                   \
  do {                                                                                 \
    if (!(c)) {                                                                        \
      printf("fsg bounds check failed: %s (%s:%d)\n", #c, __FILE__, __LINE__);         \
      __trap();                                                                        \
    }                                                                                  \
  } while (0)
#else
#define FSG_BOUND(c) \
  do {               \
  } while (0)
#endif
__device__ __forceinline__ uint32_t dyn_smem_bytes() {
  uint32_t v;
  asm("mov.u32 %0, %%dynamic_smem_size;" : "=r"(v));
  return v;
}

// ---------------------------------------------------------------------------
// Exact arithmetic in the partition's precision
// ---------------------------------------------------------------------------
__device__ __forceinline__ float sub_rn(float a, float b) { return __fsub_rn(a, b); }
__device__ __forceinline__ double sub_rn(double a, double b) { return __dsub_rn(a, b); }
__device__ __forceinline__ float mul_rn(float a, float b) { return __fmul_rn(a, b); }
__device__ __forceinline__ double mul_rn(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ float add_rn(float a, float b) { return __fadd_rn(a, b); }
__device__ __forceinline__ double add_rn(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ float div_rn(float a, float b) { return __fdiv_rn(a, b); }
__device__ __forceinline__ double div_rn(double a, double b) { return __ddiv_rn(a, b); }

// Truncation toward zero (values here are >= 0 or NaN; saturating cvt keeps
// out-of-domain lanes in range before the clamp).
template <typename J> __device__ __forceinline__ J trunc_to(float v);
template <typename J> __device__ __forceinline__ J trunc_to(double v);
template <> __device__ __forceinline__ uint32_t trunc_to<uint32_t>(float v) { return __float2uint_rz(v); }
template <> __device__ __forceinline__ uint32_t trunc_to<uint32_t>(double v) { return __double2uint_rz(v); }
template <> __device__ __forceinline__ uint64_t trunc_to<uint64_t>(float v) { return __float2ull_rz(v); }
template <> __device__ __forceinline__ uint64_t trunc_to<uint64_t>(double v) { return __double2ull_rz(v); }

// nextafter(h, +inf) for a positive finite (or +inf) value: one ulp up.
__device__ __forceinline__ float next_up(float v) {
  return __int_as_float(__float_as_int(v) + (v < INFINITY ? 1 : 0));
}
__device__ __forceinline__ double next_up(double v) {
  return __longlong_as_double(__double_as_longlong(v) + (v < (double)INFINITY ? 1ll : 0ll));
}

// Order-preserving key of a non-negative float (positive floats sort like
// their bit patterns), for exact atomic min reductions.
__device__ __forceinline__ unsigned long long order_key(float v) { return (unsigned long long)__float_as_uint(v); }
__device__ __forceinline__ unsigned long long order_key(double v) { return (unsigned long long)__double_as_longlong(v); }
template <typename T> __device__ __forceinline__ T from_key(unsigned long long k);
template <> __device__ __forceinline__ float from_key<float>(unsigned long long k) { return __uint_as_float((unsigned)k); }
template <> __device__ __forceinline__ double from_key<double>(unsigned long long k) { return __longlong_as_double((long long)k); }

// ---------------------------------------------------------------------------
// Streaming global memory access (the query stream is touched exactly once)
// ---------------------------------------------------------------------------
// Streaming-access variants (build-time, for A/B tuning): FSG_LD_VARIANT
// 0 = nc + L1::no_allocate + L2::256B prefetch, 1 = plain nc, 2 = __ldcs
// (evict-first); FSG_ST_VARIANT 0 = st.global.cs, 1 = plain st.global.
#ifndef FSG_LD_VARIANT
#define FSG_LD_VARIANT 1  // measured: +2% on cfg3 over variant 0
#endif
#ifndef FSG_ST_VARIANT
#define FSG_ST_VARIANT 0
#endif

__device__ __forceinline__ float4 ld_stream(const float4* p) {
#if FSG_LD_VARIANT == 0
  float4 v;
  asm volatile("ld.global.nc.L1::no_allocate.L2::256B.v4.f32 {%0,%1,%2,%3}, [%4];"
               : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "l"(p));
  return v;
#elif FSG_LD_VARIANT == 1
  return __ldg(p);
#else
  return __ldcs(p);
#endif
}
__device__ __forceinline__ double2 ld_stream(const double2* p) {
#if FSG_LD_VARIANT == 0
  double2 v;
  asm volatile("ld.global.nc.L1::no_allocate.L2::256B.v2.f64 {%0,%1}, [%2];"
               : "=d"(v.x), "=d"(v.y) : "l"(p));
  return v;
#elif FSG_LD_VARIANT == 1
  return __ldg(p);
#else
  return __ldcs(p);
#endif
}
__device__ __forceinline__ float ld_stream(const float* p) { return __ldcs(p); }
__device__ __forceinline__ double ld_stream(const double* p) { return __ldcs(p); }

#if FSG_ST_VARIANT == 0
__device__ __forceinline__ void st_stream(int4* p, int4 v) { __stcs(p, v); }
__device__ __forceinline__ void st_stream(longlong2* p, longlong2 v) { __stcs(p, v); }
#else
__device__ __forceinline__ void st_stream(int4* p, int4 v) { *p = v; }
__device__ __forceinline__ void st_stream(longlong2* p, longlong2 v) { *p = v; }
#endif
__device__ __forceinline__ void st_stream(int32_t* p, int32_t v) { __stcs(p, v); }
__device__ __forceinline__ void st_stream(int64_t* p, int64_t v) {
  __stcs(reinterpret_cast<long long*>(p), (long long)v);
}

// ---------------------------------------------------------------------------
// Shared-memory staging with the bulk-copy engine (cp.async.bulk + mbarrier)
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}

// One bulk copy global -> shared (dst/src 16 B aligned, bytes % 16 == 0,
// bytes < 2^20 per mbarrier phase).
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

// A table to stage: `bytes` from global `src` into shared `dst`.
struct StageSeg {
  void* dst;
  const void* src;
  uint32_t bytes;
};

// Stage up to 3 tables into shared memory.  The 16-B aligned body of each
// table goes through the bulk-copy engine (one elected thread issues, the
// mbarrier's transaction count tracks completion); any misaligned head/tail
// bytes are copied by the remaining threads.  On return all tables are
// visible to every thread of the CTA.
__device__ __forceinline__ void stage_tables(const StageSeg* segs, int nseg, uint64_t* bar) {
  const int tid = threadIdx.x;
  if (tid == 0) mbar_init(bar, 1);
  __syncthreads();
  uint32_t bulk_total = 0;
  uint32_t body_lo[3], body_hi[3];
  for (int s = 0; s < nseg; ++s) {
    uintptr_t src = reinterpret_cast<uintptr_t>(segs[s].src);
    uintptr_t dst = reinterpret_cast<uintptr_t>(segs[s].dst);
    uint32_t lo = 0, hi = 0;
    // bulk copy needs src and dst with the same alignment mod 16
    if (((src ^ dst) & 15u) == 0) {
      lo = (uint32_t)((16u - (src & 15u)) & 15u);
      if (lo > segs[s].bytes) lo = segs[s].bytes;
      hi = lo + ((segs[s].bytes - lo) & ~15u);
    }
    body_lo[s] = lo;
    body_hi[s] = hi;
    bulk_total += hi - lo;
  }
  if (tid == 0) {
    mbar_arrive_expect_tx(bar, bulk_total);
    for (int s = 0; s < nseg; ++s) {
      uint32_t off = body_lo[s];
      while (off < body_hi[s]) {
        uint32_t n = body_hi[s] - off;
        if (n > (1u << 16)) n = 1u << 16;  // keep individual copies moderate
        bulk_g2s(static_cast<char*>(segs[s].dst) + off, static_cast<const char*>(segs[s].src) + off, n,
                 bar);
        off += n;
      }
    }
  }
  // head/tail (and whole misaligned tables) byte copies
  for (int s = 0; s < nseg; ++s) {
    const unsigned char* src = static_cast<const unsigned char*>(segs[s].src);
    unsigned char* dst = static_cast<unsigned char*>(segs[s].dst);
    for (uint32_t b = tid; b < body_lo[s]; b += blockDim.x) dst[b] = src[b];
    for (uint32_t b = body_hi[s] + tid; b < segs[s].bytes; b += blockDim.x) dst[b] = src[b];
  }
  __syncthreads();
  mbar_wait(bar, 0);
}

// ---------------------------------------------------------------------------
// Warp reductions
// ---------------------------------------------------------------------------
__device__ __forceinline__ unsigned long long warp_min_u64(unsigned long long v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    unsigned long long w = __shfl_xor_sync(0xffffffffu, v, o);
    v = w < v ? w : v;
  }
  return v;
}

// Status workspace of one search (fs_search_ws_words() u64 words, zeroed
// once by its owner): [0] result (first out-of-domain position or ~0),
// [1] CTA ticket counter, [2] running max of ~position over the CTAs that
// saw a bad query; [1] and [2] are left at 0 after every launch.
constexpr int kStatusHeader = 3;

// Fold every lane's first-bad candidate into status[0] without a prior
// memset.  Warps that saw a bad query fold ~pos into status[2] (atomicMax,
// so the zero-initialised word means "none"); every CTA takes a ticket and
// the last one turns status[2] into the result (merge != 0: min with the
// current value, for several launches over one batch) and rewinds [1], [2].
// A single launch (merge == 0) also writes status[3] = status[0] ^ 2^63:
// the same order under a SIGNED comparison, "none" the int64 maximum -- the
// word a MIN all-reduce over shards takes as is (dist.sharded_batch_search).
__device__ __forceinline__ void finalize_first_bad(unsigned long long mine, unsigned long long* status, int merge) {
  __shared__ int s_last;
  if (__any_sync(0xffffffffu, mine != ~0ull)) {
    const unsigned long long w = warp_min_u64(mine);
    if ((threadIdx.x & 31) == 0 && w != ~0ull) atomicMax(status + 2, ~w);
  }
  __syncthreads();  // every warp's fold is issued before the CTA's ticket
  if (threadIdx.x == 0) {
    __threadfence();
    const unsigned int ticket = atomicAdd(reinterpret_cast<unsigned int*>(status + 1), 1u);
    s_last = ticket == gridDim.x - 1;
    if (s_last) {
      __threadfence();
      const unsigned long long first = ~__ldcg(status + 2);
      if (merge) {
        atomicMin(status, first);
      } else {
        status[0] = first;
        status[3] = first ^ (1ull << 63);
      }
      status[2] = 0;
      *reinterpret_cast<volatile unsigned int*>(status + 1) = 0u;
    }
  }
}

}  // namespace fsg
