// search.cuh — batch search kernels (the hot path).
//
// One persistent, grid-stride kernel template streams the query array Z
// (128-bit evict-first loads, 128-bit streaming stores) and resolves each
// query with an `Algo` probe.  Tables are staged into shared memory by the
// bulk-copy engine when they fit, otherwise gathered
// through L2 with ld.global.nc.  The out-of-domain check of batch_search
// (batch.py:411-413) is fused: each lane keeps the smallest bad position it
// saw, one atomic per warp folds it into the status workspace, and the CTA
// that finishes last publishes the batch's first bad position
// (finalize_first_bad, common.cuh).
//
// Probes (each cites the reference kernel it restates):
//   Direct<gap 1>     batch.py:315-317 / direct.py:272-276
//   Direct<gap 2>     batch.py:341-343 / direct.py:279-291
//   Direct<generic q> direct.py:294-300
//   DirectCache       batch.py:368-371 / direct.py:303-312
//   Bitset2           batch.py:193-200 / binsearch.py:72-86
//   Bitset1 / Bitset3 batch.py:176-185, 208-216 / binsearch.py:60-69, 89-99
//   Offset            batch.py:224-234 / binsearch.py:102-114
//   Eytzinger         batch.py:242-246 / eytzinger.py:84-89
//   Classic           binsearch.py:48-57
#pragma once

#include <type_traits>

#include "common.cuh"

// Queries per two-phase group in the rank-directory probe (gathers in flight
// per thread vs live registers / occupancy).
#ifndef FSG_RANK_GROUP
#define FSG_RANK_GROUP 8
#endif

// bitset2: subtree-record gathers in flight per group.
#ifndef FSG_B2_DEEP_GROUP
#define FSG_B2_DEEP_GROUP 4
#endif

// Queries per two-phase group in the group-record probe.
#ifndef FSG_REC_GROUP
#define FSG_REC_GROUP 4
#endif

namespace fsg {

// Device image of fs_plan with typed scalars.
template <typename T>
struct DevPlan {
  const T* x;            // knots
  const void* table;     // K / records / padded / tree
  const uint2* rank;     // rank directory of K (direct, gap 1) or NULL
  const void* rows;      // 16-B rank rows (FS_SPARSE_RANK_ROWS) or NULL
  uint64_t n1;           // N+1
  uint64_t r;            // R (direct family)
  T h, x0, xn;           // scale, domain
  int32_t q;             // gap
  int32_t pbits;         // bitset / eytzinger depth
  int32_t top_bits;      // bitset2: levels served from smem
  int32_t b2_l1, b2_l2;  // bitset2: levels [b2_l1, b2_l2) replicated per bank in smem
  int32_t b2_l3;         // bitset2: levels [b2_l2, b2_l3) in 16 copies (lane pairs share one)
  const void* b2_deep;   // bitset2: subtree records of the levels below top_bits, or NULL
  int32_t b2_deep_k;     // ... levels per record
  uint32_t off_f, off_s, off_j;  // offset search constants
  uint32_t x_smem_bytes;     // bytes of X (or padded / tree / top table) staged; 0 = global
  uint32_t table_smem_bytes; // bytes of K / records staged; 0 = global
  int32_t out_vec_ok;        // output groups 16-B aligned (1) / 32-B aligned (2) / neither (0)
  int32_t sparse_shift;      // sparse two-level table: super-bucket = 2^shift buckets
  uint32_t sparse_ndense;    // ... and its number of dense (bitmask) super-buckets
  uint32_t hot_w0, hot_nw;   // rank-directory hot window (words) staged in smem
  uint32_t hot_t0, hot_nt;   // knot window X[t0, t0 + nt) staged in smem
  __host__ __device__ __forceinline__ uint32_t x_smem_bytes_aligned() const {
    return (x_smem_bytes + 127u) & ~127u;
  }
};

template <bool S, typename V>
__device__ __forceinline__ V tload(const V* p, uint64_t i) {
  if constexpr (S) return p[i];
  else return __ldg(p + i);
}

// ---------------------------------------------------------------------------
// Direct search, gap 1 / 2 / generic.  j = trunc(RN(RN(z - x0) * h)) in the
// partition's precision (Appendix A.1), clamped to R so out-of-domain lanes
// stay in bounds (in-domain j <= R always: RN is monotone and z < XN).
// ---------------------------------------------------------------------------
template <typename T, typename J, int GAP, bool XS, bool KS>
struct DirectProbe {
  const T* X;
  const uint32_t* K;
  T h, x0;
  J r;
  int q;
  uint64_t n1;  // knots (bounds checks)
  __device__ __forceinline__ DirectProbe(const DevPlan<T>& p, unsigned char* smem) {
    n1 = p.n1;
    X = XS ? reinterpret_cast<const T*>(smem) : p.x;
    K = KS ? reinterpret_cast<const uint32_t*>(smem + p.x_smem_bytes_aligned()) : static_cast<const uint32_t*>(p.table);
    h = p.h;
    x0 = p.x0;
    r = (J)p.r;
    q = p.q;
  }
  __device__ __forceinline__ int64_t operator()(T z) const {
    J j = trunc_to<J>(mul_rn(sub_rn(z, x0), h));
    j = j < r ? j : r;
    const uint32_t t = tload<KS>(K, j);
    FSG_BOUND((uint64_t)j <= (uint64_t)r && (uint64_t)t < n1 + (uint64_t)q);  // X holds q - 1 left pads
    if constexpr (GAP == 1) {
      return (int64_t)t - (z < tload<XS>(X, t) ? 1 : 0);
    } else if constexpr (GAP == 2) {
      // xpad[w+1] = X_w with xpad[0] = X0 (left_pad): the read of X_{t-1} is
      // clamped to X0, which never satisfies z < X0 for in-domain z.
      const uint32_t tm = t ? t - 1 : 0;
      return (int64_t)t - (z < tload<XS>(X, t) ? 1 : 0) - (z < tload<XS>(X, tm) ? 1 : 0);
    } else {
      int64_t hits = 0;
      for (int m = 0; m < q; ++m) {
        const int64_t w = (int64_t)t - m;
        hits += z < tload<XS>(X, (uint64_t)(w > 0 ? w : 0)) ? 1 : 0;
      }
      return (int64_t)t - hits;
    }
  }
};

// Direct search (gap 1) over the rank directory of K: identical answers to
// DirectProbe<GAP=1> (t = K[j] is recovered exactly; when bucket j holds no
// knot, z < X[t] is implied by the monotone bucket function, so the X read
// is skipped).  One 8-B gather per query, plus an X read only for queries
// whose bucket holds a knot (#knots / R of them).
template <typename T, typename J, bool XS, bool DS>
struct RankProbe {
  const T* X;
  const uint2* D;
  T h, x0;
  J r;
  uint64_t n1;
  __device__ __forceinline__ RankProbe(const DevPlan<T>& p, unsigned char* smem) {
    n1 = p.n1;
    X = XS ? reinterpret_cast<const T*>(smem) : p.x;
    D = DS ? reinterpret_cast<const uint2*>(smem + p.x_smem_bytes_aligned()) : p.rank;
    h = p.h;
    x0 = p.x0;
    r = (J)p.r;
  }
  __device__ __forceinline__ int64_t operator()(T z) const {
    J j = trunc_to<J>(mul_rn(sub_rn(z, x0), h));
    j = j < r ? j : r;
    const uint2 d = tload<DS>(D, (uint64_t)(j >> 5));
    const uint32_t b = (uint32_t)j & 31u;
    const uint32_t t = d.y + __popc(d.x & ((1u << b) - 1u));
    const bool knot = (d.x >> b) & 1u;
    FSG_BOUND((uint64_t)j <= (uint64_t)r && (!knot || t < n1));
    // lanes whose bucket holds no knot read X[0] (a broadcast), never a
    // conflicting bank, and their answer is t - 1 regardless
    const T xv = tload<XS>(X, knot ? t : 0u);
    return (int64_t)t - ((!knot || z < xv) ? 1 : 0);
  }
#if FSG_RANK_GROUP > 0
  // Two phases over N queries: every directory gather is in flight before
  // the first is consumed; X is then read only for buckets holding a knot
  // (predicated load, no memory traffic for the other lanes).
  template <int N, typename R>
  __device__ __forceinline__ void batch(const T (&z)[N], R (&o)[N]) const {
    constexpr int G = N < FSG_RANK_GROUP ? N : FSG_RANK_GROUP;  // live-register bound
#pragma unroll
    for (int g0 = 0; g0 < N; g0 += G) {
      uint2 d[G];
      uint32_t b[G];
#pragma unroll
      for (int q = 0; q < G; ++q) {
        if (g0 + q >= N) break;  // N need not be a multiple of G (compile-time)
        J j = trunc_to<J>(mul_rn(sub_rn(z[g0 + q], x0), h));
        j = j < r ? j : r;
        b[q] = (uint32_t)j & 31u;
        FSG_BOUND((uint64_t)j <= (uint64_t)r);
        d[q] = tload<DS>(D, (uint64_t)(j >> 5));
      }
#pragma unroll
      for (int q = 0; q < G; ++q) {
        if (g0 + q >= N) break;
        const uint32_t t = d[q].y + __popc(d[q].x & ((1u << b[q]) - 1u));
        const bool knot = (d[q].x >> b[q]) & 1u;
        FSG_BOUND(!knot || t < n1);
        T xv = z[g0 + q];
        if (knot) xv = tload<XS>(X, t);
        o[g0 + q] = (R)((int64_t)t - ((!knot || z[g0 + q] < xv) ? 1 : 0));
      }
    }
  }
#endif
};

// RankProbe for tables whose directory fits in shared memory but whose X does
// not: the directory and one byte per knot (fill_knot_bytes_kernel: where
// inside its bucket the knot falls, to 1/256, from the same rounded product p
// whose floor is the bucket) are staged.  For a query in a bucket holding knot
// t, the byte of its own product against the knot's decides z < X[t] (RN is
// monotone: p_z < p_t implies z < X[t], p_z > p_t implies z > X[t]); only a tie
// (1/256 of those queries) reads X[t] through L2.  Same answers as RankProbe.
template <typename T>
struct RankBytesProbe {
  const T* X;
  uint32_t ds, bs;  // shared addresses of the directory and the knot bytes
  T h, x0;
  uint32_t r, n1;
  __device__ __forceinline__ RankBytesProbe(const DevPlan<T>& p, unsigned char* smem) {
    n1 = (uint32_t)p.n1;
    X = p.x;
    // staged as [knot bytes | directory]
    asm volatile("mov.u32 %0, %1;" : "=r"(bs) : "r"((uint32_t)__cvta_generic_to_shared(smem)));
    asm volatile("mov.u32 %0, %1;" : "=r"(ds) : "r"(bs + p.x_smem_bytes_aligned()));
    h = p.h;
    x0 = p.x0;
    r = (uint32_t)p.r;
  }
  // bucket j (clamped to R) and the query's byte inside it
  __device__ __forceinline__ void locate(T z, uint32_t& j, uint32_t& qz) const {
    const T p = mul_rn(sub_rn(z, x0), h);
    const T fl = floor(p);
    j = trunc_to<uint32_t>(fl);
    j = j < r ? j : r;
    qz = trunc_to<uint32_t>(mul_rn(sub_rn(p, fl), (T)256));
  }
  __device__ __forceinline__ uint2 word(uint32_t j) const {
    uint2 d;
    asm("ld.shared.v2.u32 {%0, %1}, [%2];" : "=r"(d.x), "=r"(d.y) : "r"(ds + 8u * (j >> 5)));
    return d;
  }
  __device__ __forceinline__ int64_t finish(const uint2& d, uint32_t j, uint32_t qz, T z) const {
    const uint32_t b = j & 31u;
    uint32_t below;
    asm("bmsk.clamp.b32 %0, 0, %1;" : "=r"(below) : "r"(b));
    const uint32_t t = d.y + __popc(d.x & below);
    const uint32_t knot = (d.x >> b) & 1u;
    FSG_BOUND(!knot || t < n1);
    uint32_t o = 256u;  // no knot in the bucket: every query byte is below it
    asm("{\n\t.reg .pred p;\n\tsetp.ne.u32 p, %2, 0;\n\t@p ld.shared.u8 %0, [%1];\n\t}" : "+r"(o) : "r"(bs + t), "r"(knot));
    uint32_t res = t - (qz < o ? 1u : 0u);
    if (qz == o) res = t - (z < __ldg(X + t) ? 1u : 0u);  // a tie in the byte (knot is set: o < 256)
    return (int64_t)(int32_t)res;
  }
  __device__ __forceinline__ int64_t operator()(T z) const {
    uint32_t j, qz;
    locate(z, j, qz);
    return finish(word(j), j, qz, z);
  }
#ifndef FSG_RANKBYTES_GROUP
#define FSG_RANKBYTES_GROUP 2
#endif
  template <int N, typename R>
  __device__ __forceinline__ void batch(const T (&z)[N], R (&o)[N]) const {
    constexpr int G = N < FSG_RANKBYTES_GROUP ? N : FSG_RANKBYTES_GROUP;
#pragma unroll
    for (int g0 = 0; g0 < N; g0 += G) {
      uint2 d[G];
      uint32_t j[G], qz[G];
#pragma unroll
      for (int q = 0; q < G; ++q) {
        if (g0 + q >= N) break;
        locate(z[g0 + q], j[q], qz[q]);
        d[q] = word(j[q]);
      }
#pragma unroll
      for (int q = 0; q < G; ++q) {
        if (g0 + q >= N) break;
        o[g0 + q] = (R)finish(d[q], j[q], qz[q], z[g0 + q]);
      }
    }
  }
};

// RankProbe through L2 over 16-B rank rows (fill_rank_rows_kernel): the
// directory word of the query's 32 buckets and the knot bytes of the row's
// first eight knots arrive in one gather (one 32-B sector either way), so the
// second gather -- X[t], for every query whose bucket holds a knot -- is left
// to ties of the bytes and to a row's ninth and later knots.  For tables whose
// directory does not fit in shared memory (cfg5 N+1 = 2^20 + 1: 1.1 -> 1.0
// gathers per query).  Same answers as RankProbe.
template <typename T>
struct RankRowsProbe {
  const T* X;
  const uint4* D;
  T h, x0;
  uint32_t r, n1;
  __device__ __forceinline__ RankRowsProbe(const DevPlan<T>& p, unsigned char*) {
    n1 = (uint32_t)p.n1;
    X = p.x;
    D = static_cast<const uint4*>(p.rows);
    h = p.h;
    x0 = p.x0;
    r = (uint32_t)p.r;
  }
  __device__ __forceinline__ void locate(T z, uint32_t& j, uint32_t& qz) const {
    const T p = mul_rn(sub_rn(z, x0), h);
    const T fl = floor(p);
    j = trunc_to<uint32_t>(fl);
    j = j < r ? j : r;
    qz = trunc_to<uint32_t>(mul_rn(sub_rn(p, fl), (T)256));
  }
  __device__ __forceinline__ int64_t finish(const uint4& d, uint32_t j, uint32_t qz, T z) const {
    const uint32_t b = j & 31u;
    uint32_t below;
    asm("bmsk.clamp.b32 %0, 0, %1;" : "=r"(below) : "r"(b));
    const uint32_t tl = __popc(d.x & below);
    const uint32_t t = d.y + tl;
    const bool knot = (d.x >> b) & 1u;
    FSG_BOUND(!knot || t < n1);
    // the knot's byte (its place inside its bucket): byte tl of the row's eight;
    // no knot: above every query byte; a ninth or later knot: a forced tie
    uint32_t o = __byte_perm(d.z, d.w, tl & 7u) & 255u;
    o = tl < 8u ? o : qz;
    o = knot ? o : 256u;
    uint32_t res = t - (qz < o ? 1u : 0u);
    if (qz == o) res = t - (z < __ldg(X + t) ? 1u : 0u);  // a tie (knot is set: o < 256)
    return (int64_t)(int32_t)res;
  }
  __device__ __forceinline__ int64_t operator()(T z) const {
    uint32_t j, qz;
    locate(z, j, qz);
    return finish(__ldg(D + (j >> 5)), j, qz, z);
  }
#ifndef FSG_RANKROWS_GROUP
#define FSG_RANKROWS_GROUP 4
#endif
  template <int N, typename R>
  __device__ __forceinline__ void batch(const T (&z)[N], R (&o)[N]) const {
    constexpr int G = N < FSG_RANKROWS_GROUP ? N : FSG_RANKROWS_GROUP;
#pragma unroll
    for (int g0 = 0; g0 < N; g0 += G) {
      uint4 d[G];
      uint32_t j[G], qz[G];
#pragma unroll
      for (int q = 0; q < G; ++q) {
        if (g0 + q >= N) break;
        locate(z[g0 + q], j[q], qz[q]);
        FSG_BOUND(j[q] <= r);
        d[q] = __ldg(D + (j[q] >> 5));
      }
#pragma unroll
      for (int q = 0; q < G; ++q) {
        if (g0 + q >= N) break;
        o[g0 + q] = (R)finish(d[q], j[q], qz[q], z[g0 + q]);
      }
    }
  }
};

// Direct search (gap 2) over the rank directory of its table (fill_rank2_
// kernel): t = K2[j] recovered exactly; a bucket holding no knot needs no X
// read (its last knot lies in an earlier bucket, so X[t] < z by the
// monotone bucket function), one holding c knots needs the c reads of
// batch.py:341-343 (t - (z < X[t]) - (z < X[t-1])).  Identical answers to
// DirectProbe<GAP=2>.
template <typename T, bool XS, bool DS>
struct Rank2Probe {
  const T* X;
  const uint4* D;
  T h, x0;
  uint32_t r;
  uint64_t n1;
  __device__ __forceinline__ Rank2Probe(const DevPlan<T>& p, unsigned char* smem) {
    n1 = p.n1;
    X = XS ? reinterpret_cast<const T*>(smem) : p.x;
    D = DS ? reinterpret_cast<const uint4*>(smem + p.x_smem_bytes_aligned()) : reinterpret_cast<const uint4*>(p.rank);
    h = p.h;
    x0 = p.x0;
    r = (uint32_t)p.r;
  }
  __device__ __forceinline__ int64_t resolve(T z, uint4 d, uint32_t b) const {
    const uint32_t le = ((1u << b) << 1) - 1u;  // bits 0..b (b = 31: all)
    const uint32_t t = d.z + __popc(d.x & le) + __popc(d.y & le) - 1u;
    const uint32_t c = ((d.x >> b) & 1u) + ((d.y >> b) & 1u);
    uint32_t miss = 0;
    FSG_BOUND(c == 0 || (t < n1 && t + 1 >= c));
    if (c >= 1) miss += z < tload<XS>(X, t) ? 1u : 0u;
    if (c == 2) miss += z < tload<XS>(X, t - 1) ? 1u : 0u;
    return (int64_t)t - (int64_t)miss;
  }
  __device__ __forceinline__ int64_t operator()(T z) const {
    uint32_t j = trunc_to<uint32_t>(mul_rn(sub_rn(z, x0), h));
    j = j < r ? j : r;
    return resolve(z, tload<DS>(D, (uint64_t)(j >> 5)), j & 31u);
  }
  // every directory gather of the group in flight before the first is used
  template <int N, typename R>
  __device__ __forceinline__ void batch(const T (&z)[N], R (&o)[N]) const {
    constexpr int G = N < FSG_RANK_GROUP ? N : FSG_RANK_GROUP;
#pragma unroll
    for (int g0 = 0; g0 < N; g0 += G) {
      uint4 d[G];
      uint32_t b[G];
#pragma unroll
      for (int q = 0; q < G; ++q) {
        if (g0 + q >= N) break;
        uint32_t j = trunc_to<uint32_t>(mul_rn(sub_rn(z[g0 + q], x0), h));
        j = j < r ? j : r;
        b[q] = j & 31u;
        d[q] = tload<DS>(D, (uint64_t)(j >> 5));
      }
#pragma unroll
      for (int q = 0; q < G; ++q) {
        if (g0 + q >= N) break;
        o[g0 + q] = (R)resolve(z[g0 + q], d[q], b[q]);
      }
    }
  }
};

// Direct search (gap q >= 2) over the count directory of its table
// (fill_countdir_kernel): t = K_q[j] recovered exactly from one 8-B word;
// the knots of bucket j are X[t - c + 1 .. t] (c = its count <= q), every
// earlier knot lies in an earlier bucket and so below z (monotone bucket
// function), hence the reference's q clamped comparisons t - #{m < q : z <
// X[t - m]} (direct.py:294-300, batch.py:341-343) reduce to the c reads of
// the bucket's own knots -- usually none.  Identical answers to
// DirectProbe<GAP=q>.
template <typename T, int B, bool XS, bool DS>
struct CountDirProbe {
  static constexpr int LG = B == 2 ? 4 : 3;  // buckets per word: 16 / 8
  const T* X;
  const uint2* D;
  T h, x0;
  uint32_t r;
  uint64_t n1;
  __device__ __forceinline__ CountDirProbe(const DevPlan<T>& p, unsigned char* smem) {
    n1 = p.n1;
    X = XS ? reinterpret_cast<const T*>(smem) : p.x;
    D = DS ? reinterpret_cast<const uint2*>(smem + p.x_smem_bytes_aligned()) : p.rank;
    h = p.h;
    x0 = p.x0;
    r = (uint32_t)p.r;
  }
  // (sum of the counts of fields 0..b, count of field b) of a counts word
  static __device__ __forceinline__ void sums(uint32_t c, uint32_t b, uint32_t& s, uint32_t& cb) {
    const uint32_t hi = B * (b + 1);
    const uint32_t v = hi >= 32 ? c : c & ((1u << hi) - 1u);
    if constexpr (B == 2) {
      s = __popc(v & 0x55555555u) + 2u * __popc(v & 0xAAAAAAAAu);
    } else {
      const uint32_t bytes = (v & 0x0F0F0F0Fu) + ((v >> 4) & 0x0F0F0F0Fu);
      s = (bytes * 0x01010101u) >> 24;
    }
    cb = (c >> (B * b)) & ((1u << B) - 1u);
  }
  __device__ __forceinline__ int64_t resolve(T z, uint2 d, uint32_t b) const {
    uint32_t s, c;
    sums(d.x, b, s, c);
    const uint32_t t = d.y + s - 1u;
    uint32_t miss = 0;
    FSG_BOUND(c == 0 || (t < n1 && t + 1 >= c));
    for (uint32_t k = 0; k < c; ++k) miss += z < tload<XS>(X, t - k) ? 1u : 0u;
    return (int64_t)t - (int64_t)miss;
  }
  __device__ __forceinline__ int64_t operator()(T z) const {
    uint32_t j = trunc_to<uint32_t>(mul_rn(sub_rn(z, x0), h));
    j = j < r ? j : r;
    return resolve(z, tload<DS>(D, (uint64_t)(j >> LG)), j & ((1u << LG) - 1u));
  }
  // every directory gather of the group in flight before the first is used
  template <int N, typename R>
  __device__ __forceinline__ void batch(const T (&z)[N], R (&o)[N]) const {
    constexpr int G = N < FSG_RANK_GROUP ? N : FSG_RANK_GROUP;
#pragma unroll
    for (int g0 = 0; g0 < N; g0 += G) {
      uint2 d[G];
      uint32_t b[G];
#pragma unroll
      for (int q = 0; q < G; ++q) {
        if (g0 + q >= N) break;
        uint32_t j = trunc_to<uint32_t>(mul_rn(sub_rn(z[g0 + q], x0), h));
        j = j < r ? j : r;
        b[q] = j & ((1u << LG) - 1u);
        d[q] = tload<DS>(D, (uint64_t)(j >> LG));
      }
#pragma unroll
      for (int q = 0; q < G; ++q) {
        if (g0 + q >= N) break;
        o[g0 + q] = (R)resolve(z[g0 + q], d[q], b[q]);
      }
    }
  }
};

// Direct search (gap 1) over the two-level sparse encoding of K (fill_sparse_
// kernel), staged in shared memory: C (super-bucket ranks) and F (16-bit
// knot offsets) after X when X fits (else X via L2 -- read only for buckets
// holding a knot).  t = K[j] = C[J] + lower_bound(F[C[J] .. C[J+1]), j mod 2^s)
// exactly; bucket j holds knot t iff F[t] == j mod 2^s; identical answers to
// DirectProbe<GAP=1> (batch.py:315-317).
template <typename T, bool XS, bool DENSE>
struct SparseProbe {
  const T* X;
  const uint32_t* C;
  const uint16_t* F;
  const uint32_t* Dm;  // dense super-buckets: knot masks, W words each
  const uint16_t* Dp;  //                     per-word knot prefix counts
  T h, x0;
  uint32_t r, s, mask, wshift;
  uint64_t n1;
  __device__ __forceinline__ SparseProbe(const DevPlan<T>& p, unsigned char* smem) {
    n1 = p.n1;
    X = XS ? reinterpret_cast<const T*>(smem) : p.x;
    unsigned char* cf = smem + p.x_smem_bytes_aligned();
    const uint64_t nc = ((uint64_t)p.r >> p.sparse_shift) + 2;
    C = reinterpret_cast<const uint32_t*>(cf);
    F = reinterpret_cast<const uint16_t*>(cf + 4 * nc);
    const uint64_t dm_off = (4 * nc + 2 * p.n1 + 3) & ~3ull;
    Dm = reinterpret_cast<const uint32_t*>(cf + dm_off);
    Dp = reinterpret_cast<const uint16_t*>(cf + dm_off + 4ull * p.sparse_ndense * (1ull << (p.sparse_shift - 5)));
    h = p.h;
    x0 = p.x0;
    r = (uint32_t)p.r;
    s = (uint32_t)p.sparse_shift;
    mask = (1u << s) - 1u;
    wshift = s - 5;
  }
  __device__ __forceinline__ int64_t operator()(T z) const {
    uint32_t j = trunc_to<uint32_t>(mul_rn(sub_rn(z, x0), h));
    j = j < r ? j : r;
    const uint32_t J = j >> s, jl = j & mask;
    FSG_BOUND(J <= (r >> s));
    const uint32_t c = C[J];
    uint32_t t;
    bool knot;
    if (DENSE && (c & kDenseFlag)) {  // dense super-bucket: mask word + prefix, like the rank directory
      const uint32_t lo = c & ~kDenseFlag;
      const uint32_t widx = ((uint32_t)F[lo] << wshift) + (jl >> 5);
      const uint32_t m = Dm[widx], b = jl & 31u;
      t = lo + Dp[widx] + __popc(m & ((1u << b) - 1u));
      knot = (m >> b) & 1u;
    } else {  // lower_bound of jl among the super-bucket's knot offsets
      uint32_t lo = c, hi = DENSE ? C[J + 1] & ~kDenseFlag : C[J + 1];
      const uint32_t end = hi;
      while (lo < hi) {
        const uint32_t mid = (lo + hi) >> 1;
        if (F[mid] < jl) lo = mid + 1;
        else hi = mid;
      }
      t = lo;
      knot = lo < end && F[lo] == jl;
    }
    FSG_BOUND(!knot || t < n1);
    T xv = z;
    if (knot) xv = tload<XS>(X, t);
    return (int64_t)t - ((!knot || z < xv) ? 1 : 0);
  }
};

// Rank of jl among the eight 12-bit offset fields of a 16-B record (g.y..g.w,
// field k = 0x800 | offset at bit 12k, unused fields 0x7FF > any jl):
// lt = #{offsets < jl}, knot = (field lt == jl).  96-bit SWAR: (0x800 |
// offset) - jl keeps the field's bit 11 iff offset >= jl (no borrow leaves a
// field); Y = jl in every 12-bit field.
__device__ __forceinline__ void rec12_count(const uint4& g, uint32_t jl, uint32_t& lt, bool& knot) {
  const uint32_t y0 = jl * 0x01001001u;
  const uint32_t y1 = jl * 0x10010010u + (jl >> 8);
  const uint32_t y2 = jl * 0x00100100u + (jl >> 4);
  uint32_t d0, d1, d2;
  asm("sub.cc.u32 %0, %3, %6;\n\tsubc.cc.u32 %1, %4, %7;\n\tsubc.u32 %2, %5, %8;"
      : "=r"(d0), "=r"(d1), "=r"(d2)
      : "r"(g.y), "r"(g.z), "r"(g.w), "r"(y0), "r"(y1), "r"(y2));
  // guard bits at 11, 23, 35, 47, 59, 71, 83, 95: word0 bits 11, 23;
  // word1 bits 3, 15, 27; word2 bits 7, 19, 31
  const uint32_t ge = __popc(d0 & 0x00800800u) + __popc(d1 & 0x08008008u) + __popc(d2 & 0x80080080u);
  lt = 8u - ge;
  // field lt (bits 12 lt .. 12 lt + 11) through a funnel shift of its word
  // pair, chosen with predicated selects (ptxas otherwise branches on the
  // word index: a reconvergence region per query)
  const uint32_t bit = 12u * lt;
  uint32_t a0, a1;
  asm("{\n\t.reg .pred p, q;\n\tsetp.lt.u32 p, %2, 32;\n\tsetp.lt.u32 q, %2, 64;\n\t"
      "selp.b32 %0, %4, %5, q;\n\tselp.b32 %0, %3, %0, p;\n\tselp.b32 %1, %4, %5, p;\n\t}"
      : "=r"(a0), "=r"(a1)
      : "r"(bit), "r"(g.y), "r"(g.z), "r"(g.w));
  knot = lt < 8u && ((__funnelshift_r(a0, a1, bit & 31u) & 0x7FFu) == jl);
}

// Direct search (gap 1) over the group records of K (fill_sparse_rec_kernel),
// staged in shared memory after X when X fits.  One LDS per query; SLOTS
// selects the layout: 6 (16 B, 16-bit offsets), 2 (8 B, 16-bit offsets),
// 8 (16 B, 12-bit fields), 3 (8 B, 13-bit fields beside a 24-bit base).
// t = K[j] = base + #{record offsets < j mod 2^s}, counted branch-free with
// a SWAR compare of the packed offsets (guard bit per field; sentinels never
// count); bucket j holds knot t iff offset slot t - base equals j mod 2^s.  Only a
// query in an overflowing super-bucket (more than SLOTS knots) whose bucket
// lies past its last recorded knot continues with a lower_bound over F (OVF).
// Identical answers to DirectProbe<GAP=1> (batch.py:315-317).
template <typename T, int SLOTS, bool XS, bool OVF>
struct SparseRecProbe {
  using Rec = typename RecWord<SLOTS>::type;
  const T* X;
  uint32_t xs;  // shared-window address of X (XS)
  const Rec* G;
  const uint16_t* F;
  T h, x0;
  uint32_t r, s, mask;
  uint64_t n1;
  __device__ __forceinline__ SparseRecProbe(const DevPlan<T>& p, unsigned char* smem) {
    n1 = p.n1;
    X = XS ? reinterpret_cast<const T*>(smem) : p.x;
    // held in a register (volatile mov): ptxas would otherwise rebuild the
    // shared-window address (S2R + 3 ALU) in front of every X load
    asm volatile("mov.u32 %0, %1;" : "=r"(xs) : "r"((uint32_t)__cvta_generic_to_shared(smem)));
    unsigned char* g = smem + p.x_smem_bytes_aligned();
    G = reinterpret_cast<const Rec*>(g);
    F = reinterpret_cast<const uint16_t*>(g + sizeof(Rec) * (((uint64_t)p.r >> p.sparse_shift) + 2));
    h = p.h;
    x0 = p.x0;
    r = (uint32_t)p.r;
    s = (uint32_t)p.sparse_shift;
    mask = (1u << s) - 1u;
  }
  __device__ __forceinline__ uint32_t bucket(T z) const {
    uint32_t j = trunc_to<uint32_t>(mul_rn(sub_rn(z, x0), h));
    return j < r ? j : r;
  }
  // X[t]: a shared-window load from the pinned address (no generic-address
  // rematerialisation per query; int32 outputs +3%, int64 outputs measure
  // better with the generic load), or an L2 gather
  template <bool PINNED = true>
  __device__ __forceinline__ T xat(uint32_t t) const {
    if constexpr (XS && !PINNED) {
      return X[t];
    } else if constexpr (XS) {
      T v;
      if constexpr (sizeof(T) == 4) asm("ld.shared.f32 %0, [%1];" : "=f"(v) : "r"(xs + 4u * t));
      else asm("ld.shared.f64 %0, [%1];" : "=d"(v) : "r"(xs + 8u * t));
      return v;
    } else {
      return __ldg(X + t);
    }
  }
  // a record's first knot index and overflow flag (8-B/3-offset records keep
  // them in bits 0..23 and 24, the others in 31 bits and bit 31)
  static __device__ __forceinline__ uint32_t base_of(Rec g) {
    if constexpr (SLOTS == 3) return g.x & 0xFFFFFFu;
    else return g.x & ~kDenseFlag;
  }
  static __device__ __forceinline__ bool overflows(Rec g) {
    if constexpr (SLOTS == 3) return (g.x >> 24) & 1u;
    else return (g.x & kDenseFlag) != 0;
  }
  // (t, knot) of bucket j from its group record g
  __device__ __forceinline__ void resolve(Rec g, uint32_t j, uint32_t& t, bool& knot) const {
    constexpr uint32_t H = 0x80008000u;
    const uint32_t jl = j & mask;
    // (w + hm) & H: bit 15 / 31 set iff the low / high offset >= jl
    // (offsets and jl < 2^15: no borrow crosses a half)
    const uint32_t hm = H - jl * 0x10001u;
    uint32_t ge, lt;
    if constexpr (SLOTS == 3) {
      // 64-bit SWAR: fields (0x1000 | offset) - jl at bits 25 + 13k keep their
      // guard bit (37, 50, 63) iff offset >= jl; bits 0..24 are untouched
      const uint32_t ylo = jl << 25, yhi = jl * 0x80040u + (jl >> 7);
      uint32_t dlo, dhi;
      asm("sub.cc.u32 %0, %2, %4;\n\tsubc.u32 %1, %3, %5;" : "=r"(dlo), "=r"(dhi) : "r"(g.x), "r"(g.y), "r"(ylo),
          "r"(yhi));
      (void)dlo;
      ge = __popc(dhi & 0x80040020u);
      lt = 3u - ge;
      const unsigned long long w64 = ((unsigned long long)g.y << 32) | g.x;
      const uint32_t fv = (uint32_t)(w64 >> (lt < 3u ? 25u + 13u * lt : 63u));  // field lt
      knot = lt < 3u && (fv & 0xFFFu) == jl;
    } else if constexpr (SLOTS == 8) {
      rec12_count(g, jl, lt, knot);
      (void)ge;
    } else {
      uint32_t w;
      if constexpr (SLOTS == 6) {
        ge = __popc((g.y + hm) & H) + __popc((g.z + hm) & H) + __popc((g.w + hm) & H);
        const uint32_t l6 = SLOTS - ge;
        w = l6 < 2 ? g.y : (l6 < 4 ? g.z : g.w);
      } else {
        ge = __popc((g.y + hm) & H);
        w = g.y;
      }
      lt = SLOTS - ge;
      knot = lt < SLOTS && ((w >> ((lt & 1u) << 4)) & 0xFFFFu) == jl;
    }
    t = base_of(g) + lt;
    FSG_BOUND((j >> s) <= (r >> s) && (!knot || t < n1));
    if constexpr (OVF) {
      if (overflows(g) && lt == SLOTS) {  // past the last recorded knot of an overflowing super-bucket
        uint32_t lo = t, hi = base_of(G[(j >> s) + 1]);
        const uint32_t end = hi;
        FSG_BOUND(t <= end && end <= n1);
        while (lo < hi) {
          const uint32_t mid = (lo + hi) >> 1;
          if (F[mid] < jl) lo = mid + 1;
          else hi = mid;
        }
        t = lo;
        knot = lo < end && F[lo] == jl;
      }
    }
  }
  __device__ __forceinline__ int64_t operator()(T z) const {
    const uint32_t j = bucket(z);
    uint32_t t;
    bool knot;
    resolve(G[j >> s], j, t, knot);
    T xv = z;
    if (knot) xv = xat(t);
    return (int64_t)t - ((!knot || z < xv) ? 1 : 0);
  }
  // every record load of a group issued before the first is resolved
  template <int N, typename R>
  __device__ __forceinline__ void batch(const T (&z)[N], R (&o)[N]) const {
    // live-register bound (2-4 regs per record); the wide-field layouts (3
    // and 8 offsets) measure best two at a time (cfg2 470 -> 496, cfg5 N+1 =
    // 32769 403 -> 410 Gq/s; profiles/r01/tune_sparse_records.txt)
#ifndef FSG_REC_GROUP_WIDE
#define FSG_REC_GROUP_WIDE 2
#endif
    constexpr int GW = (SLOTS == 3 || SLOTS == 8) ? FSG_REC_GROUP_WIDE : FSG_REC_GROUP;
    constexpr int GR = N < GW ? N : GW;
#pragma unroll
    for (int g0 = 0; g0 < N; g0 += GR) {
      Rec g[GR];
      uint32_t j[GR];
#pragma unroll
      for (int q = 0; q < GR; ++q) {
        if (g0 + q >= N) break;
        j[q] = bucket(z[g0 + q]);
        g[q] = G[j[q] >> s];
      }
      if constexpr (XS) {
#pragma unroll
        for (int q = 0; q < GR; ++q) {
          if (g0 + q >= N) break;
          uint32_t t;
          bool knot;
          resolve(g[q], j[q], t, knot);
          T xv = z[g0 + q];
          if (knot) xv = xat<sizeof(R) == 4>(t);
          o[g0 + q] = (R)((int64_t)t - ((!knot || z[g0 + q] < xv) ? 1 : 0));
        }
      } else {  // X through L2: every X gather of the group in flight before the first is used
        uint32_t t[GR];
        bool knot[GR];
        T xv[GR];
#pragma unroll
        for (int q = 0; q < GR; ++q) {
          if (g0 + q >= N) break;
          resolve(g[q], j[q], t[q], knot[q]);
          xv[q] = z[g0 + q];
          if (knot[q]) xv[q] = xat(t[q]);
        }
#pragma unroll
        for (int q = 0; q < GR; ++q) {
          if (g0 + q >= N) break;
          o[g0 + q] = (R)((int64_t)t[q] - ((!knot[q] || z[g0 + q] < xv[q]) ? 1 : 0));
        }
      }
    }
  }
};

// Direct search (gap 1) over the count words of K (fill_count_words_kernel),
// staged in shared memory after X when X fits.  A word {mask, base} covers 16
// stripes of 2^k buckets (one k for the table) with a 2-bit knot count each.
// For bucket j: b = (j >> k) & 15, m = mask below bit 2b, and
//   t = base + popc(m) + popc(m & 0xAAAAAAAA)
// knots lie in earlier stripes -- all below z, the bucket function being
// monotone (direct.py:194-197) -- while knots of later stripes lie above it, so
// only the c = (mask >> 2b) & 3 knots X[t .. t+c-1] of the query's own stripe
// need comparing: the answer of batch.py:315-317 is t - 1 + #{X[t+e] <= z}.
// Common path (c <= 1): one predicated X load and one compare, as the rank
// directory does.  Rare path (c >= 2, or a flagged word whose counts
// saturated): a forward scan X[s], X[s+1], ... <= z from s = t (s = base for
// a flagged word), which stops at the first knot above z -- exact for any
// number of knots in a stripe, so correctness never depends on k; the
// planner picks the finest k that fits and reports how many queries go the
// rare way (uniformly drawn knots: ~lambda^2 / 2 of them at lambda knots per
// stripe).  A popcount decode instead of the group records' SWAR counts.
//
// XM = where the stripe's knot is compared: 1 = X staged in shared memory;
// 0 = X read through L2; 2 = X too large to stage but one byte per knot is:
// O[i] = knot i's bucket inside its stripe (k <= 8), staged after the words.
// A knot in a lower bucket than the query's lies below z and one in a higher
// bucket above it (monotone buckets again), so X itself is read -- through
// L2 -- only when both share a bucket (2^-k of the stripe's queries).
template <typename T, int XM>
struct CountWordProbe {
  const T* X;
  uint32_t xs, ws, os;  // shared addresses of X (XM 1), the words, the offsets (XM 2)
  T h, x0;
  uint32_t r, k, n1, smask;
  __device__ __forceinline__ CountWordProbe(const DevPlan<T>& p, unsigned char* smem) {
    n1 = (uint32_t)p.n1;
    X = p.x;
    // held in registers (volatile mov): ptxas would otherwise rebuild the
    // shared-window addresses in front of every load
    asm volatile("mov.u32 %0, %1;" : "=r"(xs) : "r"((uint32_t)__cvta_generic_to_shared(smem)));
    asm volatile("mov.u32 %0, %1;" : "=r"(ws) : "r"(xs + p.x_smem_bytes_aligned()));
    h = p.h;
    x0 = p.x0;
    r = (uint32_t)p.r;
    k = (uint32_t)p.sparse_shift;
    smask = (1u << k) - 1u;
    os = ws + 8u * ((r >> (k + kCountWordShift)) + 1u);
  }
  __device__ __forceinline__ uint32_t bucket(T z) const {
    uint32_t j = trunc_to<uint32_t>(mul_rn(sub_rn(z, x0), h));
    return j < r ? j : r;
  }
  __device__ __forceinline__ uint2 word(uint32_t j) const {
    uint2 g;
    const uint32_t a = ws + 8u * ((j >> k) >> kCountWordShift);
    FSG_BOUND(a + 8u - xs <= dyn_smem_bytes());
    asm("ld.shared.v2.u32 {%0, %1}, [%2];" : "=r"(g.x), "=r"(g.y) : "r"(a));
    return g;
  }
  __device__ __forceinline__ T xat(uint32_t t) const {
    FSG_BOUND(t < n1);
    if constexpr (XM == 1) {
      T v;
      if constexpr (sizeof(T) == 4) asm("ld.shared.f32 %0, [%1];" : "=f"(v) : "r"(xs + 4u * t));
      else asm("ld.shared.f64 %0, [%1];" : "=d"(v) : "r"(xs + 8u * t));
      return v;
    } else {
      return __ldg(X + t);
    }
  }
  __device__ __forceinline__ uint32_t oat(uint32_t t) const {
    uint32_t o;
    FSG_BOUND(t < n1 && os + t + 1u - xs <= dyn_smem_bytes());
    asm("ld.shared.u8 %0, [%1];" : "=r"(o) : "r"(os + t));
    return o;
  }
  // knots in earlier stripes -> t, knots in the query's stripe -> c
  __device__ __forceinline__ void resolve(const uint2& g, uint32_t j, uint32_t& t, uint32_t& c) const {
    const uint32_t b2 = ((j >> k) & 15u) * 2u;
    uint32_t below;
    asm("bmsk.clamp.b32 %0, 0, %1;" : "=r"(below) : "r"(b2));
    const uint32_t m = g.x & below;
    t = g.y + __popc(m) + __popc(m & 0xAAAAAAAAu);  // the flag bit rides along; flagged words go the rare way
    c = (g.x >> b2) & 3u;
  }
  __device__ __forceinline__ int64_t finish(const uint2& g, uint32_t j, uint32_t t, uint32_t c, T z) const {
    const bool flagged = (int32_t)g.y < 0;
    uint32_t res;
    bool rare = c > 1u || flagged;
    // the stripe's first knot (its offset byte / X[t]) through a predicated
    // load: a branch here would put a reconvergence region, and an exposed
    // load latency, around every query of the group
    const uint32_t take = (c != 0u && !flagged) ? 1u : 0u;
    FSG_BOUND(!take || t < n1);
    if constexpr (XM == 2) {
      const uint32_t jo = j & smask;
      uint32_t o = jo + 1u;  // no knot: neither below nor beside the query
      asm("{\n\t.reg .pred p;\n\tsetp.ne.u32 p, %2, 0;\n\t@p ld.shared.u8 %0, [%1];\n\t}" : "+r"(o) : "r"(os + t), "r"(take));
      res = t - (o < jo ? 0u : 1u);
      rare = rare || o == jo;
    } else {
      T xv = z;
      if constexpr (XM == 1) {
        if constexpr (sizeof(T) == 4)
          asm("{\n\t.reg .pred p;\n\tsetp.ne.u32 p, %2, 0;\n\t@p ld.shared.f32 %0, [%1];\n\t}" : "+f"(xv) : "r"(xs + 4u * t), "r"(take));
        else
          asm("{\n\t.reg .pred p;\n\tsetp.ne.u32 p, %2, 0;\n\t@p ld.shared.f64 %0, [%1];\n\t}" : "+d"(xv) : "r"(xs + 8u * t), "r"(take));
      } else {
        if constexpr (sizeof(T) == 4)
          asm("{\n\t.reg .pred p;\n\tsetp.ne.u32 p, %2, 0;\n\t@p ld.global.nc.f32 %0, [%1];\n\t}" : "+f"(xv) : "l"(X + t), "r"(take));
        else
          asm("{\n\t.reg .pred p;\n\tsetp.ne.u32 p, %2, 0;\n\t@p ld.global.nc.f64 %0, [%1];\n\t}" : "+d"(xv) : "l"(X + t), "r"(take));
      }
      res = t - ((take == 0u || z < xv) ? 1u : 0u);
    }
    if (rare) {
      if (XM == 2 && !flagged) {
        // the stripe's knots by their buckets; X decides only a shared bucket
        // (a gap-1 table holds one knot per bucket: nothing after it counts)
        const uint32_t jo = j & smask;
        res = t - 1u;
        for (uint32_t e = 0; e < c; ++e) {
          const uint32_t o = oat(t + e);
          if (o < jo) {
            ++res;
          } else {
            if (o == jo && xat(t + e) <= z) ++res;
            break;
          }
        }
      } else {  // scan the stripe's (a flagged word's) knots
        uint32_t e = flagged ? (g.y & ~kCountFlag) : t;
        while (e < n1 && xat(e) <= z) ++e;
        res = e - 1u;
      }
    }
    return (int64_t)(int32_t)res;
  }
  __device__ __forceinline__ int64_t operator()(T z) const {
    const uint32_t j = bucket(z);
    const uint2 g = word(j);
    uint32_t t, c;
    resolve(g, j, t, c);
    return finish(g, j, t, c, z);
  }
  // every word load of a group issued before the first is resolved
#ifndef FSG_COUNT_GROUP
#define FSG_COUNT_GROUP 4  // 1: 464, 2: 486, 4: 493 Gq/s on cfg2 (unroll 2)
#endif
  template <int N, typename R>
  __device__ __forceinline__ void batch(const T (&z)[N], R (&o)[N]) const {
    constexpr int G = N < FSG_COUNT_GROUP ? N : FSG_COUNT_GROUP;
#pragma unroll
    for (int g0 = 0; g0 < N; g0 += G) {
      uint2 g[G];
      uint32_t j[G];
#pragma unroll
      for (int q = 0; q < G; ++q) {
        if (g0 + q >= N) break;
        j[q] = bucket(z[g0 + q]);
        g[q] = word(j[q]);
      }
#pragma unroll
      for (int q = 0; q < G; ++q) {
        if (g0 + q >= N) break;
        uint32_t t, c;
        resolve(g[q], j[q], t, c);
        o[g0 + q] = (R)finish(g[q], j[q], t, c, z[g0 + q]);
      }
    }
  }
};

// RankProbe with a shared-memory hot window: directory words [w0, w0 + nw)
// and knots X[t0 .. t0 + nt) are staged (X window at smem offset 0, the
// directory window after it); lanes outside the window gather through L2.
// Same answers as RankProbe -- only where each word is read from differs.
template <typename T>
struct HotRankProbe {
  const T* X;
  const uint2* D;
  const T* Xs;
  const uint2* Ds;
  T h, x0;
  uint32_t r, w0, nw, t0, nt;
  uint64_t n1;
  __device__ __forceinline__ HotRankProbe(const DevPlan<T>& p, unsigned char* smem) {
    n1 = p.n1;
    X = p.x;
    D = p.rank;
    Xs = reinterpret_cast<const T*>(smem);
    Ds = reinterpret_cast<const uint2*>(smem + p.x_smem_bytes_aligned());
    h = p.h;
    x0 = p.x0;
    r = (uint32_t)p.r;
    w0 = p.hot_w0;
    nw = p.hot_nw;
    t0 = p.hot_t0;
    nt = p.hot_nt;
  }
  __device__ __forceinline__ int64_t operator()(T z) const {
    uint32_t j = trunc_to<uint32_t>(mul_rn(sub_rn(z, x0), h));
    j = j < r ? j : r;
    const uint32_t w = j >> 5, wl = w - w0;
    const uint2 d = wl < nw ? Ds[wl] : __ldg(D + w);
    const uint32_t b = j & 31u;
    const uint32_t t = d.y + __popc(d.x & ((1u << b) - 1u));
    const bool knot = (d.x >> b) & 1u;
    const uint32_t tl = t - t0;
    FSG_BOUND((j >> 5) <= (r >> 5) && (!knot || t < n1));
    T xv = z;  // any value: unused unless `knot`
    if (knot) xv = tl < nt ? Xs[tl] : __ldg(X + t);
    return (int64_t)t - ((!knot || z < xv) ? 1 : 0);
  }
  // Two phases over groups of queries, as RankProbe::batch: every directory
  // word of the group (window or L2) in flight before the first is used.
  template <int N, typename R>
  __device__ __forceinline__ void batch(const T (&z)[N], R (&o)[N]) const {
    constexpr int G = N < FSG_RANK_GROUP ? N : FSG_RANK_GROUP;
#pragma unroll
    for (int g0 = 0; g0 < N; g0 += G) {
      uint2 d[G];
      uint32_t b[G];
#pragma unroll
      for (int q = 0; q < G; ++q) {
        if (g0 + q >= N) break;
        uint32_t j = trunc_to<uint32_t>(mul_rn(sub_rn(z[g0 + q], x0), h));
        j = j < r ? j : r;
        const uint32_t w = j >> 5, wl = w - w0;
        b[q] = j & 31u;
        d[q] = wl < nw ? Ds[wl] : __ldg(D + w);
      }
#pragma unroll
      for (int q = 0; q < G; ++q) {
        if (g0 + q >= N) break;
        const uint32_t t = d[q].y + __popc(d[q].x & ((1u << b[q]) - 1u));
        const bool knot = (d[q].x >> b[q]) & 1u;
        const uint32_t tl = t - t0;
        FSG_BOUND(!knot || t < n1);
        T xv = z[g0 + q];
        if (knot) xv = tl < nt ? Xs[tl] : __ldg(X + t);
        o[g0 + q] = (R)((int64_t)t - ((!knot || z[g0 + q] < xv) ? 1 : 0));
      }
    }
  }
};

// Direct search (gap 1) over the zoned records of K (fill_zoned_kernel),
// staged in shared memory after a window X[t0, t0 + nt) of the knots.  The
// buckets are cut into nz = (R >> zs) + 1 zones of 2^zs; each zone takes the
// 8-B record form its own knot density needs (fs_plan_zoned), so a table
// whose density varies by orders of magnitude (cfg4's geometric knots) fits
// in shared memory where one record shift for the whole table cannot:
//   slot records  {24-bit base, three 13-bit offsets} per 2^s buckets,
//                 s <= 11, never more than three knots (no overflow path);
//   rank records  {32-bit knot mask, base} per 32 buckets.
// Zone descriptor (u32, nz <= 64 of them at the table head, so a warp's
// descriptor loads cost at most two wavefronts): (first record - (z <<
// (zs - s))) << 5 | rank << 4 | s, so record index = ((int)d >> 5) + (j >> s).
// K[j] = base + #{knots of the record below j} exactly, and
// bucket j holds knot K[j] iff its offset / mask bit says so; X is read only
// then, from the window or through L2.  Identical answers to
// DirectProbe<GAP=1> (batch.py:315-317).
//
// STRIPED (FS_SPARSE_ZONED_RANK, fs_build_zoned_rank): every zone in rank
// words whose 32 mask bits each stand for a stripe of 2^k buckets, k per zone
// (descriptor: zone-relative first record << 5 | rank flag | k; a word covers
// 2^(k+5) buckets).  The planner picks k so that no stripe holds two knots.
// With b = (j >> k) & 31: t = base + popc(mask below b) counts the knots in
// earlier stripes, whose buckets are below j, so X_i < z for all of them
// (the bucket function is monotone); knots in later stripes lie above z; and
// if stripe b holds a knot it is X[t], compared directly: the answer is
// t - (z < X[t]), else t - 1.  The same answers with a ~10-instruction decode
// (the slot form's SWAR count and field select are gone); the price is an X
// read whenever the query's stripe -- not its exact bucket -- holds a knot.
template <typename T, bool STRIPED = false>
struct ZonedProbe {
  const T* X;
  const unsigned char* xg;  // generic address of the X window
  uint32_t xs, zd, rc;      // shared addresses: X window, zone descriptors, records
  T h, x0;
  uint32_t r, zs, zmask, t0, nt;
  uint64_t n1, nrec;
  __device__ __forceinline__ ZonedProbe(const DevPlan<T>& p, unsigned char* smem) {
    n1 = p.n1;
    nrec = p.sparse_ndense;
    X = p.x;
    asm volatile("mov.u32 %0, %1;" : "=r"(xs) : "r"((uint32_t)__cvta_generic_to_shared(smem)));
    // the window's generic address held in a register (ptxas would otherwise
    // rebuild it from the CTA's shared window in front of every load)
    unsigned long long xgv;
    asm volatile("cvta.shared.u64 %0, %1;" : "=l"(xgv) : "l"((unsigned long long)xs));
    xg = reinterpret_cast<const unsigned char*>(xgv);
    zd = xs + p.x_smem_bytes_aligned();
    const uint32_t nz = (uint32_t)(p.r >> p.sparse_shift) + 1u;
    rc = zd + 4u * ((nz + 3u) & ~3u);
    h = p.h;
    x0 = p.x0;
    r = (uint32_t)p.r;
    zs = (uint32_t)p.sparse_shift;
    zmask = (1u << zs) - 1u;
    t0 = p.hot_t0;
    nt = p.hot_nt;
  }
  __device__ __forceinline__ uint32_t bucket(T z) const {
    uint32_t j = trunc_to<uint32_t>(mul_rn(sub_rn(z, x0), h));
    return j < r ? j : r;
  }
  __device__ __forceinline__ uint32_t desc(uint32_t j) const {
    uint32_t d;
    FSG_BOUND((j >> zs) <= (r >> zs) && zd + 4u * (j >> zs) - xs < dyn_smem_bytes());
    asm("ld.shared.u32 %0, [%1];" : "=r"(d) : "r"(zd + 4u * (j >> zs)));
    return d;
  }
  __device__ __forceinline__ uint2 rec(uint32_t j, uint32_t d) const {
    uint2 g;
    // descriptors are zone-relative
    const uint32_t idx = (uint32_t)((int32_t)d >> 5) + (STRIPED ? (j >> (d & 15u)) >> 5 : j >> (d & 15u));
    const uint32_t a = rc + 8u * idx;
    FSG_BOUND(idx < nrec && a + 8u - xs <= dyn_smem_bytes());
    asm("ld.shared.v2.u32 {%0, %1}, [%2];" : "=r"(g.x), "=r"(g.y) : "r"(a));
    return g;
  }
  // Both record forms decoded branch-free and selected by the zone's rank
  // flag: lanes of one warp fall in zones of either form (cfg4's query mix
  // is half dense, half sparse), and a divergent branch would issue both
  // decodes plus its reconvergence overhead anyway.
  static __device__ __forceinline__ void resolve(const uint2& g, uint32_t d, uint32_t j, uint32_t& t, bool& knot) {
    if constexpr (STRIPED) {
      const uint32_t b = (j >> (d & 15u)) & 31u;
      uint32_t below;
      asm("bmsk.clamp.b32 %0, 0, %1;" : "=r"(below) : "r"(b));
      t = g.y + __popc(g.x & below);
      knot = (g.x >> b) & 1u;
      return;
    }
    uint32_t smask;  // the low s bits (bmsk: one instruction)
    asm("bmsk.clamp.b32 %0, 0, %1;" : "=r"(smask) : "r"(d & 15u));
    const uint32_t jl = j & smask;
    // rank view: {mask, base} (jl < 32 in rank zones; in slot zones the view
    // is discarded, and PTX clamps the counts >= 32, so no mask of jl)
    uint32_t below, kr;
    asm("bmsk.clamp.b32 %0, 0, %1;" : "=r"(below) : "r"(jl));
    asm("shr.b32 %0, %1, %2;" : "=r"(kr) : "r"(g.x), "r"(jl));
    const uint32_t tr = g.y + __popc(g.x & below);
    kr &= 1u;
    // slot view: 64-bit SWAR over the three fields 0x1000 | offset at bits
    // 25 + 13k (guard bits 37, 50, 63 survive iff offset >= jl)
    const uint32_t ylo = jl << 25, yhi = jl * 0x80040u + (jl >> 7);
    uint32_t dlo, dhi;
    asm("sub.cc.u32 %0, %2, %4;\n\tsubc.u32 %1, %3, %5;" : "=r"(dlo), "=r"(dhi) : "r"(g.x), "r"(g.y), "r"(ylo),
        "r"(yhi));
    (void)dlo;
    const uint32_t lt = 3u - __popc(dhi & 0x80040020u);
    const unsigned long long w64 = ((unsigned long long)g.y << 32) | g.x;
    const uint32_t fv = (uint32_t)(w64 >> (lt < 3u ? 25u + 13u * lt : 63u));
    const uint32_t ks = (lt < 3u && (fv & 0xFFFu) == jl) ? 1u : 0u;
    const uint32_t ts = (g.x & 0xFFFFFFu) + lt;
    uint32_t kb;
    asm("{\n\t.reg .pred p;\n\tsetp.ne.u32 p, %4, 0;\n\tselp.b32 %0, %2, %3, p;\n\tselp.b32 %1, %5, %6, p;\n\t}"
        : "=r"(t), "=r"(kb)
        : "r"(tr), "r"(ts), "r"(d & kZonedRankFlag), "r"(kr), "r"(ks));
    knot = kb != 0;
  }
  // X[t] if `knot`, else z: one predicated generic load from the staged
  // window or global memory (no branch between the two)
  __device__ __forceinline__ T xsel(uint32_t t, bool knot, T z) const {
    const uint32_t tl = t - t0;
    FSG_BOUND(!knot || t < n1);
    const T* p = tl < nt ? reinterpret_cast<const T*>(xg) + tl : X + t;
    T v = z;
    if constexpr (sizeof(T) == 4)
      asm("{\n\t.reg .pred p;\n\tsetp.ne.u32 p, %2, 0;\n\t@p ld.f32 %0, [%1];\n\t}" : "+f"(v) : "l"(p), "r"((uint32_t)knot));
    else
      asm("{\n\t.reg .pred p;\n\tsetp.ne.u32 p, %2, 0;\n\t@p ld.f64 %0, [%1];\n\t}" : "+d"(v) : "l"(p), "r"((uint32_t)knot));
    return v;
  }
  __device__ __forceinline__ int64_t operator()(T z) const {
    const uint32_t j = bucket(z);
    const uint32_t d = desc(j);
    uint32_t t;
    bool knot;
    resolve(rec(j, d), d, j, t, knot);
    const T xv = xsel(t, knot, z);
    return (int64_t)t - (int64_t)((uint32_t)!knot | (uint32_t)(z < xv));
  }
  // descriptors of a group, then its records, then the resolves: every load
  // of a phase in flight before the first is consumed
#ifndef FSG_ZONED_GROUP
#define FSG_ZONED_GROUP 2  // cfg4: 1 452, 2 465, 3 457, 4 450, 8 436 Gq/s
#endif
  template <int N, typename R>
  __device__ __forceinline__ void batch(const T (&z)[N], R (&o)[N]) const {
    constexpr int G = N < FSG_ZONED_GROUP ? N : FSG_ZONED_GROUP;
#pragma unroll
    for (int g0 = 0; g0 < N; g0 += G) {
      uint32_t j[G], d[G];
      uint2 g[G];
#pragma unroll
      for (int q = 0; q < G; ++q) {
        if (g0 + q >= N) break;
        j[q] = bucket(z[g0 + q]);
        d[q] = desc(j[q]);
      }
#pragma unroll
      for (int q = 0; q < G; ++q) {
        if (g0 + q >= N) break;
        g[q] = rec(j[q], d[q]);
      }
#pragma unroll
      for (int q = 0; q < G; ++q) {
        if (g0 + q >= N) break;
        uint32_t t;
        bool knot;
        resolve(g[q], d[q], j[q], t, knot);
        const T xv = xsel(t, knot, z[g0 + q]);
        o[g0 + q] = (R)((int64_t)t - (int64_t)((uint32_t)!knot | (uint32_t)(z[g0 + q] < xv)));
      }
    }
  }
};

// Cache-fused records: {u32 idx, f32 val} (8 B) / {u32 idx, u32 pad, f64 val}
// (16 B), direct.py:39-44.  One gather resolves the query.
template <typename T, typename J, bool RS>
struct CacheProbe;

template <typename J, bool RS>
struct CacheProbe<float, J, RS> {
  const uint2* R;
  float h, x0;
  J r;
  __device__ __forceinline__ CacheProbe(const DevPlan<float>& p, unsigned char* smem) {
    R = RS ? reinterpret_cast<const uint2*>(smem) : static_cast<const uint2*>(p.table);
    h = p.h;
    x0 = p.x0;
    r = (J)p.r;
  }
  __device__ __forceinline__ int64_t operator()(float z) const {
    J j = trunc_to<J>(mul_rn(sub_rn(z, x0), h));
    j = j < r ? j : r;
    const uint2 rec = tload<RS>(R, j);
    return (int64_t)rec.x - (z < __uint_as_float(rec.y) ? 1 : 0);
  }
};

template <typename J, bool RS>
struct CacheProbe<double, J, RS> {
  const double2* R;
  double h, x0;
  J r;
  __device__ __forceinline__ CacheProbe(const DevPlan<double>& p, unsigned char* smem) {
    R = RS ? reinterpret_cast<const double2*>(smem) : static_cast<const double2*>(p.table);
    h = p.h;
    x0 = p.x0;
    r = (J)p.r;
  }
  __device__ __forceinline__ int64_t operator()(double z) const {
    J j = trunc_to<J>(mul_rn(sub_rn(z, x0), h));
    j = j < r ? j : r;
    const double2 rec = tload<RS>(R, j);
    const uint32_t idx = (uint32_t)(unsigned long long)__double_as_longlong(rec.x);
    return (int64_t)idx - (z < rec.y ? 1 : 0);
  }
};

// Branch-free bit-setting search over the right-padded array (Alg 3).
// The first `top_bits` levels read a shared-memory copy of the nodes those
// levels can touch; deeper levels gather from global.  With top_bits ==
// pbits the whole padded array is in shared memory.
//
// Shared layout of the top levels (filled by the prologue), three regions:
//   P1  levels [0, l1)       level order: level l's 2^l candidates
//                            r = (m << (p-l)) | 2^(p-1-l) at [2^l - 1, 2^(l+1) - 1).
//                            In the sorted padded array every node of a level
//                            l <= 7 shares one bank; in level order they are
//                            consecutive words (l1 <= 6: at most 32 of them,
//                            conflict-free).
//   R   levels [l1, l2)      level order, each node replicated 32 times and
//                            interleaved (word = node * 32 + copy): lane c reads
//                            copy c, always bank c, so these levels are
//                            conflict-free for random queries.
//   P2  levels [l2, top)     level order again (too large to replicate).
// In every region a node is carried as its shared-window address, and the
// child step is a' = 2a + (z >= node ? c2 : c1) with region constants (the
// regions are stacked in level order, which makes c1 / c2 level-independent):
// one LDS, one compare, one select, one 3-input add per level.  Same
// comparisons, same values as binsearch.py:72-86.
// Bytes of bitset2's staged f32 shadow region (levels [0, l1) plain, [l1, l2)
// in 32 copies, [l2, l3) in 16, [l3, top) plain; 4-B words), 16-B aligned:
// the f64 plane follows it.
__host__ __device__ __forceinline__ uint32_t b2_shadow_bytes(int top, int l1, int l2, int l3) {
  const uint32_t words = ((1u << l1) - 1) + ((1u << l2) - (1u << l1)) * 32 + ((1u << l3) - (1u << l2)) * 16 +
                         ((1u << top) - (1u << l3));
  return (4 * words + 15) & ~15u;
}

template <typename T, bool TOP, bool DEEP = false, bool SHADOW = false>
struct Bitset2Probe {
  // f64 partitions stage their top levels as f32 shadow keys (RN of each
  // key, same region layout as f32: one bank per node instead of two) plus an
  // exact f64 plane in plain level order.  RN is monotone, so z32 > k32
  // implies z > k and z32 < k32 implies z < k: every left turn of the shadow
  // walk is exact, and a right turn can only be wrong on a tie z32 == k32.
  // The right-turn keys increase along the walk, so one exact check of the
  // last one (the node at the final prefix, z >= X[prefix]) validates the
  // whole walk; the rare failure re-descends exactly over the f64 plane.
  static constexpr bool kShadow = sizeof(T) == 8 && SHADOW;
  using K = std::conditional_t<kShadow, float, T>;  // staged key type
  const K* top;
  const double* plane;  // kShadow: exact keys of the staged levels, plain level order
  const T* xpad;
  const char* deep;  // subtree records of the global levels (fs_build_b2_deep) or NULL
  int pbits, top_bits, l1, l2, l3, deep_k;
  __device__ __forceinline__ Bitset2Probe(const DevPlan<T>& p, unsigned char* smem) {
    top = reinterpret_cast<const K*>(smem);
    plane = reinterpret_cast<const double*>(smem + b2_shadow_bytes(p.top_bits, p.b2_l1, p.b2_l2, p.b2_l3));
    xpad = static_cast<const T*>(p.table);
    pbits = p.pbits;
    top_bits = TOP ? p.top_bits : 0;
    l1 = TOP ? p.b2_l1 : 0;
    l2 = TOP ? p.b2_l2 : 0;
    l3 = TOP ? p.b2_l3 : 0;
    deep = DEEP ? static_cast<const char*>(p.b2_deep) : nullptr;
    deep_k = DEEP ? p.b2_deep_k : 0;
  }
  // One 32-B subtree record: 8 f32 / 4 f64 values, BFS order.
  struct Rec {
    T v[32 / sizeof(T)];
  };
  static __device__ __forceinline__ Rec ld_rec(const char* p) {
    Rec r;
    if constexpr (sizeof(T) == 4) {
      asm volatile("ld.global.nc.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                   : "=f"(r.v[0]), "=f"(r.v[1]), "=f"(r.v[2]), "=f"(r.v[3]), "=f"(r.v[4]), "=f"(r.v[5]),
                     "=f"(r.v[6]), "=f"(r.v[7])
                   : "l"(p));
    } else {
      asm volatile("ld.global.nc.v4.f64 {%0,%1,%2,%3}, [%4];"
                   : "=d"(r.v[0]), "=d"(r.v[1]), "=d"(r.v[2]), "=d"(r.v[3])
                   : "l"(p));
    }
    return r;
  }
  // k_c levels of one record, selects only (no local-memory indexing):
  // returns the k_c decision bits, first decision in the high bit.
  static __device__ __forceinline__ uint32_t walk_rec(const Rec& r, T z, int kc) {
    const uint32_t b0 = z >= r.v[0];
    const T v1 = b0 ? r.v[2] : r.v[1];
    const uint32_t b1 = z >= v1;
    if constexpr (sizeof(T) == 4) {
      if (kc == 3) {
        const T v2 = b0 ? (b1 ? r.v[6] : r.v[5]) : (b1 ? r.v[4] : r.v[3]);
        return (b0 << 2) | (b1 << 1) | (uint32_t)(z >= v2);
      }
    }
    return (b0 << 1) | b1;
  }
  static __device__ __forceinline__ void prologue(const DevPlan<T>& p, unsigned char* smem) {
    if constexpr (TOP) {
      K* dst = reinterpret_cast<K*>(smem);
      const T* src = static_cast<const T*>(p.table);
      const uint32_t n1w = (1u << p.b2_l1) - 1;                                   // P1 words
      const uint32_t nrw = ((1u << p.b2_l2) - (1u << p.b2_l1)) * 32u;            // R words
      const uint32_t nhw = ((1u << p.b2_l3) - (1u << p.b2_l2)) * 16u;            // H words
      const uint32_t total = n1w + nrw + nhw + ((1u << p.top_bits) - (1u << p.b2_l3));  // + P2 words
      for (uint32_t w = threadIdx.x; w < total; w += blockDim.x) {
        // level-order node index of word w (P1 | R: 32 copies per node |
        // H: 16 copies per node | P2)
        const uint32_t node = w < n1w               ? w
                              : w < n1w + nrw       ? n1w + ((w - n1w) >> 5)
                              : w < n1w + nrw + nhw ? (1u << p.b2_l2) - 1 + ((w - n1w - nrw) >> 4)
                                                    : (1u << p.b2_l3) - 1 + (w - n1w - nrw - nhw);
        const int l = 31 - __clz(node + 1);
        const uint32_t m = node + 1 - (1u << l);
        const uint64_t r = ((uint64_t)m << (p.pbits - l)) | (1ull << (p.pbits - 1 - l));
        if constexpr (kShadow) dst[w] = __double2float_rn(__ldg(src + r));
        else dst[w] = __ldg(src + r);
      }
      if constexpr (kShadow) {  // the exact plane: node n of level l at n, plain level order
        double* pl = reinterpret_cast<double*>(smem + b2_shadow_bytes(p.top_bits, p.b2_l1, p.b2_l2, p.b2_l3));
        for (uint32_t n = threadIdx.x; n < (1u << p.top_bits) - 1; n += blockDim.x) {
          const int l = 31 - __clz(n + 1);
          const uint32_t m = n + 1 - (1u << l);
          pl[n] = __ldg(src + (((uint64_t)m << (p.pbits - l)) | (1ull << (p.pbits - 1 - l))));
        }
      }
      __syncthreads();
    }
  }
  static __device__ __forceinline__ K lds(uint32_t a) {
    K v;
    if constexpr (sizeof(K) == 4) asm volatile("ld.shared.f32 %0, [%1];" : "=f"(v) : "r"(a));
    else asm volatile("ld.shared.f64 %0, [%1];" : "=d"(v) : "r"(a));
    return v;
  }
#ifndef FSG_B2_PIPE_MIX
#define FSG_B2_PIPE_MIX 1
#endif
  // One level: a' = 2a + (z >= node(a) ? c2 : c1).  The compare is an ALU
  // op; the rest is either ALU (select + 3-input add) or, through an opaque
  // multiplier ptxas cannot strength-reduce, the FMA pipe's IMAD.  ncu shows
  // the all-ALU form saturating the ALU pipe (91%) with FMA idle (6%);
  // alternating two forms across the lockstep queries balances the pipes
  // (f32; profiles/r01/tune_bitset2_pipes.txt):
  //   FORM 0: FSETP, SEL, IMAD            (ALU 2, FMA 1)
  //   FORM 1: FSETP, IMAD, predicated IMAD (ALU 1, FMA 2)
  template <int FORM>
  static __device__ __forceinline__ uint32_t step(uint32_t a, K z, uint32_t c1, uint32_t c2, uint32_t two,
                                                  uint32_t one) {
    const K v = lds(a);
#if FSG_B2_PIPE_MIX
    // f64 compares issue on the FP64 pipe, which leaves the ALU room: the
    // all-ALU form measures best there
    if constexpr (sizeof(K) == 8) {
      return a + a + (z >= v ? c2 : c1);
    } else {
      uint32_t r;
      if constexpr (FORM == 0) {
        asm("mad.lo.u32 %0, %1, %2, %3;" : "=r"(r) : "r"(a), "r"(two), "r"(z >= v ? c2 : c1));
      } else {
        asm("mad.lo.u32 %0, %1, %2, %3;" : "=r"(r) : "r"(a), "r"(two), "r"(c1));
        asm("{\n\t.reg .pred p;\n\tsetp.ge.f32 p, %1, %2;\n\t@p mad.lo.u32 %0, %3, %4, %0;\n\t}"
            : "+r"(r) : "f"(z), "f"(v), "r"(c2 - c1), "r"(one));
      }
      return r;
    }
#else
    return a + a + (z >= v ? c2 : c1);
#endif
  }
  // Levels [0, top_bits) for N queries in lockstep; returns, per query, the
  // bit prefix i (the index reached after top_bits levels, low bits clear).
  template <int N>
  __device__ __forceinline__ void descend_top(const K (&z)[N], uint32_t (&i)[N]) const {
    constexpr uint32_t sz = sizeof(K);
    const uint32_t base = (uint32_t)__cvta_generic_to_shared(top);
    uint32_t two, one;  // opaque to ptxas: keeps the IMADs on the FMA pipe
    asm volatile("mov.u32 %0, 2;" : "=r"(two));
    asm volatile("mov.u32 %0, 1;" : "=r"(one));
    uint32_t a[N];
#pragma unroll
    for (int q = 0; q < N; ++q) a[q] = base;
    {  // P1: a = base + s * sz
      const uint32_t c1 = sz - base, c2 = 2 * sz - base;
      for (int l = 0; l < l1; ++l) {
#pragma unroll
        for (int q = 0; q + 1 < N; q += 2) {
          a[q] = step<0>(a[q], z[q], c1, c2, two, one);
          a[q + 1] = step<1>(a[q + 1], z[q + 1], c1, c2, two, one);
        }
        if constexpr (N & 1) a[N - 1] = step<0>(a[N - 1], z[N - 1], c1, c2, two, one);
      }
    }
    uint32_t b2 = base, s0 = 0;  // the P2 region: a = b2 + (s - s0) * sz
    if (l2 > l1) {  // R: a = B_l + m * 32sz + lane * sz, B_l = rb + (2^l - 2^l1) * 32sz
      const uint32_t lane = threadIdx.x & 31u;
      const uint32_t rb = base + ((1u << l1) - 1) * sz;
      const uint32_t c1 = (1u << l1) * 32u * sz - rb - lane * sz, c2 = c1 + 32u * sz;
#pragma unroll
      for (int q = 0; q < N; ++q) a[q] = rb + ((a[q] - base) / sz - ((1u << l1) - 1)) * 32u * sz + lane * sz;
      for (int l = l1; l < l2; ++l) {
#pragma unroll
        for (int q = 0; q + 1 < N; q += 2) {
          a[q] = step<0>(a[q], z[q], c1, c2, two, one);
          a[q + 1] = step<1>(a[q + 1], z[q + 1], c1, c2, two, one);
        }
        if constexpr (N & 1) a[N - 1] = step<0>(a[N - 1], z[N - 1], c1, c2, two, one);
      }
      b2 = rb + ((1u << l2) - (1u << l1)) * 32u * sz;  // B_l2: H (or P2) starts here
      s0 = (1u << l2) - 1;
      if (l3 > l2) {  // H: a = B_l + m * 16sz + (lane & 15) * sz, B_l = b2 + (2^l - 2^l2) * 16sz
        const uint32_t lh = lane & 15u;
#pragma unroll
        for (int q = 0; q < N; ++q) a[q] = b2 + (a[q] - b2 - lane * sz) / (32u * sz) * (16u * sz) + lh * sz;
        const uint32_t h1 = (1u << l2) * 16u * sz - b2 - lh * sz, h2 = h1 + 16u * sz;
        for (int l = l2; l < l3; ++l) {
#pragma unroll
          for (int q = 0; q + 1 < N; q += 2) {
            a[q] = step<0>(a[q], z[q], h1, h2, two, one);
            a[q + 1] = step<1>(a[q + 1], z[q + 1], h1, h2, two, one);
          }
          if constexpr (N & 1) a[N - 1] = step<0>(a[N - 1], z[N - 1], h1, h2, two, one);
        }
        const uint32_t b3 = b2 + ((1u << l3) - (1u << l2)) * 16u * sz;  // B_l3: P2 starts here
#pragma unroll
        for (int q = 0; q < N; ++q) a[q] = b3 + (a[q] - b3 - lh * sz) / (16u * sz) * sz;
        b2 = b3;
        s0 = (1u << l3) - 1;
      } else {
#pragma unroll
        for (int q = 0; q < N; ++q) a[q] = b2 + (a[q] - b2 - lane * sz) / (32u * sz) * sz;
      }
    }
    {  // P2 (or the rest of P1 when nothing is replicated)
      const uint32_t c1 = (s0 + 1) * sz - b2, c2 = c1 + sz;
      for (int l = l2 > l1 ? (l3 > l2 ? l3 : l2) : l1; l < top_bits; ++l) {
#pragma unroll
        for (int q = 0; q + 1 < N; q += 2) {
          a[q] = step<0>(a[q], z[q], c1, c2, two, one);
          a[q + 1] = step<1>(a[q + 1], z[q + 1], c1, c2, two, one);
        }
        if constexpr (N & 1) a[N - 1] = step<0>(a[N - 1], z[N - 1], c1, c2, two, one);
      }
    }
#pragma unroll
    for (int q = 0; q < N; ++q) {
      i[q] = ((a[q] - b2) / sz + s0 - ((1u << top_bits) - 1)) << (pbits - top_bits);
      FSG_BOUND((i[q] >> (pbits - top_bits)) < (1u << top_bits));
    }
  }
  // N queries descend in lockstep: N independent smem/L2 loads per level.
  template <int N, typename R>
  __device__ __forceinline__ void batch(const T (&z)[N], R (&o)[N]) const {
    uint32_t s[N];
#pragma unroll
    for (int q = 0; q < N; ++q) s[q] = 0;
    int lvl = top_bits;
    if constexpr (TOP && kShadow) {
      float zk[N];
#pragma unroll
      for (int q = 0; q < N; ++q) zk[q] = __double2float_rn(z[q]);
      descend_top<N>(zk, s);
      const int lo = pbits - top_bits;  // s: prefix << lo
#pragma unroll
      for (int q = 0; q < N; ++q) {
        // the last right turn's node: level pbits - 1 - ctz(s), prefix above it
        bool ok = true;
        if (s[q]) {
          const int b = __ffs(s[q]) - 1;
          const int l = pbits - 1 - b;
          FSG_BOUND(l < top_bits && (s[q] >> (b + 1)) < (1u << l));
          ok = z[q] >= plane[(1u << l) - 1 + (s[q] >> (b + 1))];
        }
        if (!ok) {  // a tie went right wrongly: redo the staged levels exactly
          uint32_t i = 0;
          for (int l = 0; l < top_bits; ++l) i = 2 * i + (z[q] >= plane[(1u << l) - 1 + i] ? 1u : 0u);
          s[q] = i << lo;
        }
      }
    } else if constexpr (TOP) {
      descend_top<N>(z, s);
    }
    if constexpr (DEEP) {
      {  // global levels in k-level chunks: one 32-B gather per chunk
        uint64_t off = 0;
        for (; pbits - lvl >= 2; ) {
          const int kc = pbits - lvl < deep_k ? pbits - lvl : deep_k;
          const int sh = pbits - lvl;
          constexpr int G = N < FSG_B2_DEEP_GROUP ? N : FSG_B2_DEEP_GROUP;  // records in flight per group (32 B each)
#pragma unroll
          for (int g0 = 0; g0 < N; g0 += G) {
            Rec r[G];
#pragma unroll
            for (int q = 0; q < G; ++q)
              if (g0 + q < N) {
                FSG_BOUND((s[g0 + q] >> sh) < (1u << lvl));
                r[q] = ld_rec(deep + off + (uint64_t)(s[g0 + q] >> sh) * 32);
              }
#pragma unroll
            for (int q = 0; q < G; ++q)
              if (g0 + q < N) s[g0 + q] |= walk_rec(r[q], z[g0 + q], kc) << (sh - kc);
          }
          off += (32ull << lvl);
          lvl += kc;
        }
      }
    }
    for (; lvl < pbits; ++lvl) {
      const uint32_t bit = 1u << (pbits - 1 - lvl);
#pragma unroll
      for (int q = 0; q < N; ++q) {
        const uint32_t r = s[q] | bit;
        FSG_BOUND(r < (1u << pbits));
        if (z[q] >= __ldg(xpad + r)) s[q] = r;
      }
    }
#pragma unroll
    for (int q = 0; q < N; ++q) o[q] = (R)s[q];
  }
  __device__ __forceinline__ int64_t operator()(T z) const {
    const T zz[1] = {z};
    int64_t o[1];
    batch<1, int64_t>(zz, o);
    return o[0];
  }
};

// The other comparison kernels of batch.ALGORITHMS, on X in smem or global.
template <typename T, int ALGO, bool XS>
struct CompareProbe {
  const T* X;
  uint32_t n;
  int pbits;
  uint32_t F, S, Jc;
  // Sorted X in shared memory is stored XOR-swizzled within 128-B rows:
  // element i sits at i ^ (hash(i >> R) & (2^R - 1)).  The searches probe
  // elements 2^k apart, which in plain order share one bank (up to 32-way
  // conflicts, ~63 G queries/s on cfg3); swizzled they spread over the
  // banks.  The Eytzinger tree is already in level order and is not swizzled.
  static constexpr bool kSwz = XS && ALGO != 5;
  static __device__ __forceinline__ uint32_t swz(uint32_t i) {
    constexpr int R = sizeof(T) == 4 ? 5 : 4;  // elements per 128-B row: 2^R
    const uint32_t hi = i >> R;
    return i ^ ((hi ^ (hi >> R) ^ (hi >> (2 * R)) ^ (hi >> (3 * R))) & ((1u << R) - 1));
  }
  __device__ __forceinline__ T x(uint32_t i) const {
    if constexpr (kSwz) return X[swz(i)];
    else return tload<XS>(X, i);
  }
  static __device__ __forceinline__ void prologue(const DevPlan<T>& p, unsigned char* smem) {
    if constexpr (kSwz) {
      T* dst = reinterpret_cast<T*>(smem);
      for (uint32_t i = threadIdx.x; i < p.n1; i += blockDim.x) dst[swz(i)] = __ldg(p.x + i);
      __syncthreads();
    }
  }
  __device__ __forceinline__ CompareProbe(const DevPlan<T>& p, unsigned char* smem) {
    X = XS ? reinterpret_cast<const T*>(smem)
           : (ALGO == 5 ? static_cast<const T*>(p.table) : p.x);
    n = (uint32_t)(p.n1 - 1);
    pbits = p.pbits;
    F = p.off_f;
    S = p.off_s;
    Jc = p.off_j;
  }
  __device__ __forceinline__ int64_t operator()(T z) const {
    if constexpr (ALGO == 0) {  // classic, binsearch.py:48-57
      uint32_t low = 0, high = n;
      while (high - low > 1) {
        const uint32_t mid = (low + high) >> 1;
        if (z < x(mid)) high = mid;
        else low = mid;
      }
      return low;
    } else if constexpr (ALGO == 1) {  // bitset1, binsearch.py:60-69
      uint32_t i = 0;
      for (uint32_t k = 1u << (pbits - 1); k; k >>= 1) {
        const uint32_t r = i | k;
        if (r < n && z >= x(r)) i = r;
      }
      return i;
    } else if constexpr (ALGO == 3) {  // bitset3, binsearch.py:89-99
      uint32_t i = 0;
      for (uint32_t k = 1u << (pbits - 1); k; k >>= 1) {
        const uint32_t r = i | k;
        const uint32_t w = r < n ? r : n;
        if (z >= x(w)) i = r;
      }
      return i;
    } else if constexpr (ALGO == 4) {  // offset, binsearch.py:102-114
      uint32_t i = z >= x(F) ? F : 0;
      uint32_t s = S;
      for (uint32_t it = 0; it < Jc; ++it) {
        const uint32_t half = s >> 1;
        uint32_t f = i + half;
        f = f < n ? f : n;  // never binds in domain; keeps bad lanes in bounds
        if (z >= x(f)) i = f;
        s -= half;
      }
      return i;
    } else {  // eytzinger, eytzinger.py:84-89 (X points at the tree)
      uint64_t k = 1;
      for (int l = 0; l < pbits; ++l) k = 2 * k + (z >= tload<XS>(X, k - 1) ? 1 : 0);
      return (int64_t)k - (int64_t(1) << pbits) - 1;
    }
  }
  // N queries in lockstep (independent load chains per step), the same
  // comparisons per query as operator(); classic keeps one query at a time
  // (its masked lockstep measured 15% slower).
  template <int N, typename R>
  __device__ __forceinline__ void batch(const T (&z)[N], R (&o)[N]) const {
    if constexpr (ALGO == 0) {  // data-dependent trip count: one query at a time measures best
#pragma unroll
      for (int q = 0; q < N; ++q) o[q] = (R)(*this)(z[q]);
    } else if constexpr (ALGO == 1 || ALGO == 3) {
      uint32_t i[N];
#pragma unroll
      for (int q = 0; q < N; ++q) i[q] = 0;
      for (uint32_t k = 1u << (pbits - 1); k; k >>= 1) {
#pragma unroll
        for (int q = 0; q < N; ++q) {
          const uint32_t r = i[q] | k;
          if constexpr (ALGO == 1) {
            if (r < n && z[q] >= x(r)) i[q] = r;
          } else {
            if (z[q] >= x(r < n ? r : n)) i[q] = r;
          }
        }
      }
#pragma unroll
      for (int q = 0; q < N; ++q) o[q] = (R)i[q];
    } else if constexpr (ALGO == 4) {
      uint32_t i[N];
      const T xf = x(F);
#pragma unroll
      for (int q = 0; q < N; ++q) i[q] = z[q] >= xf ? F : 0;
      uint32_t s = S;
      for (uint32_t it = 0; it < Jc; ++it) {
        const uint32_t half = s >> 1;
#pragma unroll
        for (int q = 0; q < N; ++q) {
          uint32_t f = i[q] + half;
          f = f < n ? f : n;
          if (z[q] >= x(f)) i[q] = f;
        }
        s -= half;
      }
#pragma unroll
      for (int q = 0; q < N; ++q) o[q] = (R)i[q];
    } else {
      uint64_t k[N];
#pragma unroll
      for (int q = 0; q < N; ++q) k[q] = 1;
      for (int l = 0; l < pbits; ++l) {
#pragma unroll
        for (int q = 0; q < N; ++q) k[q] = 2 * k[q] + (z[q] >= tload<XS>(X, k[q] - 1) ? 1 : 0);
      }
#pragma unroll
      for (int q = 0; q < N; ++q) o[q] = (R)((int64_t)k[q] - (int64_t(1) << pbits) - 1);
    }
  }
};

// ---------------------------------------------------------------------------
// Streaming driver
// ---------------------------------------------------------------------------
// Query groups: VW consecutive queries per vector access.  VW = 4 (16-B f32
// / 32-B f64 loads) everywhere; f32 queries with int32 outputs may use VW = 8
// (one 32-B load and one 32-B store per group; FSG_F32_VW8).
template <typename T, int VW> struct VecLoad;
template <> struct VecLoad<float, 4> {
  static constexpr uint32_t kAlign = 16;
  float v[4];
  __device__ __forceinline__ void load(const float* p) {
    float4 a = ld_stream(reinterpret_cast<const float4*>(p));
    v[0] = a.x; v[1] = a.y; v[2] = a.z; v[3] = a.w;
  }
};
template <> struct VecLoad<float, 8> {
  static constexpr uint32_t kAlign = 32;
  float v[8];
  __device__ __forceinline__ void load(const float* p) {
    asm volatile("ld.global.nc.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=f"(v[0]), "=f"(v[1]), "=f"(v[2]), "=f"(v[3]), "=f"(v[4]), "=f"(v[5]), "=f"(v[6]), "=f"(v[7])
                 : "l"(p));
  }
};
// f64 groups are one 32-B load (LDG.E.256; the head peel aligns them to
// 32 B): two 16-B halves per lane would touch twice the L1 lines per
// instruction (16 wavefronts per warp's 1 KB instead of 8; ncu on cfg2).
#ifndef FSG_F64_LD256
#define FSG_F64_LD256 1
#endif
template <> struct VecLoad<double, 4> {
  static constexpr uint32_t kAlign = FSG_F64_LD256 ? 32 : 16;
  double v[4];
  __device__ __forceinline__ void load(const double* p) {
#if FSG_F64_LD256
    asm volatile("ld.global.nc.v4.f64 {%0,%1,%2,%3}, [%4];"
                 : "=d"(v[0]), "=d"(v[1]), "=d"(v[2]), "=d"(v[3]) : "l"(p));
#else
    double2 a = ld_stream(reinterpret_cast<const double2*>(p));
    double2 b = ld_stream(reinterpret_cast<const double2*>(p) + 1);
    v[0] = a.x; v[1] = a.y; v[2] = b.x; v[3] = b.y;
#endif
  }
};

// Output groups: vec = 2 when the group is 32-B aligned, 1 when 16-B
// aligned, 0 otherwise (scalar stores).
template <int VW>
__device__ __forceinline__ void store_group(int32_t* p, const int32_t (&o)[VW], int vec) {
  if constexpr (VW == 8) {
    if (vec == 2) {
      asm volatile("st.global.cs.v8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(p), "r"(o[0]), "r"(o[1]), "r"(o[2]),
                   "r"(o[3]), "r"(o[4]), "r"(o[5]), "r"(o[6]), "r"(o[7])
                   : "memory");
      return;
    }
  }
  if (vec) {
#pragma unroll
    for (int h = 0; h < VW; h += 4)
      st_stream(reinterpret_cast<int4*>(p + h), make_int4(o[h], o[h + 1], o[h + 2], o[h + 3]));
  } else {
#pragma unroll
    for (int e = 0; e < VW; ++e) st_stream(p + e, o[e]);
  }
}
// int64 groups: one 32-B streaming store when the output is 32-B aligned
// (vec == 2; half the L1 lines per instruction of two 16-B halves), else two
// 16-B stores (vec == 1) or scalars
#ifndef FSG_I64_ST256
#define FSG_I64_ST256 1
#endif
template <int VW>
__device__ __forceinline__ void store_group(int64_t* p, const int64_t (&o)[VW], int vec) {
#if FSG_I64_ST256
  if (vec == 2) {
#pragma unroll
    for (int h = 0; h < VW; h += 4)
      asm volatile("st.global.cs.v4.s64 [%0], {%1,%2,%3,%4};" ::"l"(p + h), "l"(o[h]), "l"(o[h + 1]), "l"(o[h + 2]),
                   "l"(o[h + 3])
                   : "memory");
    return;
  }
#endif
  if (vec) {
#pragma unroll
    for (int h = 0; h < VW; h += 2) st_stream(reinterpret_cast<longlong2*>(p + h), make_longlong2(o[h], o[h + 1]));
  } else {
#pragma unroll
    for (int e = 0; e < VW; ++e) st_stream(p + e, o[e]);
  }
}

// Probes without a prologue
template <typename P, typename T>
__device__ __forceinline__ auto run_prologue(const DevPlan<T>& p, unsigned char* smem, int)
    -> decltype(P::prologue(p, smem), void()) {
  P::prologue(p, smem);
}
template <typename P, typename T>
__device__ __forceinline__ void run_prologue(const DevPlan<T>&, unsigned char*, long) {}

// Probes that define `template <int N> batch(const T (&)[N], int64_t (&)[N])`
// resolve a group of independent queries in lockstep (ILP across queries
// for multi-step searches); the others are applied one query at a time.
template <typename P, typename = void>
struct has_batch : std::false_type {};
template <typename P>
struct has_batch<P, std::void_t<decltype(&P::template batch<16, int64_t>)>> : std::true_type {};

template <typename P, typename T, typename R, int N>
__device__ __forceinline__ void probe_batch(const P& p, const T (&z)[N], R (&o)[N]) {
  if constexpr (has_batch<P>::value) {
    p.template batch<N, R>(z, o);
  } else {
#pragma unroll
    for (int i = 0; i < N; ++i) o[i] = (R)p(z[i]);
  }
}

struct StreamShape {
  uint64_t m;      // total queries
  uint64_t head;   // scalar queries before the first aligned group
  uint64_t nvec;   // groups of VW (vector path)
  uint64_t base;   // global position of z[0] (for first-bad reporting)
};

template <typename T, typename OutT, typename Probe, int UNROLL, int VW>
__device__ __forceinline__ void search_body(const T* __restrict__ z, OutT* __restrict__ out, StreamShape sh,
                                            DevPlan<T> plan, unsigned long long* __restrict__ status, int merge,
                                            StageSeg seg0, StageSeg seg1, int nseg) {
  extern __shared__ __align__(128) unsigned char smem[];
  __shared__ uint64_t bar;
  if (nseg > 0) {
    StageSeg segs[2] = {seg0, seg1};
    segs[0].dst = smem;
    segs[1].dst = smem + plan.x_smem_bytes_aligned();
    stage_tables(segs, nseg, &bar);
  }
  run_prologue<Probe>(plan, smem, 0);
  const Probe probe(plan, smem);
  const T x0 = plan.x0, xn = plan.xn;
  unsigned long long mybad = ~0ull;
  const uint64_t tid = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;

  auto one = [&](uint64_t pos) {
    const T v = ld_stream(z + pos);
    const bool bad = !(v >= x0 && v < xn);
    if (bad && pos < mybad) mybad = pos;
    out[pos] = (OutT)probe(v);
  };

  {
    // scalar head (< VW queries) and tail (< VW queries)
    const uint64_t tail0 = sh.head + VW * sh.nvec;
    if (tid < sh.head) one(tid);
    if (tid < sh.m - tail0) one(tail0 + tid);
    const int vec_out = plan.out_vec_ok;
    const T* zv = z + sh.head;
    OutT* ov = out + sh.head;
    for (uint64_t g0 = tid; g0 < sh.nvec; g0 += stride * UNROLL) {
      T zz[UNROLL * VW];
#pragma unroll
      for (int u = 0; u < UNROLL; ++u) {
        const uint64_t g = g0 + u * stride;
        VecLoad<T, VW> b;
        if (g < sh.nvec) {
          b.load(zv + VW * g);
        } else {
#pragma unroll
          for (int e = 0; e < VW; ++e) b.v[e] = x0;
        }
#pragma unroll
        for (int e = 0; e < VW; ++e) zz[VW * u + e] = b.v[e];
      }
      // results in the output's width: int32 halves the live registers
      using R = std::conditional_t<sizeof(OutT) == 4, int32_t, int64_t>;
      R o[UNROLL * VW];
      probe_batch<Probe, T, R, UNROLL * VW>(probe, zz, o);
#pragma unroll
      for (int u = 0; u < UNROLL; ++u) {
        const uint64_t g = g0 + u * stride;
        if (g < sh.nvec) {
          // domain check: a VW-bit mask per group; the position is formed and
          // min-merged only for a group holding a bad query (rare)
          uint32_t badmask = 0;
#pragma unroll
          for (int e = 0; e < VW; ++e) {
            const T v = zz[VW * u + e];
            badmask |= (uint32_t)!(v >= x0 && v < xn) << e;
          }
          if (badmask) {
            const uint64_t pos = sh.head + VW * g + (uint32_t)__ffs(badmask) - 1;
            if (pos < mybad) mybad = pos;
          }
          R ou[VW];
#pragma unroll
          for (int e = 0; e < VW; ++e) ou[e] = o[VW * u + e];
          store_group<VW>(ov + VW * g, ou, vec_out);
        }
      }
    }
  }
  finalize_first_bad(mybad == ~0ull ? ~0ull : mybad + sh.base, status, merge);
}

// The kernel entry points: the register budget is left to ptxas (a kernel
// above 64 registers then runs 512-thread CTAs), or bounded so that one
// 1024-thread CTA fits per SM (at most 64 registers, small spills allowed);
// which one a probe uses is measured (BoundedFor, fsgpu.cu).
template <typename T, typename OutT, typename Probe, int UNROLL, int VW>
__global__ void search_kernel(const T* __restrict__ z, OutT* __restrict__ out, StreamShape sh, DevPlan<T> plan,
                              unsigned long long* __restrict__ status, int merge, StageSeg seg0, StageSeg seg1,
                              int nseg) {
  search_body<T, OutT, Probe, UNROLL, VW>(z, out, sh, plan, status, merge, seg0, seg1, nseg);
}
template <typename T, typename OutT, typename Probe, int UNROLL, int VW>
__global__ void __launch_bounds__(1024, 1)
    search_kernel_1k(const T* __restrict__ z, OutT* __restrict__ out, StreamShape sh, DevPlan<T> plan,
                     unsigned long long* __restrict__ status, int merge, StageSeg seg0, StageSeg seg1, int nseg) {
  search_body<T, OutT, Probe, UNROLL, VW>(z, out, sh, plan, status, merge, seg0, seg1, nseg);
}

}  // namespace fsg
