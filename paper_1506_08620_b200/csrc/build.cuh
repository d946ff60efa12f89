// build.cuh — index construction kernels.
//
//   certify_prep / certify_finalize / certify_check / certify_grow
//       restate direct.compute_h_r (direct.py:135-191) op for op
//   knot_buckets_kernel  direct.knot_buckets + the f[-1] == r check
//                        (direct.py:194-197, 215-217)
//   fill_table_kernel    the np.repeat of build_index (direct.py:218-226),
//                        restated as K[j] = lower_bound(f, j) (gap 1) or
//                        upper_bound(f, j) - 1 (gap > 1): bucket-parallel,
//                        coalesced writes, O(R log(range)) instead of a
//                        per-knot scatter whose run lengths vary by 10^4x
//   fill_fused_kernel    direct.with_fused (direct.py:255-263)
//   pad_right_kernel     partition.pad_right_pow2 (partition.py:163-171)
//   eytzinger_kernel     eytzinger.build_layout (eytzinger.py:45-63)
#pragma once

#include "common.cuh"

namespace fsg {

// Device status block of the certification (lives in caller workspace).
struct CertStatus {
  unsigned long long collide_pos;  // min i+q with D[i+q] == D[i]
  unsigned long long min_key;      // order key of min RN(D[i+b] - D[i])
  unsigned long long fail;         // any pair with floor(hD[i+q]) <= floor(hD[i])
  unsigned long long inconsistent; // build_index: f[N] != r
  double h;                        // current H (exact in dtype)
  double h_start;                  // initial guess
  double growth;                   // current increment
  double r_float;                  // floor(RN(h * D_N))
  int32_t status;                  // 0 ok, 1 not distinguishable, 2 overflow
  uint32_t increments;
};

__global__ void cert_init_kernel(CertStatus* st) {
  st->collide_pos = ~0ull;
  st->min_key = ~0ull;
  st->fail = 0;
  st->inconsistent = 0;
  st->h = st->h_start = st->growth = st->r_float = 0.0;
  st->status = 0;
  st->increments = 0;
}

template <int NT>
__device__ __forceinline__ unsigned long long block_min_u64(unsigned long long v) {
  __shared__ unsigned long long red[NT / 32];
  v = warp_min_u64(v);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
  __syncthreads();
  if (threadIdx.x < 32) {
    v = threadIdx.x < NT / 32 ? red[threadIdx.x] : ~0ull;
    v = warp_min_u64(v);
  }
  __syncthreads();
  return v;  // valid in thread 0
}

// K1: collisions of the rounded offsets and the smallest gap-b difference.
// direct.py:156-166.
template <typename T, int NT>
__global__ void __launch_bounds__(NT) certify_prep(const T* __restrict__ x, uint64_t n1, uint64_t q,
                                                   uint64_t basis, CertStatus* st) {
  const T x0 = x[0];
  unsigned long long coll = ~0ull, mk = ~0ull;
  for (uint64_t i = (uint64_t)blockIdx.x * NT + threadIdx.x; i < n1; i += (uint64_t)gridDim.x * NT) {
    const T di = sub_rn(__ldg(x + i), x0);
    if (i + q < n1) {
      const T dq = sub_rn(__ldg(x + i + q), x0);
      if (dq == di && i + q < coll) coll = i + q;
    }
    if (i + basis < n1) {
      const T db = sub_rn(__ldg(x + i + basis), x0);
      const unsigned long long k = order_key(sub_rn(db, di));
      mk = k < mk ? k : mk;
    }
  }
  coll = block_min_u64<NT>(coll);
  mk = block_min_u64<NT>(mk);
  if (threadIdx.x == 0) {
    if (coll != ~0ull) atomicMin(&st->collide_pos, coll);
    if (mk != ~0ull) atomicMin(&st->min_key, mk);
  }
}

// Initial guess, overflow test and first increment.  direct.py:158-173.
template <typename T>
__global__ void certify_finalize(const T* __restrict__ x, uint64_t n1, int qbits, CertStatus* st) {
  if (st->collide_pos != ~0ull) {
    st->status = 1;
    return;
  }
  const T mn = from_key<T>(st->min_key);
  const T h = div_rn(T(1), mn);
  const T span = sub_rn(x[n1 - 1], x[0]);
  const T limit = qbits == 64 ? T(18446744073709551616.0) : T(4294967296.0);
  st->h = (double)h;
  st->h_start = (double)h;
  if (!(mul_rn(h, span) < limit)) {
    st->status = 2;
    return;
  }
  st->growth = (double)sub_rn(next_up(h), h);
}

// K2: certify every gap-q pair at the current H.  direct.py:176-178, 185.
template <typename T, int NT>
__global__ void __launch_bounds__(NT) certify_check(const T* __restrict__ x, uint64_t n1, uint64_t q,
                                                    CertStatus* st) {
  if (st->status != 0) return;
  const T x0 = x[0];
  const T h = (T)st->h;
  bool bad = false;
  for (uint64_t i = (uint64_t)blockIdx.x * NT + threadIdx.x; i + q < n1; i += (uint64_t)gridDim.x * NT) {
    const T fi = floor(mul_rn(h, sub_rn(__ldg(x + i), x0)));
    const T fq = floor(mul_rn(h, sub_rn(__ldg(x + i + q), x0)));
    bad |= !(fq > fi);
  }
  if (__syncthreads_or(bad) && threadIdx.x == 0) st->fail = 1;
  if (blockIdx.x == 0 && threadIdx.x == 0) st->r_float = (double)floor(mul_rn(h, sub_rn(x[n1 - 1], x0)));
}

// One growth step: h += growth; overflow test; growth doubles.
// direct.py:179-183.
template <typename T>
__global__ void certify_grow(const T* __restrict__ x, uint64_t n1, int qbits, CertStatus* st) {
  const T span = sub_rn(x[n1 - 1], x[0]);
  const T limit = qbits == 64 ? T(18446744073709551616.0) : T(4294967296.0);
  T h = (T)st->h;
  T g = (T)st->growth;
  h = add_rn(h, g);
  st->h = (double)h;
  st->increments += 1;
  st->fail = 0;
  if (!(mul_rn(h, span) < limit)) {
    st->status = 2;
    return;
  }
  st->growth = (double)add_rn(g, g);
}

// f_i = floor(RN(h * RN(X_i - X0))) as an integer.  direct.py:194-197.
template <typename T>
__global__ void knot_buckets_kernel(const T* __restrict__ x, uint64_t n1, T h, uint64_t r,
                                    uint64_t* __restrict__ f, CertStatus* st) {
  const T x0 = x[0];
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n1; i += (uint64_t)gridDim.x * blockDim.x) {
    const T v = floor(mul_rn(h, sub_rn(__ldg(x + i), x0)));
    const uint64_t fi = trunc_to<uint64_t>(v);
    f[i] = fi;
    if (st && i == n1 - 1 && fi != r) st->inconsistent = 1;
  }
}

// Knot bytes beside the rank directory (fs_build_knot_bytes): B[i] = floor(256
// frac(p_i)) for p_i = RN(h RN(X_i - X0)), the product whose floor is knot
// i's bucket (direct.py:194-197) -- where inside its bucket the knot falls, to
// 1/256.  RN is monotone, so for a query z with product p: p < p_i implies
// z < X_i and p > p_i implies z > X_i; comparing (bucket, byte) pairs decides
// all but ties, which read X.
template <typename T>
__global__ void fill_knot_bytes_kernel(const T* __restrict__ x, uint64_t n1, T h, uint8_t* __restrict__ B,
                                       uint64_t npad) {
  const T x0 = x[0];
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < npad; i += (uint64_t)gridDim.x * blockDim.x) {
    uint32_t q = 0;
    if (i < n1) {
      const T p = mul_rn(h, sub_rn(__ldg(x + i), x0));
      q = trunc_to<uint32_t>(mul_rn(sub_rn(p, floor(p)), (T)256));
    }
    B[i] = (uint8_t)q;
  }
}

// First index in [lo, hi) with f[i] >= key (UPPER=false) or f[i] > key (UPPER=true).
template <bool UPPER>
__device__ __forceinline__ uint64_t bound_search(const uint64_t* __restrict__ f, uint64_t lo, uint64_t hi,
                                                 uint64_t key) {
  while (lo < hi) {
    const uint64_t mid = lo + ((hi - lo) >> 1);
    const uint64_t v = __ldg(f + mid);
    const bool go_right = UPPER ? (v <= key) : (v < key);
    if (go_right) lo = mid + 1;
    else hi = mid;
  }
  return lo;
}

// K[j] for j in [0, r]: gap 1 -> lower_bound(f, j); gap > 1 -> upper_bound(f, j) - 1.
// Each CTA owns a tile of TILE consecutive buckets; thread 0 brackets the
// knot range of the tile once, then every thread searches only inside it.
template <int NT, int ITEMS, bool UPPER>
__global__ void __launch_bounds__(NT) fill_table_kernel(const uint64_t* __restrict__ f, uint64_t n1, uint64_t r,
                                                        uint32_t* __restrict__ K) {
  constexpr uint64_t TILE = (uint64_t)NT * ITEMS;
  __shared__ uint64_t rng[2];
  const uint64_t total = r + 1;
  for (uint64_t t0 = (uint64_t)blockIdx.x * TILE; t0 < total; t0 += (uint64_t)gridDim.x * TILE) {
    const uint64_t t1 = (t0 + TILE < total ? t0 + TILE : total) - 1;  // inclusive
    if (threadIdx.x == 0) {
      rng[0] = bound_search<UPPER>(f, 0, n1, t0);
      rng[1] = bound_search<UPPER>(f, 0, n1, t1);
    }
    __syncthreads();
    // lower_bound answers lie in [rng0, rng1]; upper_bound answers too.
    const uint64_t lo = rng[0], hi = rng[1] + 1 < n1 ? rng[1] + 1 : n1;
    for (uint64_t j = t0 + threadIdx.x; j <= t1; j += NT) {
      const uint64_t b = bound_search<UPPER>(f, lo, hi, j);
      K[j] = (uint32_t)(UPPER ? b - 1 : b);
    }
    __syncthreads();
  }
}

// Rank directory of the gap-1 table (see fs_build_rank in fsgpu.h): word w
// = {mask of buckets 32w..32w+31 holding a knot, K[32w]}.  One thread per
// word: K[32w] = lower_bound(f, 32w), then at most 32 knots set bits.
__global__ void fill_rank_kernel(const uint64_t* __restrict__ f, uint64_t n1, uint64_t r, uint2* __restrict__ dir) {
  const uint64_t words = (r >> 5) + 1;
  for (uint64_t w = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; w < words; w += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t j0 = w << 5;
    const uint64_t base = bound_search<false>(f, 0, n1, j0);
    uint32_t mask = 0;
    for (uint64_t i = base; i < n1; ++i) {
      const uint64_t fi = __ldg(f + i);
      if (fi >= j0 + 32) break;
      mask |= 1u << (uint32_t)(fi - j0);
    }
    dir[w] = make_uint2(mask, (uint32_t)base);
  }
}

// Rank rows (fs_build_rank_rows): the rank directory word of 32 buckets {mask,
// base} widened to 16 B with the knot bytes (fill_knot_bytes_kernel) of the
// row's first eight knots, B[base .. base+7] (zero past the last knot).
__global__ void fill_rank_rows_kernel(const uint64_t* __restrict__ f, const uint8_t* __restrict__ B, uint64_t n1,
                                      uint64_t r, uint4* __restrict__ rows) {
  const uint64_t words = (r >> 5) + 1;
  for (uint64_t w = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; w < words; w += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t j0 = w << 5;
    const uint64_t base = bound_search<false>(f, 0, n1, j0);
    uint32_t mask = 0, lo = 0, hi = 0, cnt = 0;
    for (uint64_t i = base; i < n1; ++i) {
      const uint64_t fi = __ldg(f + i);
      if (fi >= j0 + 32) break;
      mask |= 1u << (uint32_t)(fi - j0);
      const uint32_t b = __ldg(B + i);
      if (cnt < 4) lo |= b << (8 * cnt);
      else if (cnt < 8) hi |= b << (8 * (cnt - 4));
      ++cnt;
    }
    rows[w] = make_uint4(mask, (uint32_t)base, lo, hi);
  }
}

// Rank directory of the gap-2 table (fs_build_rank2).  A gap-2 certificate
// allows at most two knots per bucket (f_{i+2} > f_i), so word w holds
// m1 = buckets with >= 1 knot, m2 = buckets with 2 knots and base =
// #{i : f_i < 32w}; then K2[j] = upper_bound(f, j) - 1 =
// base + popc(m1 & le) + popc(m2 & le) - 1 with le = bits 0..j mod 32.
__global__ void fill_rank2_kernel(const uint64_t* __restrict__ f, uint64_t n1, uint64_t r, uint4* __restrict__ dir) {
  const uint64_t words = (r >> 5) + 1;
  for (uint64_t w = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; w < words; w += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t j0 = w << 5;
    const uint64_t base = bound_search<false>(f, 0, n1, j0);
    uint32_t m1 = 0, m2 = 0;
    for (uint64_t i = base; i < n1; ++i) {
      const uint64_t fi = __ldg(f + i);
      if (fi >= j0 + 32) break;
      const uint32_t bit = 1u << (uint32_t)(fi - j0);
      if (m1 & bit) m2 |= bit;
      else m1 |= bit;
    }
    dir[w] = make_uint4(m1, m2, (uint32_t)base, 0u);
  }
}

// Count directory of a gap-q table (fs_build_countdir): a gap-q certificate
// (f_{i+q} > f_i, direct.py:176-178) allows at most q knots per bucket, so
// each bucket's knot count fits B bits (B = 2 for q <= 3, 4 for q <= 15).
// Word w = {B-bit counts of buckets w 32/B .. (w+1) 32/B - 1, base =
// #{i : f_i < w 32/B}}; then K_q[j] = upper_bound(f, j) - 1 = base + (sum of
// the counts of buckets <= j in the word) - 1 (direct.py:215-228).
template <int B>
__global__ void fill_countdir_kernel(const uint64_t* __restrict__ f, uint64_t n1, uint64_t r, uint2* __restrict__ dir) {
  constexpr int LG = B == 2 ? 4 : 3;  // buckets per word: 16 / 8
  const uint64_t words = (r >> LG) + 1;
  for (uint64_t w = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; w < words; w += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t j0 = w << LG;
    const uint64_t base = bound_search<false>(f, 0, n1, j0);
    uint32_t counts = 0;
    for (uint64_t i = base; i < n1; ++i) {
      const uint64_t fi = __ldg(f + i);
      if (fi >= j0 + (1u << LG)) break;
      counts += 1u << (B * (uint32_t)(fi - j0));  // certified: a field never exceeds q < 2^B
    }
    dir[w] = make_uint2(counts, (uint32_t)base);
  }
}

// Two-level sparse encoding of the gap-1 table for R >> N: super-bucket J
// (buckets J 2^s .. (J+1) 2^s - 1) stores C[J] = K[J 2^s] = lower_bound(f,
// J 2^s); every knot i stores F[i] = f_i mod 2^s (16 bit).  The knots of
// super-bucket J are exactly [C[J], C[J+1]), so K[j] = C[j >> s] +
// #{i in it : F[i] < j mod 2^s}.  C has (r >> s) + 2 entries, the last = n1.
__global__ void fill_sparse_kernel(const uint64_t* __restrict__ f, uint64_t n1, uint64_t r, int s,
                                   uint32_t* __restrict__ C, uint16_t* __restrict__ F) {
  const uint64_t nc = (r >> s) + 2;
  const uint64_t mask = (1ull << s) - 1;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nc || i < n1;
       i += (uint64_t)gridDim.x * blockDim.x) {
    if (i < nc) C[i] = i == nc - 1 ? (uint32_t)n1 : (uint32_t)bound_search<false>(f, 0, n1, i << s);
    if (i < n1) F[i] = (uint16_t)(__ldg(f + i) & mask);
  }
}

// Group records of the gap-1 table (fs_build_sparse_rec): the same
// super-buckets as fill_sparse_kernel, each packed into one record {base |
// overflow flag, SLOTS 16-bit knot offsets} (16 B with six slots, 8 B with
// two) so that one shared-memory load resolves K[j] for super-buckets
// holding up to SLOTS knots.  base = lower_bound(f, J 2^s) = K[J 2^s];
// offsets are f_i mod 2^s of the first min(count, SLOTS) knots, ascending,
// unused slots kRecSentinel (> any j mod 2^s for s <= kRecMaxShift).  A
// super-bucket with more knots sets bit 31 of base; its further knots are
// found in F (f_i mod 2^s, u16 per knot, written when F != NULL).  ng =
// (r >> s) + 2 records, the last has base = n1 (the probe reads record J + 1
// as the end of J's knots).
template <int SLOTS>
__global__ void fill_sparse_rec_kernel(const uint64_t* __restrict__ f, uint64_t n1, uint64_t r, int s,
                                       typename RecWord<SLOTS>::type* __restrict__ G, uint16_t* __restrict__ F) {
  const uint64_t ng = (r >> s) + 2;
  const uint64_t mask = (1ull << s) - 1;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < ng || i < n1;
       i += (uint64_t)gridDim.x * blockDim.x) {
    if (i < ng) {
      const uint64_t lo = i == ng - 1 ? n1 : bound_search<false>(f, 0, n1, i << s);
      uint32_t off[SLOTS];
      uint64_t k = 0;
      for (; k < SLOTS && lo + k < n1; ++k) {
        const uint64_t fi = __ldg(f + lo + k);
        if ((fi >> s) != i) break;
        off[k] = (uint32_t)(fi & mask);
      }
      for (uint64_t e = k; e < SLOTS; ++e) off[e] = SLOTS == 8 ? 0x7FFu : SLOTS == 3 ? 0xFFFu : kRecSentinel;
      const bool ovf = k == SLOTS && lo + k < n1 && (__ldg(f + lo + k) >> s) == i;
      const uint32_t b = (uint32_t)lo | (ovf ? kDenseFlag : 0u);
      if constexpr (SLOTS == 6) {
        G[i] = make_uint4(b, off[0] | (off[1] << 16), off[2] | (off[3] << 16), off[4] | (off[5] << 16));
      } else if constexpr (SLOTS == 8) {
        // 96 bits of fields 0x800 | offset at bit 12k (field 2 and 5 straddle words)
        unsigned long long lo64 = 0, hi32 = 0;
        for (int e = 0; e < 8; ++e) {
          const unsigned long long v = 0x800ull | off[e];
          if (e < 5) lo64 |= v << (12 * e);                                  // bits 0..59
          if (e == 5) { lo64 |= v << 60; hi32 |= v >> 4; }                    // bits 60..71
          if (e > 5) hi32 |= v << (12 * e - 64);                              // bits 72..95
        }
        G[i] = make_uint4(b, (uint32_t)lo64, (uint32_t)(lo64 >> 32), (uint32_t)hi32);
      } else if constexpr (SLOTS == 3) {
        unsigned long long w = (unsigned long long)lo | (ovf ? (1ull << 24) : 0ull);
        for (int e = 0; e < 3; ++e) w |= (0x1000ull | off[e]) << (25 + 13 * e);
        G[i] = make_uint2((uint32_t)w, (uint32_t)(w >> 32));
      } else {
        G[i] = make_uint2(b, off[0] | (off[1] << 16));
      }
    }
    if (F && i < n1) F[i] = (uint16_t)(__ldg(f + i) & mask);
  }
}

// Zoned records of the gap-1 table (fs_build_zoned): one thread per 8-B
// record.  zdesc[z] = (first record - (z << (zs - s))) << 5 | rank flag | s
// for zone z (buckets
// [z 2^zs, (z+1) 2^zs)); record g of zone z covers buckets j0 .. j0 + 2^s - 1,
// j0 = z 2^zs + (g - first) 2^s, and base = lower_bound(f, j0) = K[j0].  Slot
// records pack base (bits 0..23) and the offsets f_i - j0 of the (at most
// three, by the planner's choice of s) knots in range as 0x1000 | offset at
// bits 25 + 13k, unused 0x1FFF; rank records are {mask of the 32 buckets
// holding a knot, base}.  STRIPED (fs_build_zoned_rank): every zone in rank
// records whose descriptor holds the stripe shift k instead of s; a record
// covers 2^(k+5) buckets and mask bit b is set iff a knot falls in buckets
// [j0 + b 2^k, j0 + (b+1) 2^k) (at most one does, by the planner's k).
template <bool STRIPED>
__global__ void fill_zoned_kernel(const uint64_t* __restrict__ f, uint64_t n1, int zs,
                                  const uint32_t* __restrict__ zdesc, uint32_t nz, uint2* __restrict__ R,
                                  uint64_t nrec) {
  for (uint64_t g = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; g < nrec; g += (uint64_t)gridDim.x * blockDim.x) {
    // zone z's first record = ((int)desc >> 5) + (z << (zs - s))
    auto first = [&](uint32_t k) {
      const uint32_t dk = __ldg(zdesc + k);
      return (uint64_t)((int64_t)((int32_t)dk >> 5) + ((int64_t)k << (zs - (int)(dk & 15u) - (STRIPED ? kZonedRankShift : 0))));
    };
    uint32_t z = 0;
    for (uint32_t k = 1; k < nz; ++k)
      if (first(k) <= g) z = k;
    const uint32_t d = __ldg(zdesc + z);
    const int kst = STRIPED ? (int)(d & 15u) : 0;  // stripe shift
    const int s = (int)(d & 15u) + (STRIPED ? kZonedRankShift : 0);
    const uint64_t j0 = ((uint64_t)z << zs) + ((g - first(z)) << s);
    const uint64_t j1 = j0 + (1ull << s);
    const uint64_t lo = bound_search<false>(f, 0, n1, j0);
    if (d & kZonedRankFlag) {
      uint32_t m = 0;
      for (uint64_t k = lo; k < n1; ++k) {
        const uint64_t fi = __ldg(f + k);
        if (fi >= j1) break;
        m |= 1u << ((fi - j0) >> kst);
      }
      R[g] = make_uint2(m, (uint32_t)lo);
    } else {
      unsigned long long w = lo;
      int k = 0;
      for (; k < kZonedSlots && lo + k < n1; ++k) {
        const uint64_t fi = __ldg(f + lo + k);
        if (fi >= j1) break;
        w |= (0x1000ull | (fi - j0)) << (25 + 13 * k);
      }
      for (; k < kZonedSlots; ++k) w |= 0x1FFFull << (25 + 13 * k);
      R[g] = make_uint2((uint32_t)w, (uint32_t)(w >> 32));
    }
  }
}

// Count words of the gap-1 table (fs_build_count_words): one thread per 8-B
// word.  Word g covers buckets j0 .. j0 + 2^(k+4) - 1, j0 = g 2^(k+4), in 16
// stripes of 2^k; bits 2b, 2b+1 of the mask hold the number of knots in
// stripe b, saturated at 3; base = lower_bound(f, j0) = K[j0], with bit 31
// set when a stripe of the word holds four or more knots (its counts are
// then no longer exact and the probe scans the word's knots instead).
__global__ void fill_count_words_kernel(const uint64_t* __restrict__ f, uint64_t n1, int k, uint2* __restrict__ W,
                                        uint64_t nwords) {
  const int s = k + kCountWordShift;
  for (uint64_t g = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; g < nwords; g += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t j0 = g << s, j1 = j0 + (1ull << s);
    const uint64_t lo = bound_search<false>(f, 0, n1, j0);
    uint32_t m = 0, flag = 0;
    for (uint64_t i = lo; i < n1; ++i) {
      const uint64_t fi = __ldg(f + i);
      if (fi >= j1) break;
      const uint32_t sh = 2u * (uint32_t)((fi - j0) >> k);
      if (((m >> sh) & 3u) == 3u) flag = kCountFlag;  // a fourth knot in this stripe
      else m += 1u << sh;
    }
    W[g] = make_uint2(m, (uint32_t)lo | flag);
  }
}

// Knot offsets beside the count words (fs_build_count_words with offsets):
// O[i] = f_i mod 2^k, knot i's bucket inside its stripe (k <= 8: one byte).
__global__ void fill_count_offsets_kernel(const uint64_t* __restrict__ f, uint64_t n1, int k, uint8_t* __restrict__ O,
                                          uint64_t npad) {
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < npad; i += (uint64_t)gridDim.x * blockDim.x)
    O[i] = i < n1 ? (uint8_t)(__ldg(f + i) & ((1ull << k) - 1)) : (uint8_t)0;
}

// Dense super-buckets of the sparse table (more than kDenseOcc knots): one
// CTA per dense slot builds the 2^s-bit knot mask of super-bucket
// J = dense_j[slot] in W = 2^(s-5) words plus per-word knot prefix counts,
// then flags C[J] (bit 31) and stores the slot in F[C[J]], which the dense
// path never reads as an offset.

__global__ void fill_dense_kernel(uint32_t* __restrict__ C, uint16_t* __restrict__ F, const uint32_t* __restrict__ dense_j,
                                  uint64_t ndense, int s, uint32_t* __restrict__ dmask, uint16_t* __restrict__ dpre) {
  const uint32_t W = 1u << (s - 5);
  for (uint64_t slot = blockIdx.x; slot < ndense; slot += gridDim.x) {
    const uint32_t J = dense_j[slot];
    const uint32_t lo = C[J] & ~kDenseFlag, hi = C[J + 1] & ~kDenseFlag;
    for (uint32_t w = threadIdx.x; w < W; w += blockDim.x) {
      uint32_t m = 0, pre = 0;
      for (uint32_t i = lo; i < hi; ++i) {
        const uint32_t off = F[i];
        if ((off >> 5) == w) m |= 1u << (off & 31);
        else if ((off >> 5) < w) ++pre;
      }
      dmask[slot * W + w] = m;
      dpre[slot * W + w] = (uint16_t)pre;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      F[lo] = (uint16_t)slot;
      C[J] = lo | kDenseFlag;
    }
    __syncthreads();
  }
}

// Hot window of the rank directory: for every start word a, the longest
// window [a, b) whose directory words plus the X range they reference,
// [base_a, base_b], fit in `budget` bytes; the window holding the most
// knots wins (ties -> lowest a).  Packed key (knots << 32 | ~a) max-reduced.
__global__ void hot_window_kernel(const uint2* __restrict__ dir, uint64_t words, uint32_t es, uint64_t budget,
                                  unsigned long long* __restrict__ best) {
  unsigned long long mine = 0;
  for (uint64_t a = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; a < words; a += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t base_a = __ldg(&dir[a].y);
    // cost(a, b) = 8 (b - a) + es (base_b - base_a + 1) is monotone in b
    uint64_t lo = a, hi = words - 1;  // largest b in [a, words-1] with cost <= budget
    if (8ull + es * 1ull > budget) continue;
    while (lo < hi) {
      const uint64_t mid = lo + ((hi - lo + 1) >> 1);
      const uint64_t cost = 8ull * (mid - a) + (uint64_t)es * ((uint64_t)__ldg(&dir[mid].y) - base_a + 1);
      if (cost <= budget) lo = mid;
      else hi = mid - 1;
    }
    const uint64_t knots = (uint64_t)__ldg(&dir[lo].y) - base_a;
    if (lo > a && a <= 0xffffffffull) {
      const unsigned long long key = (knots << 32) | (0xffffffffull - a);
      mine = key > mine ? key : mine;
    }
  }
  // warp max, then one atomic per warp
  for (int o = 16; o > 0; o >>= 1) {
    const unsigned long long w = __shfl_xor_sync(0xffffffffu, mine, o);
    mine = w > mine ? w : mine;
  }
  if ((threadIdx.x & 31) == 0 && mine) atomicMax(best, mine);
}

// Window end for the chosen start word (single thread): out = {b, base_a, base_b}.
__global__ void hot_window_finish(const uint2* __restrict__ dir, uint64_t words, uint32_t es, uint64_t budget,
                                  uint64_t a, uint64_t* __restrict__ out) {
  const uint64_t base_a = dir[a].y;
  uint64_t lo = a, hi = words - 1;
  while (lo < hi) {
    const uint64_t mid = lo + ((hi - lo + 1) >> 1);
    const uint64_t cost = 8ull * (mid - a) + (uint64_t)es * ((uint64_t)dir[mid].y - base_a + 1);
    if (cost <= budget) lo = mid;
    else hi = mid - 1;
  }
  out[0] = lo;
  out[1] = base_a;
  out[2] = dir[lo].y;
}

// Fused (idx, val) records.  direct.py:255-263.
__global__ void fill_fused_f32(const float* __restrict__ x, const uint32_t* __restrict__ K, uint64_t r,
                               uint2* __restrict__ rec) {
  for (uint64_t j = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; j <= r; j += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t t = K[j];
    rec[j] = make_uint2(t, __float_as_uint(__ldg(x + t)));
  }
}
__global__ void fill_fused_f64(const double* __restrict__ x, const uint32_t* __restrict__ K, uint64_t r,
                               double2* __restrict__ rec) {
  for (uint64_t j = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; j <= r; j += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t t = K[j];
    rec[j] = make_double2(__longlong_as_double((long long)(unsigned long long)t), __ldg(x + t));
  }
}

// xpad[i] = X[min(i, N)], i < 2^pbits.  partition.py:163-171.
template <typename T>
__global__ void pad_right_kernel(const T* __restrict__ x, uint64_t n1, uint64_t len, T* __restrict__ xpad) {
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < len; i += (uint64_t)gridDim.x * blockDim.x)
    xpad[i] = __ldg(x + (i < n1 ? i : n1 - 1));
}

// Heap-order tree: slot s (1-based q = s + 1) at level l = floor(log2 q)
// holds the padded knot of in-order rank (q - 2^l) * 2^(L-l) + 2^(L-l-1) - 1.
// eytzinger.py:45-63.
template <typename T>
__global__ void eytzinger_kernel(const T* __restrict__ x, uint64_t n1, int depth, T* __restrict__ tree) {
  const uint64_t size = (1ull << depth) - 1;
  for (uint64_t s = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; s < size; s += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t qs = s + 1;
    const int lvl = 63 - __clzll((long long)qs);
    const uint64_t stride = 1ull << (depth - lvl);
    const uint64_t rank = (qs - (1ull << lvl)) * stride + (stride >> 1) - 1;
    tree[s] = __ldg(x + (rank < n1 ? rank : n1 - 1));
  }
}

// ---------------------------------------------------------------------------
// bitset2 subtree records for the global levels (fs_build_b2_deep).  Chunk c
// starts at level l_c and spans k_c levels; record m of the chunk holds, in
// BFS order, the padded values the bit-setting walk (binsearch.py:72-86)
// can probe in levels l_c .. l_c + k_c - 1 when its first l_c decisions are
// the bits of m: slot s at relative depth d = floor(log2(s + 1)), path q =
// s + 1 - 2^d reads xpad[(m << (p - l)) | (q << (p - l - d)) | 2^(p - l - d - 1)].
// One thread per record slot; unused slots are zero.
// ---------------------------------------------------------------------------
template <typename T>
__global__ void b2_deep_kernel(const T* __restrict__ xpad, int pbits, int level, int kc, uint64_t nrec,
                               T* __restrict__ rec) {
  constexpr int kSlots = 32 / sizeof(T);
  const uint64_t total = nrec * kSlots;
  for (uint64_t w = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; w < total; w += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t m = w / kSlots;
    const int s = (int)(w % kSlots);
    T v = T(0);
    if (s < (1 << kc) - 1) {
      const int d = 31 - __clz(s + 1);
      const uint64_t q = (uint64_t)(s + 1 - (1 << d));
      const int sh = pbits - level;
      v = xpad[(m << sh) | (q << (sh - d)) | (1ull << (sh - d - 1))];
    }
    rec[w] = v;
  }
}

}  // namespace fsg
