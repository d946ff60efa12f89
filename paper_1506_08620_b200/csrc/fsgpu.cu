// fsgpu.cu — C-ABI implementation (include/fsgpu.h).
//
// Host-side runtime of the library: argument validation, table placement
// (shared memory vs L2), launch geometry (persistent grid sized from the
// occupancy calculator x SM count), the certification loop of
// direct.compute_h_r, and the chunked host<->device pipeline of the
// end-to-end batch_search path.  No torch types cross this boundary.
#include <cuda_runtime.h>

#include <algorithm>
#include <array>
#include <cstdio>
#include <cstring>
#include <map>
#include <mutex>
#include <string>
#include <tuple>
#include <vector>

#include "../../include/fsgpu.h"
#include "build.cuh"
#include "common.cuh"
#include "crc32.cuh"
#include "host_staging.h"
#include "search.cuh"

using namespace fsg;

namespace {

thread_local std::string g_last_error;

int fail(int code, const std::string& msg) {
  g_last_error = msg;
  return code;
}

#define FS_CUDA(expr)                                                                         \
  do {                                                                                        \
    cudaError_t e_ = (expr);                                                                  \
    if (e_ != cudaSuccess)                                                                    \
      return fail(FS_CUDA_ERROR, std::string(#expr) + ": " + cudaGetErrorString(e_));         \
  } while (0)

inline cudaStream_t as_stream(void* s) { return reinterpret_cast<cudaStream_t>(s); }

int sm_count() {
  int dev = 0, n = 148;
  if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
  return n;
}

size_t smem_budget() {
  int dev = 0, optin = 227 * 1024;
  if (cudaGetDevice(&dev) == cudaSuccess)
    cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
  return (size_t)optin - 1024;  // static smem (mbarrier, reductions) + slack
}

int bit_length(uint64_t v) { return v ? 64 - __builtin_clzll(v) : 0; }

inline uint64_t align128(uint64_t b) { return (b + 127) & ~127ull; }

int grid_1d(uint64_t work, int threads) {
  uint64_t b = (work + threads - 1) / threads;
  uint64_t cap = (uint64_t)sm_count() * 8;
  if (b > cap) b = cap;
  return (int)std::max<uint64_t>(b, 1);
}

// ---------------------------------------------------------------------------
// Placement
// ---------------------------------------------------------------------------
#ifndef FSG_B2_REPLICATE
#define FSG_B2_REPLICATE 1
#endif
constexpr bool kB2Replicate = FSG_B2_REPLICATE != 0;
constexpr int kB2ConflictFree = 6;  // levels 0..5: at most 32 consecutive words

// bitset2's staged top levels: levels [0, top) in level order, levels
// [l1, l2) stored as 32 bank-private copies (Bitset2Probe).
// bitset2's global levels as subtree records (fs_build_b2_deep): chunks of
// k levels from `top` down while at least two levels remain; 32 B per record,
// 2^level records per chunk.
constexpr int kB2DeepMinLevels = 2;
inline int b2_deep_k(int dtype) { return dtype == FS_F32 ? 3 : 2; }
// Fewest global levels worth records: two f32 levels read 8 B of the padded
// array per query, which on clustered streams stays L1-resident better than
// a 32-B record (cfg4: 166 vs 137 Gq/s); from three f32 / two f64 levels
// the records win (2^20 f32 knots 42 -> 91, cfg5 N+1 = 32769 85 -> 98,
// N+1 = 1048577 33 -> 50; profiles/r01/tune_bitset2_deep.txt).
inline int b2_deep_min_levels(int dtype) { return dtype == FS_F32 ? 3 : 2; }
inline uint64_t b2_deep_total_bytes(int pbits, int top, int k) {
  uint64_t bytes = 0;
  for (int l = top; pbits - l >= kB2DeepMinLevels; l += std::min(k, pbits - l)) bytes += (1ull << l) * 32;
  return bytes;
}
// f64 bitset2 stages f32 shadow keys plus the exact f64 plane
// (Bitset2Probe::kShadow) from this many levels: shallow trees, whose levels
// are conflict-free or replicated anyway, lose to the extra conversion and
// check (cfg5 N+1 = 33 528 -> 400, 1025 297 -> 269 Gq/s); deeper ones win on
// the halved shared-memory wavefronts (cfg2 167 -> 207, N+1 = 32769 100 ->
// 125; profiles/r02/bitset2_shadow.txt)
#ifndef FSG_B2_SHADOW_MIN_BITS
#define FSG_B2_SHADOW_MIN_BITS 13
#endif
inline bool b2_shadow(int pbits, size_t es) { return es == 8 && pbits >= FSG_B2_SHADOW_MIN_BITS; }
// bytes per staged node: a shadow word plus the exact key, else the key
inline size_t b2_node_bytes(int pbits, size_t es) { return b2_shadow(pbits, es) ? 12 : es; }
inline int b2_top_bits(int pbits, size_t es) {
  return std::min(bit_length(smem_budget() / b2_node_bytes(pbits, es) + 1) - 1, pbits);
}
// levels [0, l1) plain, [l1, l2) 32 copies, [l2, l3) 16 copies, [l3, top) plain
inline uint64_t b2_smem_bytes(int top, int l1, int l2, int l3, size_t es, bool shadow) {
  if (shadow) return b2_shadow_bytes(top, l1, l2, l3) + ((1ull << top) - 1) * 8;
  return (((1ull << l1) - 1) + ((1ull << l2) - (1ull << l1)) * 32 + ((1ull << l3) - (1ull << l2)) * 16 +
          ((1ull << top) - (1ull << l3))) *
         es;
}
#ifndef FSG_B2_HALF
#define FSG_B2_HALF 1
#endif

// count directory of a gap-q table: log2 of the buckets per 8-B word
inline int countdir_lg(int q) { return q <= 3 ? 4 : 3; }

struct Placement {
  uint32_t x_bytes = 0;      // bytes staged at smem offset 0 (X / padded / tree / top)
  uint32_t table_bytes = 0;  // bytes staged after align128(x_bytes) (K / records)
  int top_bits = 0;          // bitset2: levels staged in smem ...
  int b2_l1 = 0, b2_l2 = 0;  // ... of which [b2_l1, b2_l2) replicated per bank
  int b2_l3 = 0;             // ... and [b2_l2, b2_l3) in 16 copies (lane pairs share one)
  bool xs = false, ks = false, top = false;
  int flags = FS_PLACE_GLOBAL;
  size_t smem = 0;
  const void* seg0_src = nullptr;  // bulk-copied segments
  const void* seg1_src = nullptr;
  uint32_t seg0_bytes = 0, seg1_bytes = 0;
  int nseg = 0;
  int tune = 0;          // fs_plan.tune (launch-geometry override)
  bool records = false;  // direct served from fused records in smem
  bool hot = false;      // direct over the rank directory with a smem hot window
  bool sparse = false;   // direct over the two-level sparse table in smem
  bool zoned = false;    // ... the zoned records (with a window of X)
  int merge = 0;         // status[0] = min(status[0], result) (chunked host path)
  bool b2_shadow = false;  // bitset2 f64: f32 shadow keys + exact plane staged
};

inline bool is_zoned(int32_t format) { return format == FS_SPARSE_ZONED || format == FS_SPARSE_ZONED_RANK; }

int validate_plan(const fs_plan* p) {
  if (!p) return fail(FS_INVALID_ARG, "plan is NULL");
  if (p->dtype != FS_F32 && p->dtype != FS_F64) return fail(FS_INVALID_ARG, "dtype must be FS_F32 or FS_F64");
  if (p->n1 < 2) return fail(FS_INVALID_ARG, "a partition needs at least two knots");
  if (p->n1 - 1 >= (1ull << 32)) return fail(FS_INVALID_ARG, "table entries are 32-bit; partition is too large");
  if (!p->x) return fail(FS_INVALID_ARG, "plan.x is NULL");
  switch (p->algorithm) {
    case FS_ALGO_DIRECT:
    case FS_ALGO_DIRECT_GAP2:
    case FS_ALGO_DIRECT_GENERIC:
    case FS_ALGO_DIRECT_CACHE:
      if (!p->table) return fail(FS_INVALID_ARG, "direct plan needs its table");
      if (p->q < 1) return fail(FS_INVALID_ARG, "gap must be >= 1");
      if (p->algorithm == FS_ALGO_DIRECT_CACHE && p->q != 1)
        return fail(FS_INVALID_ARG, "fused records pair with the gap-1 kernel");
      // optional accelerators: their extents must lie inside the tables they index
      if (p->hot_words && (p->hot_word0 > (p->r >> 5) + 1 || p->hot_words > (p->r >> 5) + 1 - p->hot_word0 ||
                           p->hot_knot0 > p->n1 || p->hot_knots > p->n1 - p->hot_knot0))
        return fail(FS_INVALID_ARG, "hot window outside the rank directory / knots");
      if (p->sparse && (p->sparse_format != FS_SPARSE_TWO_LEVEL && p->sparse_format != FS_SPARSE_RECORDS &&
                        p->sparse_format != FS_SPARSE_RECORDS8 && p->sparse_format != FS_SPARSE_RECORDS12 &&
                        p->sparse_format != FS_SPARSE_RECORDS8X3 && p->sparse_format != FS_SPARSE_ZONED &&
                        p->sparse_format != FS_SPARSE_ZONED_RANK && p->sparse_format != FS_SPARSE_COUNT &&
                        p->sparse_format != FS_SPARSE_KNOT_BYTES && p->sparse_format != FS_SPARSE_RANK_ROWS))
        return fail(FS_INVALID_ARG, "unknown sparse table format");
      if (p->sparse && p->sparse_format == FS_SPARSE_RANK_ROWS &&
          (p->q != 1 || p->r >= (1ull << 32) || p->n1 - 1 >= (1ull << 31)))
        return fail(FS_INVALID_ARG, "rank rows serve the gap-1 table with R < 2^32, N < 2^31");
      if (p->sparse && p->sparse_format == FS_SPARSE_KNOT_BYTES &&
          (!p->rank || p->q != 1 || p->sparse_ndense != p->n1 || p->r >= (1ull << 32) || p->n1 - 1 >= (1ull << 31)))
        return fail(FS_INVALID_ARG, "knot bytes go with the gap-1 rank directory, one per knot");
      if (p->sparse && p->sparse_format == FS_SPARSE_COUNT &&
          (fs_count_words_bytes(p->r, p->sparse_shift, p->sparse_ndense) == 0 || p->n1 - 1 >= (1ull << 31) ||
           (p->sparse_ndense != 0 && p->sparse_ndense != p->n1)))
        return fail(FS_INVALID_ARG, "count-word parameters out of range");
      if (p->sparse && is_zoned(p->sparse_format)) {
        if (fs_zoned_bytes(p->r, p->sparse_shift, p->sparse_ndense) == 0 || p->r >= (1ull << 32) ||
            (p->sparse_format == FS_SPARSE_ZONED && p->n1 > (1ull << 24)))
          return fail(FS_INVALID_ARG, "zoned table parameters out of range");
        if (p->hot_knot0 > p->n1 || p->hot_knots > p->n1 - p->hot_knot0)
          return fail(FS_INVALID_ARG, "knot window outside the knots");
      }
      if (p->sparse && p->sparse_format == FS_SPARSE_RECORDS8X3 && p->n1 > (1ull << 24))
        return fail(FS_INVALID_ARG, "3-offset records need N+1 <= 2^24");
      if (p->sparse && !is_zoned(p->sparse_format) && p->sparse_format != FS_SPARSE_COUNT &&
          p->sparse_format != FS_SPARSE_KNOT_BYTES && p->sparse_format != FS_SPARSE_RANK_ROWS &&
          (p->sparse_shift < 5 ||
                        p->sparse_shift > (p->sparse_format == FS_SPARSE_TWO_LEVEL    ? 16
                                           : p->sparse_format == FS_SPARSE_RECORDS12 ? kRec12MaxShift
                                           : p->sparse_format == FS_SPARSE_RECORDS8X3 ? kRec3MaxShift
                                                                                      : kRecMaxShift) ||
                        p->sparse_ndense > (p->r >> p->sparse_shift) + 2))
        return fail(FS_INVALID_ARG, "sparse table parameters out of range");
      break;
    case FS_ALGO_BITSET2:
    case FS_ALGO_EYTZINGER:
      if (!p->table) return fail(FS_INVALID_ARG, "plan needs its padded/tree table");
      if (p->pbits < 1 || p->pbits > 31) return fail(FS_INVALID_ARG, "pbits out of range");
      break;
    case FS_ALGO_CLASSIC:
    case FS_ALGO_BITSET1:
    case FS_ALGO_BITSET3:
    case FS_ALGO_OFFSET:
      if (p->pbits < 1 || p->pbits > 32) return fail(FS_INVALID_ARG, "pbits out of range");
      break;
    default:
      return fail(FS_INVALID_ARG, "unknown algorithm");
  }
  return FS_OK;
}

Placement place(const fs_plan* p) {
  Placement pl;
  pl.tune = p->tune;
  const size_t es = p->dtype == FS_F32 ? 4 : 8;
  const size_t budget = smem_budget();
  const bool force_global = p->smem_policy == 1;
  // direct (gap 1): fused records staged in smem when they fit (one 8/16-B
  // conflict-light gather per query); else the rank directory; else K.
  if (p->algorithm == FS_ALGO_DIRECT && p->records && p->q == 1 && !force_global && p->r < (1ull << 32)) {
    const uint64_t rb = (p->r + 1) * (es == 4 ? 8 : 16);
    if (rb <= budget) {
      pl.records = pl.ks = true;
      pl.table_bytes = (uint32_t)rb;
      pl.seg0_src = p->records;
      pl.seg0_bytes = (uint32_t)rb;
      pl.nseg = 1;
      pl.smem = rb;
      pl.flags |= FS_PLACE_SMEM_K;
      return pl;
    }
  }
  const bool use_rank = p->algorithm == FS_ALGO_DIRECT && p->rank != nullptr && p->q == 1;
  // gap 2 over its own directory (16-B words, fs_build_rank2)
  const bool use_rank2 = p->algorithm == FS_ALGO_DIRECT_GAP2 && p->rank != nullptr && p->q == 2;
  // gap q >= 3 over its count directory (8-B words of 16 / 8 buckets, fs_build_countdir)
  const bool use_count = p->algorithm == FS_ALGO_DIRECT_GENERIC && p->rank != nullptr && p->q >= 2 && p->q <= 15;
  const bool use_dir = use_rank || use_rank2 || use_count;
  // the rank directory and a byte per knot, when X does not fit beside the directory
  if (use_rank && p->sparse && p->sparse_format == FS_SPARSE_KNOT_BYTES && !force_global && p->r < (1ull << 32)) {
    const uint64_t db = ((p->r >> 5) + 1) * 8, bb = (p->n1 + 15) & ~15ull;
    if (align128(bb) + db <= budget && align128(p->n1 * es) + db > budget) {
      // the bytes take the X segment's place (at offset 0), the directory follows
      pl.sparse = pl.ks = pl.xs = true;
      pl.x_bytes = (uint32_t)bb;
      pl.table_bytes = (uint32_t)db;
      pl.seg0_src = p->sparse;
      pl.seg0_bytes = (uint32_t)bb;
      pl.seg1_src = p->rank;
      pl.seg1_bytes = (uint32_t)db;
      pl.nseg = 2;
      pl.smem = align128(bb) + db;
      pl.flags |= FS_PLACE_SMEM_K | FS_PLACE_SMEM_SPARSE;
      return pl;
    }
  }
  // zoned records + a window of X (prepare sets them only when the rank
  // directory cannot be staged)
  if (p->algorithm == FS_ALGO_DIRECT && p->sparse && is_zoned(p->sparse_format) && p->q == 1 &&
      !force_global && p->r < (1ull << 32)) {
    const uint64_t tb = fs_zoned_bytes(p->r, p->sparse_shift, p->sparse_ndense);
    const uint64_t xb = p->hot_knots * es;
    if (tb && align128(xb) + tb <= budget) {
      pl.sparse = pl.zoned = pl.ks = true;
      pl.xs = xb > 0;
      pl.x_bytes = (uint32_t)xb;
      pl.table_bytes = (uint32_t)tb;
      if (pl.xs) {
        pl.seg0_src = static_cast<const char*>(p->x) + p->hot_knot0 * es;
        pl.seg0_bytes = (uint32_t)xb;
        pl.seg1_src = p->sparse;
        pl.seg1_bytes = (uint32_t)tb;
        pl.nseg = 2;
        pl.smem = align128(xb) + tb;
      } else {
        pl.seg0_src = p->sparse;
        pl.seg0_bytes = (uint32_t)tb;
        pl.nseg = 1;
        pl.smem = tb;
      }
      pl.flags |= FS_PLACE_SMEM_SPARSE | (pl.xs ? FS_PLACE_SMEM_X : 0);
      return pl;
    }
  }
  // rank directory (+ X) too big for smem: the two-level sparse table, if it fits
  if (p->algorithm == FS_ALGO_DIRECT && p->sparse && !is_zoned(p->sparse_format) && p->q == 1 &&
      p->sparse_format != FS_SPARSE_KNOT_BYTES && p->sparse_format != FS_SPARSE_RANK_ROWS && !force_global &&
      p->r < (1ull << 32) &&
      (p->sparse_format == FS_SPARSE_COUNT || (p->sparse_shift >= 5 && p->sparse_shift <= 16))) {
    const uint64_t xb = p->n1 * es;
    const uint64_t dir_b = ((p->r >> 5) + 1) * 8;
    const uint64_t cfb = p->sparse_format == FS_SPARSE_COUNT
                             ? fs_count_words_bytes(p->r, p->sparse_shift, p->sparse_ndense)
                         : p->sparse_format != FS_SPARSE_TWO_LEVEL
                             ? fs_sparse_rec_bytes(p->sparse_format, p->n1, p->r, p->sparse_shift, p->sparse_ndense)
                             : fs_sparse_bytes(p->n1, p->r, p->sparse_shift, p->sparse_ndense);
    const bool rank_fits = use_rank && align128(xb) + dir_b <= budget;
    // a sparse layout that cannot stage X beside it reads X through L2 like
    // the rank directory does, with a dearer decode: the staged directory
    // wins whenever it fits alone (gaps U[1,5], N+1 = 65535, R / N = 3:
    // 555 vs 270 G queries/s f32, 405 vs 226 f64; profiles/r02/unif_layouts.txt)
    // (count words built with knot offsets are the layout for an X that is not staged)
    const bool sparse_xs = align128(xb) + cfb <= budget && !(p->sparse_format == FS_SPARSE_COUNT && p->sparse_ndense);
    const bool rank_alone_fits = use_rank && dir_b <= budget;
    if (!rank_fits && cfb <= budget && (sparse_xs || !rank_alone_fits)) {
      pl.sparse = pl.ks = true;
      pl.xs = sparse_xs;
      pl.x_bytes = pl.xs ? (uint32_t)xb : 0;
      pl.table_bytes = (uint32_t)cfb;
      if (pl.xs) {
        pl.seg0_src = p->x;
        pl.seg0_bytes = (uint32_t)xb;
        pl.seg1_src = p->sparse;
        pl.seg1_bytes = (uint32_t)cfb;
        pl.nseg = 2;
        pl.smem = align128(xb) + cfb;
        pl.flags |= FS_PLACE_SMEM_X;
      } else {
        pl.seg0_src = p->sparse;
        pl.seg0_bytes = (uint32_t)cfb;
        pl.nseg = 1;
        pl.smem = cfb;
      }
      pl.flags |= FS_PLACE_SMEM_SPARSE;
      return pl;
    }
  }
  // rank directory too big for smem but a hot window is set: stage the window
  if (use_rank && p->hot_words && !force_global && p->r < (1ull << 32) && ((p->r >> 5) + 1) * 8 > budget) {
    const uint64_t xb = p->hot_knots * es, db = p->hot_words * 8;
    if (align128(xb) + db <= budget) {
      pl.hot = pl.xs = pl.ks = true;
      pl.x_bytes = (uint32_t)xb;
      pl.table_bytes = (uint32_t)db;
      pl.seg0_src = static_cast<const char*>(p->x) + p->hot_knot0 * es;
      pl.seg0_bytes = (uint32_t)xb;
      pl.seg1_src = static_cast<const char*>(p->rank) + p->hot_word0 * 8;
      pl.seg1_bytes = (uint32_t)db;
      pl.nseg = 2;
      pl.smem = align128(xb) + db;
      pl.flags |= FS_PLACE_SMEM_HOT;
      return pl;
    }
  }
  switch (use_dir ? -1 : p->algorithm) {
    case -1:  // direct (gap 1 / 2) over its rank directory: X and/or directory in smem
    case FS_ALGO_DIRECT:
    case FS_ALGO_DIRECT_GAP2:
    case FS_ALGO_DIRECT_GENERIC: {
      const uint64_t xb = p->n1 * es;
      const uint64_t kb = use_rank    ? ((p->r >> 5) + 1) * 8
                          : use_rank2 ? ((p->r >> 5) + 1) * 16
                          : use_count ? ((p->r >> countdir_lg(p->q)) + 1) * 8
                                      : (p->r + 1) * 4;
      const void* tab = use_dir ? p->rank : p->table;
      if (force_global || p->r >= (1ull << 32)) break;
      if (align128(xb) + kb <= budget) {
        pl.xs = pl.ks = true;
      } else if (use_dir && kb <= budget) {
        pl.ks = true;  // every query reads the directory, few read X
      } else if (xb <= budget && !use_count) {
        pl.xs = true;
      } else if (kb <= budget) {
        pl.ks = true;
      }
      if (pl.xs) {
        pl.x_bytes = (uint32_t)xb;
        pl.seg0_src = p->x;
        pl.seg0_bytes = (uint32_t)xb;
        pl.nseg = 1;
        pl.flags |= FS_PLACE_SMEM_X;
      }
      if (pl.ks) {
        pl.table_bytes = (uint32_t)kb;
        if (pl.xs) {
          pl.seg1_src = tab;
          pl.seg1_bytes = (uint32_t)kb;
          pl.nseg = 2;
        } else {
          pl.seg0_src = tab;
          pl.seg0_bytes = (uint32_t)kb;
          pl.nseg = 1;
        }
        pl.flags |= FS_PLACE_SMEM_K;
      }
      pl.smem = pl.xs && pl.ks ? align128(pl.x_bytes) + pl.table_bytes : (pl.xs ? pl.x_bytes : pl.table_bytes);
      break;
    }
    case FS_ALGO_DIRECT_CACHE: {
      const uint64_t rb = (p->r + 1) * (es == 4 ? 8 : 16);
      if (!force_global && p->r < (1ull << 32) && rb <= budget) {
        pl.ks = true;
        pl.table_bytes = (uint32_t)rb;
        pl.seg0_src = p->table;
        pl.seg0_bytes = (uint32_t)rb;
        pl.nseg = 1;
        pl.smem = rb;
        pl.flags |= FS_PLACE_SMEM_K;
      }
      break;
    }
    case FS_ALGO_BITSET2: {
      if (force_global) break;
      // the probed nodes are staged by the kernel prologue (Bitset2Probe):
      // as many levels as fit, then bank-private copies of the levels below
      // the conflict-free top six, as far as the remaining budget allows
      pl.top = true;
      pl.b2_shadow = b2_shadow(p->pbits, es);
      const int tb = b2_top_bits(p->pbits, es);
      pl.top_bits = tb;
      pl.flags |= tb == p->pbits ? FS_PLACE_SMEM_X : FS_PLACE_SMEM_TOP;
      pl.b2_l1 = pl.b2_l2 = pl.b2_l3 = std::min(kB2ConflictFree, tb);
      // (only when every level is in smem: with global levels below, the L1
      // the larger carve-out takes away costs more than the conflicts)
      while (kB2Replicate && tb == p->pbits && pl.b2_l2 < tb &&
             b2_smem_bytes(tb, pl.b2_l1, pl.b2_l2 + 1, pl.b2_l2 + 1, es, pl.b2_shadow) <= budget)
        ++pl.b2_l2;
      // f64: the next levels in 16 copies where the rest of the budget allows
      // (a lane pair shares a copy: ~1.3 instead of ~3.5 wavefronts per level;
      // cfg5 N+1 = 1025 281 -> 307, cfg2 158 -> 166 Gq/s).  f32 loses (cfg3
      // 382 -> 364): its issue-bound loop pays more for the two region
      // transitions than it saves (profiles/r01/tune_bitset2_half.txt)
      pl.b2_l3 = pl.b2_l2;
      while (FSG_B2_HALF && es == 8 && kB2Replicate && tb == p->pbits && pl.b2_l2 > pl.b2_l1 && pl.b2_l3 < tb &&
             b2_smem_bytes(tb, pl.b2_l1, pl.b2_l2, pl.b2_l3 + 1, es, pl.b2_shadow) <= budget)
        ++pl.b2_l3;
      pl.x_bytes = (uint32_t)b2_smem_bytes(tb, pl.b2_l1, pl.b2_l2, pl.b2_l3, es, pl.b2_shadow);
      pl.smem = pl.x_bytes;
      break;
    }
    default: {  // classic / bitset1 / bitset3 / offset on X; eytzinger on its tree
      if (force_global) break;
      const bool tree = p->algorithm == FS_ALGO_EYTZINGER;
      // sorted X is staged XOR-swizzled by the kernel prologue (whole 128-B
      // rows, CompareProbe::swz); the Eytzinger tree by the bulk copy
      const uint64_t xb = tree ? ((1ull << p->pbits) - 1) * es : align128(p->n1 * es);
      if (xb <= budget) {
        pl.xs = true;
        pl.x_bytes = (uint32_t)xb;
        if (tree) {
          pl.seg0_src = p->table;
          pl.seg0_bytes = (uint32_t)xb;
          pl.nseg = 1;
        }
        pl.smem = xb;
        pl.flags |= FS_PLACE_SMEM_X;
      }
      break;
    }
  }
  return pl;
}

// Small batches of the direct family skip table staging: when staging the
// tables into every CTA would move more bytes than the queries themselves,
// L2 gathers win (measured on cfg1, 1e6 queries: 122 vs 109 Gq/s).  The
// comparison searches keep their smem placement (their L2 path is far slower).
Placement place_for_batch(const fs_plan* p, uint64_t m) {
  Placement pl = place(p);
  if (pl.top && pl.b2_l2 > pl.b2_l1) {
    // the replicated levels cost every CTA an L2 -> smem copy; a batch smaller
    // than that traffic keeps the plain level-order layout
    const size_t es = p->dtype == FS_F32 ? 4 : 8;
    const uint64_t query_bytes = m * (es + 4);
    if (query_bytes < (uint64_t)pl.smem * sm_count()) {
      pl.b2_l2 = pl.b2_l3 = pl.b2_l1;
      pl.x_bytes = (uint32_t)b2_smem_bytes(pl.top_bits, pl.b2_l1, pl.b2_l2, pl.b2_l3, es, pl.b2_shadow);
      pl.smem = pl.x_bytes;
    }
    return pl;
  }
  const bool direct_family = p->algorithm == FS_ALGO_DIRECT || p->algorithm == FS_ALGO_DIRECT_CACHE ||
                             p->algorithm == FS_ALGO_DIRECT_GAP2 || p->algorithm == FS_ALGO_DIRECT_GENERIC;
  if (!direct_family || pl.smem == 0 || p->smem_policy != 0 || pl.hot) return pl;
  const uint64_t query_bytes = m * ((p->dtype == FS_F32 ? 4 : 8) + 4);
  const uint64_t staging_bytes = (uint64_t)pl.smem * sm_count() / 2;
  if (query_bytes >= staging_bytes) return pl;
  fs_plan g = *p;
  g.smem_policy = 1;
  Placement gl = place(&g);
  gl.tune = pl.tune;
  return gl;
}

// ---------------------------------------------------------------------------
// Launch
// ---------------------------------------------------------------------------
#ifndef FSG_UNROLL
#define FSG_UNROLL 3  // 4-query groups in flight per thread per iteration (f32; 3 > 4 > 2 measured on cfg3)
#endif
#ifndef FSG_UNROLL_F64
#define FSG_UNROLL_F64 2  // f64: same bytes in flight, half the live registers
#endif
#ifndef FSG_UNROLL_F64_SMEM
#define FSG_UNROLL_F64_SMEM 3
#endif
// group records: unroll 2 and (see BoundedFor) the 1024-thread register
// bound measure best (profiles/r01/tune_sparse_records.txt)
#ifndef FSG_UNROLL_F64_REC
#define FSG_UNROLL_F64_REC 2
#endif
#ifndef FSG_REC_BOUNDED
#define FSG_REC_BOUNDED 1
#endif
template <typename T>
constexpr int kUnroll = sizeof(T) == 8 ? FSG_UNROLL_F64 : FSG_UNROLL;
// Per-probe override: f64 probes whose whole table sits in smem have short,
// latency-light chains and take one more 4-query group in flight
// (profiles/r01/tune_unroll_f64.txt: records +2.6%, sparse with X in smem
// +3.6%; the L2-gathering and bitset2 probes lose with it).
// Queries per vector group: 8 for f32 queries with int32 outputs (one 32-B
// load and one 32-B store per group) when FSG_F32_VW8, else 4.
#ifndef FSG_F32_VW8
#define FSG_F32_VW8 1
#endif
#ifndef FSG_F32_I64_VW8
#define FSG_F32_I64_VW8 0
#endif
template <typename T, typename OutT, typename Probe>
struct VecWidthFor {
  static constexpr int value =
      (FSG_F32_VW8 && sizeof(T) == 4 && (sizeof(OutT) == 4 || FSG_F32_I64_VW8)) ? 8 : 4;
};
// 8-query groups in flight per thread: one for the smem-resident probes
// (cfg3 direct 797 -> 832 Gq/s, the torch copy ceiling; two groups: 720),
// two for the L2-gather rank directory and bitset2 (cfg4 347 -> 373,
// bitset2 cfg3 364 -> 382); profiles/r01/tune_vw8.txt.
#ifndef FSG_UNROLL_VW8
#define FSG_UNROLL_VW8 1
#endif
template <typename Probe>
struct UnrollVW8For {
  static constexpr int value = FSG_UNROLL_VW8;
};
#ifndef FSG_UNROLL_VW8_RANK
#define FSG_UNROLL_VW8_RANK 2
#endif
template <typename J, bool XS, bool DS>
struct UnrollVW8For<RankProbe<float, J, XS, DS>> {
  static constexpr int value = FSG_UNROLL_VW8_RANK;
};
template <>
struct UnrollVW8For<HotRankProbe<float>> {
  static constexpr int value = FSG_UNROLL_VW8_RANK;
};
template <>
struct UnrollVW8For<RankRowsProbe<float>> {
  static constexpr int value = FSG_UNROLL_VW8_RANK;
};
#ifndef FSG_UNROLL_VW8_ZONED
#define FSG_UNROLL_VW8_ZONED 1  // one 8-query group per thread (2: cfg4 465 -> 448 Gq/s)
#endif
template <bool STRIPED>
struct UnrollVW8For<ZonedProbe<float, STRIPED>> {
  static constexpr int value = FSG_UNROLL_VW8_ZONED;
};
template <bool TOP, bool DEEP>
struct UnrollVW8For<Bitset2Probe<float, TOP, DEEP>> {
  static constexpr int value = 2;
};
template <typename T, typename Probe>
struct UnrollFor {
  static constexpr int value = kUnroll<T>;
};
template <typename J>
struct UnrollFor<double, CacheProbe<double, J, true>> {
  static constexpr int value = 3;
};
// f32 records with int64 outputs (the 4-query-group path): two groups
// (cfg3 487 -> 500 Gq/s; profiles/r01/tune_i64_unroll.txt)
template <typename J>
struct UnrollFor<float, CacheProbe<float, J, true>> {
  static constexpr int value = 2;
};
template <bool DENSE>
struct UnrollFor<double, SparseProbe<double, true, DENSE>> {
  static constexpr int value = FSG_UNROLL_F64_SMEM;
};
template <int SLOTS, bool XS, bool OVF>
struct UnrollFor<double, SparseRecProbe<double, SLOTS, XS, OVF>> {
  static constexpr int value = FSG_UNROLL_F64_REC;
};
// count words: three 4-query groups per thread, the word loads of a whole
// group in flight (cfg2 486 -> 514, cfg5 N+1 = 1025 515 -> 550 Gq/s over two
// groups of two loads; four groups 453; profiles/r02/count_words.txt)
#ifndef FSG_UNROLL_F64_COUNT
#define FSG_UNROLL_F64_COUNT 3
#endif
template <int XM>
struct UnrollFor<double, CountWordProbe<double, XM>> {
  static constexpr int value = FSG_UNROLL_F64_COUNT;
};
// The light three-offset probe takes a third group with int32 outputs (cfg2
// 459 -> 470 Gq/s; int64 outputs 370 -> 355 and the other probes lose with
// it: profiles/r01/tune_sparse_records.txt).
template <typename T, typename Probe, typename OutT>
struct UnrollOutFor {
  static constexpr int value = UnrollFor<T, Probe>::value;
};
#ifndef FSG_UNROLL_REC3
#define FSG_UNROLL_REC3 3
#endif
#ifndef FSG_UNROLL_REC12
#define FSG_UNROLL_REC12 FSG_UNROLL_F64_REC
#endif
template <bool XS, bool OVF>
struct UnrollOutFor<double, SparseRecProbe<double, 3, XS, OVF>, int32_t> {
  static constexpr int value = FSG_UNROLL_REC3;
};
template <bool XS, bool OVF>
struct UnrollOutFor<double, SparseRecProbe<double, 8, XS, OVF>, int32_t> {
  static constexpr int value = FSG_UNROLL_REC12;
};
// Probes launched through the 1024-thread-bounded entry point: the sparse
// probe with X in smem exceeds 64 registers with int64 outputs and gains
// from 1024-thread CTAs despite small spills (cfg2 int64 222 -> 264 Gq/s);
// the f64 records probe loses (399 -> 335), so the default stays unbounded
// (profiles/r01/tune_launch_bounds.txt).
// Group records: bounded, except the 8-B probe with int64 outputs (it fits
// in 64 registers unbounded and loses 403 -> 370 Gq/s on cfg5 N+1 = 1025
// when bounded; the 16-B overflow probe needs 69 unbounded, cfg2 304 -> 390).
template <typename T, typename Probe, typename OutT>
struct BoundedFor {
  static constexpr bool value = false;
};
template <typename T, bool DENSE, typename OutT>
struct BoundedFor<T, SparseProbe<T, true, DENSE>, OutT> {
  static constexpr bool value = true;
};
// bitset2 with its top levels in smem runs one 1024-thread CTA per SM: the
// 16-copy region's address arithmetic would otherwise take it past 64
// registers (66-72) and halve the resident warps.
#ifndef FSG_B2_BOUNDED
#define FSG_B2_BOUNDED 1
#endif
template <typename T, bool DEEP, bool SHADOW, typename OutT>
struct BoundedFor<T, Bitset2Probe<T, true, DEEP, SHADOW>, OutT> {
  static constexpr bool value = FSG_B2_BOUNDED;
};
#ifndef FSG_ZONED_BOUNDED
#define FSG_ZONED_BOUNDED 1
#endif
template <typename T, bool STRIPED, typename OutT>
struct BoundedFor<T, ZonedProbe<T, STRIPED>, OutT> {
  static constexpr bool value = FSG_ZONED_BOUNDED;
};
// knot bytes beside the directory: 1024-thread CTAs, two 8-query groups per
// thread for f32, two queries per load phase (uniform-gap N+1 = 65535: f32 625
// -> 680, f64 467 -> 493 Gq/s over the unbounded / one-group / four-query
// build; profiles/r02/knot_bytes.txt)
#ifndef FSG_RANKBYTES_BOUNDED
#define FSG_RANKBYTES_BOUNDED 1
#endif
template <typename T, typename OutT>
struct BoundedFor<T, RankBytesProbe<T>, OutT> {
  static constexpr bool value = FSG_RANKBYTES_BOUNDED;
};
#ifndef FSG_UNROLL_VW8_RANKBYTES
#define FSG_UNROLL_VW8_RANKBYTES 2
#endif
template <>
struct UnrollVW8For<RankBytesProbe<float>> {
  static constexpr int value = FSG_UNROLL_VW8_RANKBYTES;
};
#ifndef FSG_UNROLL_F64_RANKBYTES
#define FSG_UNROLL_F64_RANKBYTES FSG_UNROLL_F64
#endif
template <>
struct UnrollFor<double, RankBytesProbe<double>> {
  static constexpr int value = FSG_UNROLL_F64_RANKBYTES;
};
#ifndef FSG_COUNT_BOUNDED
#define FSG_COUNT_BOUNDED 1
#endif
template <typename T, int XM, typename OutT>
struct BoundedFor<T, CountWordProbe<T, XM>, OutT> {
  static constexpr bool value = FSG_COUNT_BOUNDED;
};
template <typename T, int SLOTS, bool XS, bool OVF, typename OutT>
struct BoundedFor<T, SparseRecProbe<T, SLOTS, XS, OVF>, OutT> {
  static constexpr bool value = FSG_REC_BOUNDED && !(SLOTS == 2 && sizeof(OutT) == 8);
};



// Launch geometry per (device, kernel, dynamic smem, candidate set), and the
// largest dynamic-smem attribute set per (device, kernel): process-wide,
// idempotent caches so a launch costs no runtime queries after the first
// (the occupancy calculator and cudaFuncSetAttribute were ~10 us per call).
std::mutex g_geo_mu;
std::map<std::tuple<const void*, int, size_t, int>, std::pair<int, int>> g_geo;
std::map<std::pair<const void*, int>, size_t> g_smem_attr;

int launch_geometry(const void* fn, size_t smem, int mode, int* threads_out, int* per_sm_out) {
  int dev = 0;
  FS_CUDA(cudaGetDevice(&dev));
  std::lock_guard<std::mutex> lock(g_geo_mu);
  const auto key = std::make_tuple(fn, dev, smem, mode);
  auto it = g_geo.find(key);
  if (it != g_geo.end()) {
    *threads_out = it->second.first;
    *per_sm_out = it->second.second;
    return FS_OK;
  }
  if (smem > 0) {
    size_t& cur = g_smem_attr[std::make_pair(fn, dev)];
    if (smem > cur) {
      FS_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
      cur = smem;
    }
  }
  const int cands_big[] = {1024, 512, 256, 128};
  const int cands_small[] = {512, 256, 128, 0};
  const int cands_tuned[] = {mode > 0 ? mode : 0, 0, 0, 0};
  const int* cands = mode > 0 ? cands_tuned : (mode == -1 ? cands_big : cands_small);
  int threads = 0, per_sm = 0;
  for (int c = 0; c < 4 && cands[c]; ++c) {
    FS_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, cands[c], smem));
    if (per_sm >= 1) {
      threads = cands[c];
      break;
    }
  }
  if (per_sm < 1) return fail(FS_TOO_LARGE, "search kernel does not fit on an SM with this table placement");
  g_geo[key] = std::make_pair(threads, per_sm);
  *threads_out = threads;
  *per_sm_out = per_sm;
  return FS_OK;
}

template <typename T, typename OutT, typename Probe>
int launch_probe(const DevPlan<T>& dp, const Placement& pl, const T* z, uint64_t m, OutT* out,
                 unsigned long long* first_bad, uint64_t base, cudaStream_t st) {
  constexpr int VW = VecWidthFor<T, OutT, Probe>::value;
  constexpr int kU = VW == 8 ? UnrollVW8For<Probe>::value : UnrollOutFor<T, Probe, OutT>::value;
  auto kern = [] {
    if constexpr (BoundedFor<T, Probe, OutT>::value) return search_kernel_1k<T, OutT, Probe, kU, VW>;
    else return search_kernel<T, OutT, Probe, kU, VW>;
  }();
  const size_t smem = pl.smem;
  // Kernels that stage tables in shared memory run best with ~1024 threads
  // per SM in one wide CTA (measured on cfg3: 1x1024 95% of HBM peak vs
  // 3x512 86%; fewer resident warps contend less for the smem crossbar the
  // table gathers share with the stream).  L2-gather kernels use 512-thread
  // CTAs at full occupancy (geometry-insensitive within 1%); with a hot
  // window, 1024-thread CTAs at full occupancy (cfg4 390 -> 405 Gq/s;
  // profiles/r01/tune_tail_records_rejected.txt).
  const bool smem_resident = pl.smem > 0 && !pl.hot;  // a hot window still gathers through L2
  const int mode = (pl.tune & 0xfff) ? (pl.tune & 0xfff) : (smem_resident || pl.hot ? -1 : -2);
  int threads = 0, per_sm = 0;
  int rc = launch_geometry(reinterpret_cast<const void*>(kern), smem, mode, &threads, &per_sm);
  if (rc) return rc;
  int cap = (pl.tune >> 12) & 0xff;
  if (!pl.tune && smem_resident) cap = std::max(1, 1024 / threads);  // ~1024 threads per SM
  if (cap && per_sm > cap) per_sm = cap;

  StreamShape sh;
  sh.m = m;
  sh.base = base;
  const uintptr_t za = reinterpret_cast<uintptr_t>(z);
  constexpr uint32_t va = VecLoad<T, VW>::kAlign;  // query groups start va-aligned
  uint64_t head = ((va - (za & (va - 1))) & (va - 1)) / sizeof(T);
  if (head > m) head = m;
  sh.head = head;
  sh.nvec = (m - head) / VW;
  DevPlan<T> d = dp;
  const uintptr_t oa = reinterpret_cast<uintptr_t>(out) + head * sizeof(OutT);
  d.out_vec_ok = (oa & 15) ? 0 : (oa & 31) ? 1 : 2;

  const uint64_t full = (uint64_t)per_sm * sm_count();
  // one group per thread at least: a small batch spreads over every SM
  // instead of filling a few CTAs kU groups deep (cfg1 bitset2 80 -> see
  // profiles/r01/tune_vw8.txt)
  uint64_t want = (sh.nvec + (uint64_t)threads - 1) / (uint64_t)threads;
  const int grid = (int)std::max<uint64_t>(1, std::min<uint64_t>(full, want));

  StageSeg s0{nullptr, pl.seg0_src, pl.seg0_bytes};
  StageSeg s1{nullptr, pl.seg1_src, pl.seg1_bytes};
  kern<<<grid, threads, smem, st>>>(z, out, sh, d, first_bad, pl.merge, s0, s1, pl.nseg);
  FS_CUDA(cudaGetLastError());
  return FS_OK;
}

template <typename T>
DevPlan<T> make_devplan(const fs_plan* p, const Placement& pl) {
  DevPlan<T> d{};
  d.x = static_cast<const T*>(p->x);
  d.table = p->table;
  d.rank = static_cast<const uint2*>(p->rank);
  d.rows = p->sparse && p->sparse_format == FS_SPARSE_RANK_ROWS ? p->sparse : nullptr;
  d.n1 = p->n1;
  d.r = p->r;
  d.h = (T)p->h;
  d.x0 = (T)p->x0;
  d.xn = (T)p->xn;
  d.q = p->q;
  d.pbits = p->pbits;
  d.top_bits = pl.top_bits;
  d.b2_l1 = pl.b2_l1;
  d.b2_l2 = pl.b2_l2;
  d.b2_l3 = pl.b2_l3;
  // subtree records apply only to the staged-top split they were built for
  const bool deep = pl.top && p->b2_deep && p->b2_deep_top == pl.top_bits &&
                    p->b2_deep_k == b2_deep_k(p->dtype);
  d.b2_deep = deep ? p->b2_deep : nullptr;
  d.b2_deep_k = deep ? p->b2_deep_k : 0;
  const uint64_t n = p->n1 - 1;
  d.off_f = (uint32_t)((n + 1) >> 1);
  d.off_s = (uint32_t)(n + 1 - d.off_f);
  d.off_j = (uint32_t)(bit_length(n + 1) - 1);
  d.sparse_shift = p->sparse_shift;
  d.sparse_ndense = p->sparse_ndense;
  d.hot_w0 = (uint32_t)p->hot_word0;
  d.hot_nw = pl.hot ? (uint32_t)p->hot_words : 0;
  d.hot_t0 = (uint32_t)p->hot_knot0;
  d.hot_nt = pl.hot || pl.zoned ? (uint32_t)p->hot_knots : 0;
  d.x_smem_bytes = pl.xs || pl.top ? pl.x_bytes : 0;
  d.table_smem_bytes = pl.ks ? pl.table_bytes : 0;
  // With only K staged it sits at offset 0.
  if (!pl.xs && !pl.top) d.x_smem_bytes = 0;
  return d;
}

template <typename T, typename OutT, typename J, int GAP>
int dispatch_direct(const DevPlan<T>& d, const Placement& pl, const T* z, uint64_t m, OutT* out,
                    unsigned long long* fb, uint64_t base, cudaStream_t st) {
  if (pl.xs && pl.ks) return launch_probe<T, OutT, DirectProbe<T, J, GAP, true, true>>(d, pl, z, m, out, fb, base, st);
  if (pl.xs) return launch_probe<T, OutT, DirectProbe<T, J, GAP, true, false>>(d, pl, z, m, out, fb, base, st);
  if (pl.ks) return launch_probe<T, OutT, DirectProbe<T, J, GAP, false, true>>(d, pl, z, m, out, fb, base, st);
  return launch_probe<T, OutT, DirectProbe<T, J, GAP, false, false>>(d, pl, z, m, out, fb, base, st);
}

// gap-q count directory (B bits per bucket); X staged only beside a staged directory
template <typename T, typename OutT, int B>
int dispatch_countdir(const DevPlan<T>& d, const Placement& pl, const T* z, uint64_t m, OutT* out,
                      unsigned long long* fb, uint64_t base, cudaStream_t st) {
  if (pl.xs && pl.ks) return launch_probe<T, OutT, CountDirProbe<T, B, true, true>>(d, pl, z, m, out, fb, base, st);
  if (pl.ks) return launch_probe<T, OutT, CountDirProbe<T, B, false, true>>(d, pl, z, m, out, fb, base, st);
  return launch_probe<T, OutT, CountDirProbe<T, B, false, false>>(d, pl, z, m, out, fb, base, st);
}

template <typename T, typename OutT, int SLOTS>
int dispatch_records(const DevPlan<T>& d, const Placement& pl, bool ovf, const T* z, uint64_t m, OutT* out,
                     unsigned long long* fb, uint64_t base, cudaStream_t st) {
  if (ovf) {
    if (pl.xs) return launch_probe<T, OutT, SparseRecProbe<T, SLOTS, true, true>>(d, pl, z, m, out, fb, base, st);
    return launch_probe<T, OutT, SparseRecProbe<T, SLOTS, false, true>>(d, pl, z, m, out, fb, base, st);
  }
  if (pl.xs) return launch_probe<T, OutT, SparseRecProbe<T, SLOTS, true, false>>(d, pl, z, m, out, fb, base, st);
  return launch_probe<T, OutT, SparseRecProbe<T, SLOTS, false, false>>(d, pl, z, m, out, fb, base, st);
}

template <typename T, typename OutT, int ALGO>
int dispatch_compare(const DevPlan<T>& d, const Placement& pl, const T* z, uint64_t m, OutT* out,
                     unsigned long long* fb, uint64_t base, cudaStream_t st) {
  if (pl.xs) return launch_probe<T, OutT, CompareProbe<T, ALGO, true>>(d, pl, z, m, out, fb, base, st);
  return launch_probe<T, OutT, CompareProbe<T, ALGO, false>>(d, pl, z, m, out, fb, base, st);
}

template <typename T, typename OutT>
int dispatch(const fs_plan* p, const Placement& pl, const T* z, uint64_t m, OutT* out, unsigned long long* fb,
             uint64_t base, cudaStream_t st) {
  const DevPlan<T> d = make_devplan<T>(p, pl);
  const bool wide = p->r >= (1ull << 32);
  switch (p->algorithm) {
    case FS_ALGO_DIRECT:
      if (pl.records) return launch_probe<T, OutT, CacheProbe<T, uint32_t, true>>(d, pl, z, m, out, fb, base, st);
      if (pl.hot) return launch_probe<T, OutT, HotRankProbe<T>>(d, pl, z, m, out, fb, base, st);
      if (pl.zoned && p->sparse_format == FS_SPARSE_ZONED_RANK)
        return launch_probe<T, OutT, ZonedProbe<T, true>>(d, pl, z, m, out, fb, base, st);
      if (pl.zoned) return launch_probe<T, OutT, ZonedProbe<T>>(d, pl, z, m, out, fb, base, st);
      if (pl.sparse && p->sparse_format == FS_SPARSE_KNOT_BYTES)
        return launch_probe<T, OutT, RankBytesProbe<T>>(d, pl, z, m, out, fb, base, st);
      if (pl.sparse && p->sparse_format == FS_SPARSE_COUNT) {
        if (pl.xs) return launch_probe<T, OutT, CountWordProbe<T, 1>>(d, pl, z, m, out, fb, base, st);
        if (p->sparse_ndense) return launch_probe<T, OutT, CountWordProbe<T, 2>>(d, pl, z, m, out, fb, base, st);
        return launch_probe<T, OutT, CountWordProbe<T, 0>>(d, pl, z, m, out, fb, base, st);
      }
      if (pl.sparse && p->sparse_format == FS_SPARSE_RECORDS)
        return dispatch_records<T, OutT, 6>(d, pl, p->sparse_ndense != 0, z, m, out, fb, base, st);
      if (pl.sparse && p->sparse_format == FS_SPARSE_RECORDS8X3)
        return dispatch_records<T, OutT, 3>(d, pl, p->sparse_ndense != 0, z, m, out, fb, base, st);
      if (pl.sparse && p->sparse_format == FS_SPARSE_RECORDS12)
        return dispatch_records<T, OutT, 8>(d, pl, p->sparse_ndense != 0, z, m, out, fb, base, st);
      if (pl.sparse && p->sparse_format == FS_SPARSE_RECORDS8)
        return dispatch_records<T, OutT, 2>(d, pl, p->sparse_ndense != 0, z, m, out, fb, base, st);
      if (pl.sparse) {
        if (p->sparse_ndense) {
          if (pl.xs) return launch_probe<T, OutT, SparseProbe<T, true, true>>(d, pl, z, m, out, fb, base, st);
          return launch_probe<T, OutT, SparseProbe<T, false, true>>(d, pl, z, m, out, fb, base, st);
        }
        if (pl.xs) return launch_probe<T, OutT, SparseProbe<T, true, false>>(d, pl, z, m, out, fb, base, st);
        return launch_probe<T, OutT, SparseProbe<T, false, false>>(d, pl, z, m, out, fb, base, st);
      }
      // nothing staged and 16-B rank rows built: one gather brings the directory word and its knots' bytes
      if (d.rows && !wide && pl.smem == 0)
        return launch_probe<T, OutT, RankRowsProbe<T>>(d, pl, z, m, out, fb, base, st);
      if (p->rank && p->q == 1) {
        if (wide) return launch_probe<T, OutT, RankProbe<T, uint64_t, false, false>>(d, pl, z, m, out, fb, base, st);
        if (pl.xs && pl.ks) return launch_probe<T, OutT, RankProbe<T, uint32_t, true, true>>(d, pl, z, m, out, fb, base, st);
        if (pl.xs) return launch_probe<T, OutT, RankProbe<T, uint32_t, true, false>>(d, pl, z, m, out, fb, base, st);
        if (pl.ks) return launch_probe<T, OutT, RankProbe<T, uint32_t, false, true>>(d, pl, z, m, out, fb, base, st);
        return launch_probe<T, OutT, RankProbe<T, uint32_t, false, false>>(d, pl, z, m, out, fb, base, st);
      }
      if (wide) return launch_probe<T, OutT, DirectProbe<T, uint64_t, 1, false, false>>(d, pl, z, m, out, fb, base, st);
      return dispatch_direct<T, OutT, uint32_t, 1>(d, pl, z, m, out, fb, base, st);
    case FS_ALGO_DIRECT_GAP2:
      if (wide) return launch_probe<T, OutT, DirectProbe<T, uint64_t, 2, false, false>>(d, pl, z, m, out, fb, base, st);
      if (p->rank && p->q == 2) {
        if (pl.xs && pl.ks) return launch_probe<T, OutT, Rank2Probe<T, true, true>>(d, pl, z, m, out, fb, base, st);
        if (pl.xs) return launch_probe<T, OutT, Rank2Probe<T, true, false>>(d, pl, z, m, out, fb, base, st);
        if (pl.ks) return launch_probe<T, OutT, Rank2Probe<T, false, true>>(d, pl, z, m, out, fb, base, st);
        return launch_probe<T, OutT, Rank2Probe<T, false, false>>(d, pl, z, m, out, fb, base, st);
      }
      return dispatch_direct<T, OutT, uint32_t, 2>(d, pl, z, m, out, fb, base, st);
    case FS_ALGO_DIRECT_GENERIC:
      if (wide) return launch_probe<T, OutT, DirectProbe<T, uint64_t, 3, false, false>>(d, pl, z, m, out, fb, base, st);
      if (p->rank && p->q >= 2 && p->q <= 3) return dispatch_countdir<T, OutT, 2>(d, pl, z, m, out, fb, base, st);
      if (p->rank && p->q >= 4 && p->q <= 15) return dispatch_countdir<T, OutT, 4>(d, pl, z, m, out, fb, base, st);
      return dispatch_direct<T, OutT, uint32_t, 3>(d, pl, z, m, out, fb, base, st);
    case FS_ALGO_DIRECT_CACHE:
      if (wide) return launch_probe<T, OutT, CacheProbe<T, uint64_t, false>>(d, pl, z, m, out, fb, base, st);
      if (pl.ks) return launch_probe<T, OutT, CacheProbe<T, uint32_t, true>>(d, pl, z, m, out, fb, base, st);
      return launch_probe<T, OutT, CacheProbe<T, uint32_t, false>>(d, pl, z, m, out, fb, base, st);
    case FS_ALGO_BITSET2:
      if constexpr (sizeof(T) == 8) {
        if (pl.top && pl.b2_shadow && d.b2_deep)
          return launch_probe<T, OutT, Bitset2Probe<T, true, true, true>>(d, pl, z, m, out, fb, base, st);
        if (pl.top && pl.b2_shadow)
          return launch_probe<T, OutT, Bitset2Probe<T, true, false, true>>(d, pl, z, m, out, fb, base, st);
      }
      if (pl.top && d.b2_deep) return launch_probe<T, OutT, Bitset2Probe<T, true, true>>(d, pl, z, m, out, fb, base, st);
      if (pl.top) return launch_probe<T, OutT, Bitset2Probe<T, true>>(d, pl, z, m, out, fb, base, st);
      return launch_probe<T, OutT, Bitset2Probe<T, false>>(d, pl, z, m, out, fb, base, st);
    case FS_ALGO_CLASSIC: return dispatch_compare<T, OutT, 0>(d, pl, z, m, out, fb, base, st);
    case FS_ALGO_BITSET1: return dispatch_compare<T, OutT, 1>(d, pl, z, m, out, fb, base, st);
    case FS_ALGO_BITSET3: return dispatch_compare<T, OutT, 3>(d, pl, z, m, out, fb, base, st);
    case FS_ALGO_OFFSET: return dispatch_compare<T, OutT, 4>(d, pl, z, m, out, fb, base, st);
    case FS_ALGO_EYTZINGER: return dispatch_compare<T, OutT, 5>(d, pl, z, m, out, fb, base, st);
  }
  return fail(FS_INVALID_ARG, "unknown algorithm");
}

// Launch the search over z[0..m) (global positions base..base+m); no memset.
int launch_search(const fs_plan* p, const Placement& pl, const void* z, uint64_t m, void* out, int out_bytes,
                  unsigned long long* fb, uint64_t base, cudaStream_t st) {
  if (m == 0) return FS_OK;
  if (p->dtype == FS_F32) {
    if (out_bytes == 4)
      return dispatch<float, int32_t>(p, pl, static_cast<const float*>(z), m, static_cast<int32_t*>(out), fb, base, st);
    return dispatch<float, int64_t>(p, pl, static_cast<const float*>(z), m, static_cast<int64_t*>(out), fb, base, st);
  }
  if (out_bytes == 4)
    return dispatch<double, int32_t>(p, pl, static_cast<const double*>(z), m, static_cast<int32_t*>(out), fb, base, st);
  return dispatch<double, int64_t>(p, pl, static_cast<const double*>(z), m, static_cast<int64_t*>(out), fb, base, st);
}

int check_search_args(const fs_plan* p, const void* z, uint64_t m, const void* out, int out_bytes,
                      const void* fb) {
  int rc = validate_plan(p);
  if (rc) return rc;
  if (out_bytes != 4 && out_bytes != 8) return fail(FS_INVALID_ARG, "out_bytes must be 4 (int32) or 8 (int64)");
  if (!fb) return fail(FS_INVALID_ARG, "first_bad word is NULL");
  if (m && (!z || !out)) return fail(FS_INVALID_ARG, "query/output pointer is NULL");
  const size_t es = p->dtype == FS_F32 ? 4 : 8;
  if (reinterpret_cast<uintptr_t>(z) % es || reinterpret_cast<uintptr_t>(out) % out_bytes)
    return fail(FS_INVALID_ARG, "query/output arrays must be element-aligned");
  return FS_OK;
}

// ---------------------------------------------------------------------------
// Certification driver
// ---------------------------------------------------------------------------
template <typename T>
int certify_impl(const T* x, uint64_t n1, int qbits, int q, CertStatus* st, T* h_out, T* h_start_out,
                 uint64_t* r_out, uint32_t* incr_out, int64_t* pos_out, cudaStream_t s) {
  constexpr int NT = 256;
  const uint64_t n = n1 - 1;
  const uint64_t basis = std::min<uint64_t>((uint64_t)q, n);
  const int grid = grid_1d(n1, NT);
  cert_init_kernel<<<1, 1, 0, s>>>(st);
  certify_prep<T, NT><<<grid, NT, 0, s>>>(x, n1, (uint64_t)q, basis, st);
  certify_finalize<T><<<1, 1, 0, s>>>(x, n1, qbits, st);
  certify_check<T, NT><<<grid, NT, 0, s>>>(x, n1, (uint64_t)q, st);
  FS_CUDA(cudaGetLastError());
  CertStatus hs;
  for (;;) {
    FS_CUDA(cudaMemcpyAsync(&hs, st, sizeof(hs), cudaMemcpyDeviceToHost, s));
    FS_CUDA(cudaStreamSynchronize(s));
    if (hs.status != 0 || hs.fail == 0) break;
    certify_grow<T><<<1, 1, 0, s>>>(x, n1, qbits, st);
    certify_check<T, NT><<<grid, NT, 0, s>>>(x, n1, (uint64_t)q, st);
    FS_CUDA(cudaGetLastError());
  }
  if (h_out) *h_out = (T)hs.h;
  if (h_start_out) *h_start_out = (T)hs.h_start;
  if (incr_out) *incr_out = hs.increments;
  if (hs.status == 1) {
    if (pos_out) *pos_out = (int64_t)hs.collide_pos;
    return fail(FS_NOT_DISTINGUISHABLE, "rounded offsets collide");
  }
  if (hs.status == 2) return fail(FS_OVERFLOW, "floor(H * D_N) >= 2**qbits");
  if (r_out) *r_out = (uint64_t)hs.r_float;
  return FS_OK;
}

}  // namespace

// ===========================================================================
// C-ABI
// ===========================================================================
extern "C" {

#ifndef FSG_SRC_SHA16
#define FSG_SRC_SHA16 "unknown"
#endif
const char* fs_version(void) { return "fsgpu 0.1.0 (sm_100a) src " FSG_SRC_SHA16; }

const char* fs_last_error(void) { return g_last_error.c_str(); }

size_t fs_workspace_bytes(void) { return (sizeof(CertStatus) + 255) & ~(size_t)255; }

int fs_certify(int32_t dtype, const void* x_dev, uint64_t n1, int32_t qbits, int32_t q, void* ws_dev, void* h_out,
               void* h_start_out, uint64_t* r_out, uint32_t* increments_out, int64_t* pos_out, void* stream) {
  if (qbits != 32 && qbits != 64) return fail(FS_INVALID_ARG, "qbits must be 32 or 64");
  if (q < 1) return fail(FS_INVALID_ARG, "gap must be >= 1");
  if (n1 < 2) return fail(FS_INVALID_ARG, "a partition needs at least two values");
  if (!x_dev || !ws_dev) return fail(FS_INVALID_ARG, "NULL pointer");
  auto* st = static_cast<CertStatus*>(ws_dev);
  if (dtype == FS_F32)
    return certify_impl<float>(static_cast<const float*>(x_dev), n1, qbits, q, st, static_cast<float*>(h_out),
                               static_cast<float*>(h_start_out), r_out, increments_out, pos_out, as_stream(stream));
  if (dtype == FS_F64)
    return certify_impl<double>(static_cast<const double*>(x_dev), n1, qbits, q, st, static_cast<double*>(h_out),
                                static_cast<double*>(h_start_out), r_out, increments_out, pos_out, as_stream(stream));
  return fail(FS_INVALID_ARG, "dtype must be FS_F32 or FS_F64");
}

int fs_build_table(int32_t dtype, const void* x_dev, uint64_t n1, double h, uint64_t r, int32_t q, uint32_t* k_dev,
                   uint64_t* f_scratch_dev, void* ws_dev, void* stream) {
  if (n1 < 2) return fail(FS_INVALID_ARG, "a partition needs at least two values");
  if (n1 - 1 >= (1ull << 32)) return fail(FS_INVALID_ARG, "table entries are 32-bit; partition is too large");
  if (q < 1) return fail(FS_INVALID_ARG, "gap must be >= 1");
  if (!x_dev || !k_dev || !f_scratch_dev || !ws_dev) return fail(FS_INVALID_ARG, "NULL pointer");
  cudaStream_t s = as_stream(stream);
  auto* st = static_cast<CertStatus*>(ws_dev);
  cert_init_kernel<<<1, 1, 0, s>>>(st);
  const int g = grid_1d(n1, 256);
  if (dtype == FS_F32)
    knot_buckets_kernel<float><<<g, 256, 0, s>>>(static_cast<const float*>(x_dev), n1, (float)h, r, f_scratch_dev, st);
  else if (dtype == FS_F64)
    knot_buckets_kernel<double><<<g, 256, 0, s>>>(static_cast<const double*>(x_dev), n1, h, r, f_scratch_dev, st);
  else
    return fail(FS_INVALID_ARG, "dtype must be FS_F32 or FS_F64");
  FS_CUDA(cudaGetLastError());
  unsigned long long inconsistent = 0;
  FS_CUDA(cudaMemcpyAsync(&inconsistent, &st->inconsistent, sizeof(inconsistent), cudaMemcpyDeviceToHost, s));
  FS_CUDA(cudaStreamSynchronize(s));
  if (inconsistent) return fail(FS_INCONSISTENT, "(h, r) pair is inconsistent with this partition");
  constexpr int NT = 256, ITEMS = 16;
  const uint64_t tiles = (r + 1 + (uint64_t)NT * ITEMS - 1) / ((uint64_t)NT * ITEMS);
  const int grid = (int)std::min<uint64_t>(tiles, (uint64_t)sm_count() * 8);
  if (q == 1)
    fill_table_kernel<NT, ITEMS, false><<<grid, NT, 0, s>>>(f_scratch_dev, n1, r, k_dev);
  else
    fill_table_kernel<NT, ITEMS, true><<<grid, NT, 0, s>>>(f_scratch_dev, n1, r, k_dev);
  FS_CUDA(cudaGetLastError());
  return FS_OK;
}

int fs_knot_buckets(int32_t dtype, const void* x_dev, uint64_t n1, double h, uint64_t* f_dev, void* stream) {
  if (!x_dev || !f_dev || n1 < 1) return fail(FS_INVALID_ARG, "bad arguments");
  cudaStream_t s = as_stream(stream);
  const int g = grid_1d(n1, 256);
  // r = ~0 never matches, and the status pointer is unused when NULL-checked below
  if (dtype == FS_F32)
    knot_buckets_kernel<float><<<g, 256, 0, s>>>(static_cast<const float*>(x_dev), n1, (float)h, ~0ull, f_dev, nullptr);
  else if (dtype == FS_F64)
    knot_buckets_kernel<double><<<g, 256, 0, s>>>(static_cast<const double*>(x_dev), n1, h, ~0ull, f_dev, nullptr);
  else
    return fail(FS_INVALID_ARG, "dtype must be FS_F32 or FS_F64");
  FS_CUDA(cudaGetLastError());
  return FS_OK;
}

int fs_build_rank(int32_t dtype, const void* x_dev, uint64_t n1, double h, uint64_t r, uint64_t* f_scratch_dev,
                  void* dir_dev, void* stream) {
  if (!x_dev || !f_scratch_dev || !dir_dev || n1 < 2) return fail(FS_INVALID_ARG, "bad arguments");
  if (n1 - 1 >= (1ull << 32)) return fail(FS_INVALID_ARG, "table entries are 32-bit; partition is too large");
  int rc = fs_knot_buckets(dtype, x_dev, n1, h, f_scratch_dev, stream);
  if (rc) return rc;
  cudaStream_t s = as_stream(stream);
  const uint64_t words = (r >> 5) + 1;
  fill_rank_kernel<<<grid_1d(words, 256), 256, 0, s>>>(f_scratch_dev, n1, r, static_cast<uint2*>(dir_dev));
  FS_CUDA(cudaGetLastError());
  return FS_OK;
}

int fs_build_rank_rows(int32_t dtype, const void* x_dev, uint64_t n1, double h, uint64_t r, uint64_t* f_scratch_dev,
                       void* bytes_scratch_dev, void* rows_dev, void* stream) {
  if (!x_dev || !f_scratch_dev || !bytes_scratch_dev || !rows_dev || n1 < 2) return fail(FS_INVALID_ARG, "bad arguments");
  if (n1 - 1 >= (1ull << 31) || r >= (1ull << 32)) return fail(FS_TOO_LARGE, "rank rows need R < 2^32, N < 2^31");
  int rc = fs_knot_buckets(dtype, x_dev, n1, h, f_scratch_dev, stream);
  if (rc) return rc;
  rc = fs_build_knot_bytes(dtype, x_dev, n1, h, bytes_scratch_dev, stream);
  if (rc) return rc;
  cudaStream_t s = as_stream(stream);
  const uint64_t words = (r >> 5) + 1;
  fill_rank_rows_kernel<<<grid_1d(words, 256), 256, 0, s>>>(f_scratch_dev, static_cast<const uint8_t*>(bytes_scratch_dev),
                                                          n1, r, static_cast<uint4*>(rows_dev));
  FS_CUDA(cudaGetLastError());
  return FS_OK;
}

int fs_build_rank2(int32_t dtype, const void* x_dev, uint64_t n1, double h, uint64_t r, uint64_t* f_scratch_dev,
                   void* dir_dev, void* stream) {
  if (!x_dev || !f_scratch_dev || !dir_dev || n1 < 2) return fail(FS_INVALID_ARG, "bad arguments");
  if (n1 - 1 >= (1ull << 32)) return fail(FS_INVALID_ARG, "table entries are 32-bit; partition is too large");
  int rc = fs_knot_buckets(dtype, x_dev, n1, h, f_scratch_dev, stream);
  if (rc) return rc;
  cudaStream_t s = as_stream(stream);
  const uint64_t words = (r >> 5) + 1;
  fill_rank2_kernel<<<grid_1d(words, 256), 256, 0, s>>>(f_scratch_dev, n1, r, static_cast<uint4*>(dir_dev));
  FS_CUDA(cudaGetLastError());
  return FS_OK;
}

uint64_t fs_countdir_bytes(int32_t q, uint64_t r) {
  if (q < 2 || q > 15) return 0;
  return ((r >> countdir_lg(q)) + 1) * 8;
}

int fs_build_countdir(int32_t dtype, const void* x_dev, uint64_t n1, double h, uint64_t r, int32_t q,
                      uint64_t* f_scratch_dev, void* dir_dev, void* stream) {
  if (!x_dev || !f_scratch_dev || !dir_dev || n1 < 2) return fail(FS_INVALID_ARG, "bad arguments");
  if (q < 2 || q > 15) return fail(FS_INVALID_ARG, "count directories serve gaps 2..15");
  if (n1 - 1 >= (1ull << 32) || r >= (1ull << 32)) return fail(FS_INVALID_ARG, "table entries are 32-bit");
  int rc = fs_knot_buckets(dtype, x_dev, n1, h, f_scratch_dev, stream);
  if (rc) return rc;
  cudaStream_t s = as_stream(stream);
  const uint64_t words = (r >> countdir_lg(q)) + 1;
  if (q <= 3)
    fill_countdir_kernel<2><<<grid_1d(words, 256), 256, 0, s>>>(f_scratch_dev, n1, r, static_cast<uint2*>(dir_dev));
  else
    fill_countdir_kernel<4><<<grid_1d(words, 256), 256, 0, s>>>(f_scratch_dev, n1, r, static_cast<uint2*>(dir_dev));
  FS_CUDA(cudaGetLastError());
  return FS_OK;
}

uint64_t fs_sparse_bytes(uint64_t n1, uint64_t r, int32_t shift, uint64_t ndense) {
  if (shift < 5 || shift > 16) return 0;
  const uint64_t nc = (r >> shift) + 2, words = ndense << (shift - 5);
  const uint64_t head = (4 * nc + 2 * n1 + 3) & ~3ull;  // C | F | pad to 4
  return (head + words * 4 + words * 2 + 15) & ~15ull;  // | masks | prefixes
}

int fs_plan_sparse(int32_t dtype, const void* x_dev, uint64_t n1, double h, uint64_t r, uint64_t budget_bytes,
                   int32_t with_x, uint64_t* f_scratch_dev, int32_t* shift_out, uint64_t* ndense_out,
                   uint64_t* bytes_out, void* stream) {
  if (!x_dev || !f_scratch_dev || n1 < 2 || !shift_out) return fail(FS_INVALID_ARG, "bad arguments");
  if (n1 - 1 >= (1ull << 31) || r >= (1ull << 32)) return fail(FS_TOO_LARGE, "sparse table needs R < 2^32, N < 2^31");
  const uint64_t xb = with_x ? align128(n1 * (dtype == FS_F32 ? 4 : 8)) : 0;
  if (xb + 2 * n1 > budget_bytes) return fail(FS_TOO_LARGE, "knot offsets alone exceed the budget");
  int rc = fs_knot_buckets(dtype, x_dev, n1, h, f_scratch_dev, stream);
  if (rc) return rc;
  std::vector<uint64_t> f(n1);
  FS_CUDA(cudaMemcpyAsync(f.data(), f_scratch_dev, n1 * 8, cudaMemcpyDeviceToHost, as_stream(stream)));
  FS_CUDA(cudaStreamSynchronize(as_stream(stream)));
  for (int s = 5; s <= 16; ++s) {
    const uint64_t nc = (r >> s) + 2;
    if (xb + fs_sparse_bytes(n1, r, s, 0) > budget_bytes) continue;  // C + F alone too big
    std::vector<uint32_t> occ(nc, 0);
    for (uint64_t i = 0; i < n1; ++i) ++occ[f[i] >> s];
    uint64_t ndense = 0;
    for (uint32_t o : occ) ndense += o > kDenseOcc;
    const uint64_t bytes = fs_sparse_bytes(n1, r, s, ndense);
    if (ndense <= 65535 && xb + bytes <= budget_bytes) {
      *shift_out = s;
      if (ndense_out) *ndense_out = ndense;
      if (bytes_out) *bytes_out = bytes;
      return FS_OK;
    }
  }
  return fail(FS_TOO_LARGE, "no sparse layout fits the budget");
}

int fs_build_sparse(int32_t dtype, const void* x_dev, uint64_t n1, double h, uint64_t r, int32_t shift,
                    uint64_t* f_scratch_dev, void* sparse_dev, void* stream) {
  if (!x_dev || !f_scratch_dev || !sparse_dev || n1 < 2 || shift < 5 || shift > 16)
    return fail(FS_INVALID_ARG, "bad arguments");
  if (n1 - 1 >= (1ull << 31) || r >= (1ull << 32)) return fail(FS_TOO_LARGE, "sparse table needs R < 2^32, N < 2^31");
  int rc = fs_knot_buckets(dtype, x_dev, n1, h, f_scratch_dev, stream);
  if (rc) return rc;
  cudaStream_t s = as_stream(stream);
  const uint64_t nc = (r >> shift) + 2;
  uint32_t* C = static_cast<uint32_t*>(sparse_dev);
  uint16_t* F = reinterpret_cast<uint16_t*>(C + nc);
  fill_sparse_kernel<<<grid_1d(std::max(nc, n1), 256), 256, 0, s>>>(f_scratch_dev, n1, r, shift, C, F);
  FS_CUDA(cudaGetLastError());
  // dense super-buckets: slot order = increasing J (the same count fs_plan_sparse made)
  std::vector<uint32_t> c(nc);
  FS_CUDA(cudaMemcpyAsync(c.data(), C, nc * 4, cudaMemcpyDeviceToHost, s));
  FS_CUDA(cudaStreamSynchronize(s));
  std::vector<uint32_t> dense_j;
  for (uint64_t J = 0; J + 1 < nc; ++J)
    if (c[J + 1] - c[J] > kDenseOcc) dense_j.push_back((uint32_t)J);
  if (dense_j.empty()) return FS_OK;
  if (dense_j.size() > 65535) return fail(FS_TOO_LARGE, "too many dense super-buckets");
  const uint64_t words = (uint64_t)dense_j.size() << (shift - 5);
  const uint64_t head = (4 * nc + 2 * n1 + 3) & ~3ull;
  uint32_t* dmask = reinterpret_cast<uint32_t*>(static_cast<char*>(sparse_dev) + head);
  uint16_t* dpre = reinterpret_cast<uint16_t*>(dmask + words);
  // the f scratch is free again: it carries the dense super-bucket list
  FS_CUDA(cudaMemcpyAsync(f_scratch_dev, dense_j.data(), dense_j.size() * 4, cudaMemcpyHostToDevice, s));
  const int grid = (int)std::min<uint64_t>(dense_j.size(), (uint64_t)sm_count() * 8);
  fill_dense_kernel<<<grid, 128, 0, s>>>(C, F, reinterpret_cast<const uint32_t*>(f_scratch_dev), dense_j.size(), shift,
                                        dmask, dpre);
  FS_CUDA(cudaGetLastError());
  FS_CUDA(cudaStreamSynchronize(s));
  return FS_OK;
}

namespace {
bool is_record_format(int32_t format) {
  return format == FS_SPARSE_RECORDS || format == FS_SPARSE_RECORDS8 || format == FS_SPARSE_RECORDS12 ||
         format == FS_SPARSE_RECORDS8X3;
}
int record_max_shift(int32_t format) {
  return format == FS_SPARSE_RECORDS12 ? kRec12MaxShift : format == FS_SPARSE_RECORDS8X3 ? kRec3MaxShift : kRecMaxShift;
}
int record_bytes(int32_t format) { return format == FS_SPARSE_RECORDS8 || format == FS_SPARSE_RECORDS8X3 ? 8 : 16; }
uint64_t record_slots(int32_t format) {
  return format == FS_SPARSE_RECORDS ? 6 : format == FS_SPARSE_RECORDS12 ? 8 : format == FS_SPARSE_RECORDS8X3 ? 3 : 2;
}
}  // namespace

uint64_t fs_sparse_rec_bytes(int32_t format, uint64_t n1, uint64_t r, int32_t shift, uint64_t novf) {
  if (!is_record_format(format) || shift < 5 || shift > record_max_shift(format)) return 0;
  const uint64_t ng = (r >> shift) + 2;
  return (record_bytes(format) * ng + (novf ? 2 * n1 : 0) + 15) & ~15ull;
}

int fs_plan_sparse_rec(int32_t format, int32_t dtype, const void* x_dev, uint64_t n1, double h, uint64_t r,
                       uint64_t budget_bytes, int32_t with_x, uint64_t* f_scratch_dev, int32_t* shift_out,
                       uint64_t* novf_out, uint64_t* bytes_out, uint32_t* past_last_ppm_out, void* stream) {
  if (!x_dev || !f_scratch_dev || n1 < 2 || !shift_out) return fail(FS_INVALID_ARG, "bad arguments");
  if (!is_record_format(format)) return fail(FS_INVALID_ARG, "not a record format");
  if (n1 - 1 >= (1ull << 31) || r >= (1ull << 32)) return fail(FS_TOO_LARGE, "group records need R < 2^32, N < 2^31");
  if (format == FS_SPARSE_RECORDS8X3 && n1 > (1ull << 24)) return fail(FS_TOO_LARGE, "3-offset records need N+1 <= 2^24");
  const uint64_t slots = record_slots(format);
  const int max_shift = record_max_shift(format);
  const uint64_t xb = with_x ? align128(n1 * (dtype == FS_F32 ? 4 : 8)) : 0;
  if (xb + fs_sparse_rec_bytes(format, n1, r, max_shift, 0) > budget_bytes)
    return fail(FS_TOO_LARGE, "no group-record layout fits the budget");
  // every layout holds each knot in a record slot or in F: at least
  // min(n1 / slots records, 2 n1 bytes of F) -- skip the scan when even that
  // exceeds the budget (large N: the directory stays in L2)
  if (xb + std::min<uint64_t>((n1 / slots) * (uint64_t)record_bytes(format), 2 * n1) > budget_bytes)
    return fail(FS_TOO_LARGE, "no group-record layout fits the budget");
  int rc = fs_knot_buckets(dtype, x_dev, n1, h, f_scratch_dev, stream);
  if (rc) return rc;
  std::vector<uint64_t> f(n1);
  FS_CUDA(cudaMemcpyAsync(f.data(), f_scratch_dev, n1 * 8, cudaMemcpyDeviceToHost, as_stream(stream)));
  FS_CUDA(cudaStreamSynchronize(as_stream(stream)));
  // per shift: overflowing records and the buckets lying past their last
  // recorded knot (the only ones whose queries leave the record); f is sorted
  struct Cand {
    int s;
    uint64_t novf, past;
  };
  std::vector<Cand> cands;
  for (int s = 5; s <= max_shift; ++s) {
    if (xb + fs_sparse_rec_bytes(format, n1, r, s, 0) > budget_bytes) continue;
    uint64_t novf = 0, past = 0;
    for (uint64_t i = 0; i < n1;) {
      const uint64_t J = f[i] >> s;
      uint64_t e = i;
      while (e < n1 && (f[e] >> s) == J) ++e;
      if (e - i > slots) {
        ++novf;
        const uint64_t end = std::min(((J + 1) << s) - 1, r);  // last bucket of the super-bucket
        past += end - f[i + slots - 1];
      }
      i = e;
    }
    if (xb + fs_sparse_rec_bytes(format, n1, r, s, novf) <= budget_bytes) cands.push_back({s, novf, past});
  }
  // the fewest queries past a last recorded knot; among shifts within 1e-3
  // of that, the largest (smallest table)
  uint64_t min_past = ~0ull;
  for (const Cand& c : cands) min_past = std::min(min_past, c.past);
  int best = -1;
  uint64_t best_novf = 0, best_past = 0;
  for (const Cand& c : cands)
    if ((double)(c.past - min_past) <= 1e-3 * (double)(r + 1) && c.s > best) {
      best = c.s;
      best_novf = c.novf;
      best_past = c.past;
    }
  if (best < 0) return fail(FS_TOO_LARGE, "no group-record layout fits the budget");
  *shift_out = best;
  if (novf_out) *novf_out = best_novf;
  if (bytes_out) *bytes_out = fs_sparse_rec_bytes(format, n1, r, best, best_novf);
  if (past_last_ppm_out) *past_last_ppm_out = (uint32_t)(1e6 * (double)best_past / (double)(r + 1));
  return FS_OK;
}

int fs_build_sparse_rec(int32_t format, int32_t dtype, const void* x_dev, uint64_t n1, double h, uint64_t r,
                        int32_t shift, uint64_t novf, uint64_t* f_scratch_dev, void* buf_dev, void* stream) {
  if (!is_record_format(format)) return fail(FS_INVALID_ARG, "not a record format");
  if (!x_dev || !f_scratch_dev || !buf_dev || n1 < 2 || shift < 5 || shift > record_max_shift(format))
    return fail(FS_INVALID_ARG, "bad arguments");
  if (format == FS_SPARSE_RECORDS8X3 && n1 > (1ull << 24)) return fail(FS_TOO_LARGE, "3-offset records need N+1 <= 2^24");
  if (n1 - 1 >= (1ull << 31) || r >= (1ull << 32)) return fail(FS_TOO_LARGE, "group records need R < 2^32, N < 2^31");
  int rc = fs_knot_buckets(dtype, x_dev, n1, h, f_scratch_dev, stream);
  if (rc) return rc;
  cudaStream_t s = as_stream(stream);
  const uint64_t ng = (r >> shift) + 2;
  const int grid = grid_1d(std::max(ng, n1), 256);
  if (format == FS_SPARSE_RECORDS || format == FS_SPARSE_RECORDS12) {
    uint4* G = static_cast<uint4*>(buf_dev);
    uint16_t* F = novf ? reinterpret_cast<uint16_t*>(G + ng) : nullptr;
    if (format == FS_SPARSE_RECORDS) fill_sparse_rec_kernel<6><<<grid, 256, 0, s>>>(f_scratch_dev, n1, r, shift, G, F);
    else fill_sparse_rec_kernel<8><<<grid, 256, 0, s>>>(f_scratch_dev, n1, r, shift, G, F);
  } else {
    uint2* G = static_cast<uint2*>(buf_dev);
    uint16_t* F = novf ? reinterpret_cast<uint16_t*>(G + ng) : nullptr;
    if (format == FS_SPARSE_RECORDS8) fill_sparse_rec_kernel<2><<<grid, 256, 0, s>>>(f_scratch_dev, n1, r, shift, G, F);
    else fill_sparse_rec_kernel<3><<<grid, 256, 0, s>>>(f_scratch_dev, n1, r, shift, G, F);
  }
  FS_CUDA(cudaGetLastError());
  FS_CUDA(cudaStreamSynchronize(s));
  return FS_OK;
}

// ---------------------------------------------------------------------------
// Zoned records (FS_SPARSE_ZONED)
// ---------------------------------------------------------------------------
namespace {
// Per-zone record form for zone shift zs from the sorted knot buckets f:
// descriptors (first record << 5 | rank flag | s) and the record count.
// Slot records take the largest s in [kZonedMinShift, min(kZonedMaxShift,
// zs)] whose records hold at most kZonedSlots knots of the zone; a zone where
// none does takes 32-bucket rank words.  false if zs is out of range or
// needs > 64 zones.
bool zone_plan(const std::vector<uint64_t>& f, uint64_t r, int zs, std::vector<uint32_t>& desc, uint64_t& nrec) {
  if (zs < kZonedMinZoneShift || zs > 31) return false;
  const uint64_t nz = (r >> zs) + 1;
  if (nz > kZonedMaxZones) return false;
  const int smax = std::min(kZonedMaxShift, zs);
  // maxc[z][s - kZonedMinShift]: most knots in one 2^s-bucket record of zone z
  constexpr int NS = kZonedMaxShift - kZonedMinShift + 1;
  std::vector<std::array<uint32_t, NS>> maxc(nz);
  for (auto& a : maxc) a.fill(0);
  for (int si = 0; si + kZonedMinShift <= smax; ++si) {
    const int sh = kZonedMinShift + si;
    for (size_t i = 0; i < f.size();) {
      const uint64_t key = f[i] >> sh;
      size_t e = i;
      while (e < f.size() && (f[e] >> sh) == key) ++e;
      uint32_t& m = maxc[f[i] >> zs][si];
      m = std::max<uint32_t>(m, (uint32_t)(e - i));
      i = e;
    }
  }
  desc.assign(nz, 0);
  nrec = 0;
  for (uint64_t z = 0; z < nz; ++z) {
    const uint64_t zb = std::min<uint64_t>(1ull << zs, r + 1 - (z << zs));  // buckets of the zone
    int s = -1;
    for (int si = smax - kZonedMinShift; si >= 0; --si)
      if (maxc[z][si] <= (uint32_t)kZonedSlots) {
        s = kZonedMinShift + si;
        break;
      }
    const bool rank = s < 0;
    if (rank) s = kZonedRankShift;
    if (nrec >= (1ull << 27)) return false;
    // first record relative to the zone's start in records (may be negative):
    // the probe's record index is then (int)d >> 5 plus j >> s, no zone mask
    const int64_t rel = (int64_t)nrec - (int64_t)(z << (zs - s));
    desc[z] = ((uint32_t)rel << 5) | (rank ? kZonedRankFlag : 0u) | (uint32_t)s;
    nrec += (zb + (1ull << s) - 1) >> s;
  }
  return nrec < (1ull << 27);
}


// Striped rank words (FS_SPARSE_ZONED_RANK): per zone the stripe shift k (a
// mask bit per 2^k buckets, a word per 2^(k+5)).  kmax(zone) is the largest
// k <= min(kZonedMaxStripe, zs - 5) whose stripes hold at most one knot each:
// consecutive knot buckets a < b of a zone share a 2^k stripe iff k exceeds
// the highest bit in which they differ.  Starting from kmax everywhere (the
// smallest table), stripes are then refined while the table stays within
// `table_budget` bytes: each step halves the stripes of the zone that has the
// most buckets inside knot-holding stripes (cnt << k: the uniform queries that
// must read X), if that still fits, else the next such zone.  Deterministic
// in (f, r, zs, table_budget); re-running it with the budget set to its own
// result's size reproduces the plan (fs_build_zoned_rank does).
bool zone_plan_rank(const std::vector<uint64_t>& f, uint64_t r, int zs, uint64_t table_budget,
                    std::vector<uint32_t>& desc, uint64_t& nrec, uint64_t* xread_buckets) {
  if (zs < kZonedMinZoneShift || zs > 31) return false;
  const uint64_t nz = (r >> zs) + 1;
  if (nz > kZonedMaxZones) return false;
  const int kcap = std::min(kZonedMaxStripe, zs - kZonedRankShift);
  std::vector<int> k(nz, kcap);
  std::vector<uint64_t> cnt(nz, 0), zb(nz);
  for (uint64_t z = 0; z < nz; ++z) zb[z] = std::min<uint64_t>(1ull << zs, r + 1 - (z << zs));
  for (size_t i = 0; i < f.size(); ++i) {
    const uint64_t z = f[i] >> zs;
    if (z >= nz) return false;
    ++cnt[z];
    if (i + 1 < f.size() && (f[i + 1] >> zs) == z) {
      if (f[i + 1] <= f[i]) return false;  // not a gap-1 table
      const int hb = 63 - __builtin_clzll(f[i] ^ f[i + 1]);
      k[z] = std::min(k[z], hb);
    }
  }
  auto words = [&](uint64_t z, int kz) { return (zb[z] + (1ull << (kz + kZonedRankShift)) - 1) >> (kz + kZonedRankShift); };
  uint64_t total = 0;
  for (uint64_t z = 0; z < nz; ++z) total += words(z, k[z]);
  const uint64_t head = 4 * ((nz + 3) & ~3ull);
  if (head + 8 * total > table_budget || total >= (1ull << 27)) return false;
  for (;;) {
    // zones by descending cnt << k (ties: lower zone first)
    int64_t pick = -1;
    std::vector<uint64_t> order;
    for (uint64_t z = 0; z < nz; ++z)
      if (k[z] > 0 && cnt[z] > 0) order.push_back(z);
    std::stable_sort(order.begin(), order.end(),
                     [&](uint64_t a, uint64_t b) { return (cnt[a] << k[a]) > (cnt[b] << k[b]); });
    for (uint64_t z : order) {
      const uint64_t t2 = total - words(z, k[z]) + words(z, k[z] - 1);
      if (head + 8 * t2 <= table_budget && t2 < (1ull << 27)) {
        pick = (int64_t)z;
        total = t2;
        break;
      }
    }
    if (pick < 0) break;
    --k[pick];
  }
  desc.assign(nz, 0);
  nrec = 0;
  uint64_t xr = 0;
  for (uint64_t z = 0; z < nz; ++z) {
    const int s = k[z] + kZonedRankShift;
    const int64_t rel = (int64_t)nrec - (int64_t)(z << (zs - s));
    desc[z] = ((uint32_t)rel << 5) | kZonedRankFlag | (uint32_t)k[z];
    nrec += words(z, k[z]);
    xr += std::min<uint64_t>(cnt[z] << k[z], zb[z]);
  }
  if (xread_buckets) *xread_buckets = xr;
  return true;
}

// knot buckets f_i (sorted) computed on the device, read back for the planner
int zoned_knot_buckets(int32_t dtype, const void* x_dev, uint64_t n1, double h, uint64_t* f_scratch_dev,
                       std::vector<uint64_t>& f, cudaStream_t s) {
  int rc = fs_knot_buckets(dtype, x_dev, n1, h, f_scratch_dev, s);
  if (rc) return rc;
  f.resize(n1);
  FS_CUDA(cudaMemcpyAsync(f.data(), f_scratch_dev, n1 * 8, cudaMemcpyDeviceToHost, s));
  FS_CUDA(cudaStreamSynchronize(s));
  return FS_OK;
}
}  // namespace

int fs_build_knot_bytes(int32_t dtype, const void* x_dev, uint64_t n1, double h, void* buf_dev, void* stream) {
  if (!x_dev || !buf_dev || n1 < 2) return fail(FS_INVALID_ARG, "bad arguments");
  cudaStream_t s = as_stream(stream);
  const uint64_t npad = (n1 + 15) & ~15ull;
  const int g = grid_1d(npad, 256);
  if (dtype == FS_F32)
    fill_knot_bytes_kernel<float><<<g, 256, 0, s>>>(static_cast<const float*>(x_dev), n1, (float)h,
                                                   static_cast<uint8_t*>(buf_dev), npad);
  else if (dtype == FS_F64)
    fill_knot_bytes_kernel<double><<<g, 256, 0, s>>>(static_cast<const double*>(x_dev), n1, h,
                                                    static_cast<uint8_t*>(buf_dev), npad);
  else
    return fail(FS_INVALID_ARG, "dtype must be FS_F32 or FS_F64");
  FS_CUDA(cudaGetLastError());
  return FS_OK;
}

uint64_t fs_count_words_bytes(uint64_t r, int32_t k, uint64_t noff) {
  if (k < 0 || k > kCountMaxShift || r >= (1ull << 32) || (noff && k > kCountMaxOffsetShift)) return 0;
  return 8 * ((r >> (k + kCountWordShift)) + 1) + ((noff + 15) & ~15ull);
}

int fs_plan_count_words(int32_t dtype, const void* x_dev, uint64_t n1, double h, uint64_t r, uint64_t budget_bytes,
                        int32_t mode, uint64_t* f_scratch_dev, int32_t* k_out, uint64_t* bytes_out,
                        uint64_t* xread_ppm_out, uint64_t* rare_ppm_out, void* stream) {
  if (!x_dev || !f_scratch_dev || n1 < 2 || !k_out) return fail(FS_INVALID_ARG, "bad arguments");
  if (dtype != FS_F32 && dtype != FS_F64) return fail(FS_INVALID_ARG, "dtype must be FS_F32 or FS_F64");
  if (mode < 0 || mode > 2) return fail(FS_INVALID_ARG, "mode: 0 words alone, 1 beside X, 2 beside knot offsets");
  if (n1 - 1 >= (1ull << 31) || r >= (1ull << 32)) return fail(FS_TOO_LARGE, "count words need R < 2^32, N < 2^31");
  const uint64_t es = dtype == FS_F32 ? 4 : 8;
  // what is staged beside the words: nothing, all of X, or a byte per knot
  const uint64_t beside = mode == 1 ? align128(n1 * es) : mode == 2 ? ((n1 + 15) & ~15ull) : 0;
  if (budget_bytes < beside + 128 + 8) return fail(FS_TOO_LARGE, "no count-word layout fits the budget");
  const uint64_t table_budget = budget_bytes - beside - 128;
  int k = 0;
  while (k <= kCountMaxShift && fs_count_words_bytes(r, k, 0) > table_budget) ++k;
  if (mode == 2 && k > kCountMaxOffsetShift)
    return fail(FS_TOO_LARGE, "knot offsets are bytes: no stripe shift <= 8 fits the budget");
  if (k > kCountMaxShift) return fail(FS_TOO_LARGE, "no count-word layout fits the budget");
  // more knots than stripes: nearly every query would scan (the planner's caller would refuse it anyway)
  if (n1 > ((r >> k) + 1)) return fail(FS_TOO_LARGE, "count words: more knots than stripes");
  std::vector<uint64_t> f;
  int rc = zoned_knot_buckets(dtype, x_dev, n1, h, f_scratch_dev, f, as_stream(stream));
  if (rc) return rc;
  // buckets whose queries read X or a knot offset (stripes holding a knot) and
  // whose queries scan (stripes holding two or more; every stripe of a flagged word)
  uint64_t xread = 0, rare = 0;
  const uint64_t sw = 1ull << k, ww = 1ull << (k + kCountWordShift);
  for (size_t i = 0; i < f.size();) {
    size_t e = i + 1;
    while (e < f.size() && (f[e] >> k) == (f[i] >> k)) ++e;
    const uint64_t width = std::min<uint64_t>(sw, r + 1 - ((f[i] >> k) << k));
    xread += width;
    if (e - i >= 2) rare += width;
    else if (mode == 2) rare += 1;  // beside offsets, the knot's own bucket is decided by X on the scan path
    if (e - i >= 4) rare += std::min<uint64_t>(ww, r + 1 - ((f[i] >> (k + kCountWordShift)) << (k + kCountWordShift)));
    i = e;
  }
  *k_out = k;
  if (bytes_out) *bytes_out = fs_count_words_bytes(r, k, mode == 2 ? n1 : 0);
  if (xread_ppm_out) *xread_ppm_out = (uint64_t)((long double)xread * 1e6L / (long double)(r + 1));
  if (rare_ppm_out) *rare_ppm_out = (uint64_t)((long double)std::min<uint64_t>(rare, r + 1) * 1e6L / (long double)(r + 1));
  return FS_OK;
}

int fs_build_count_words(int32_t dtype, const void* x_dev, uint64_t n1, double h, uint64_t r, int32_t k,
                         int32_t with_offsets, uint64_t* f_scratch_dev, void* buf_dev, void* stream) {
  if (!x_dev || !f_scratch_dev || !buf_dev || n1 < 2) return fail(FS_INVALID_ARG, "bad arguments");
  if (dtype != FS_F32 && dtype != FS_F64) return fail(FS_INVALID_ARG, "dtype must be FS_F32 or FS_F64");
  if (n1 - 1 >= (1ull << 31) || r >= (1ull << 32)) return fail(FS_TOO_LARGE, "count words need R < 2^32, N < 2^31");
  const uint64_t bytes = fs_count_words_bytes(r, k, with_offsets ? n1 : 0);
  if (!bytes) return fail(FS_INVALID_ARG, "stripe shift out of range");
  cudaStream_t s = as_stream(stream);
  int rc = fs_knot_buckets(dtype, x_dev, n1, h, f_scratch_dev, s);
  if (rc) return rc;
  const uint64_t nwords = fs_count_words_bytes(r, k, 0) / 8;
  fill_count_words_kernel<<<grid_1d(nwords, 256), 256, 0, s>>>(f_scratch_dev, n1, k, static_cast<uint2*>(buf_dev), nwords);
  FS_CUDA(cudaGetLastError());
  if (with_offsets) {
    const uint64_t npad = (n1 + 15) & ~15ull;
    fill_count_offsets_kernel<<<grid_1d(npad, 256), 256, 0, s>>>(f_scratch_dev, n1, k,
                                                                static_cast<uint8_t*>(buf_dev) + 8 * nwords, npad);
    FS_CUDA(cudaGetLastError());
  }
  return FS_OK;
}

uint64_t fs_zoned_bytes(uint64_t r, int32_t zs, uint64_t nrec) {
  if (zs < kZonedMinZoneShift || zs > 31) return 0;
  const uint64_t nz = (r >> zs) + 1;
  if (nz > kZonedMaxZones) return 0;
  return 4 * ((nz + 3) & ~3ull) + 8 * nrec;
}

int fs_plan_zoned(int32_t dtype, const void* x_dev, uint64_t n1, double h, uint64_t r, uint64_t budget_bytes,
                  uint64_t* f_scratch_dev, int32_t* zs_out, uint64_t* nrec_out, uint64_t* bytes_out,
                  uint64_t* t0_out, uint64_t* nt_out, void* stream) {
  if (!x_dev || !f_scratch_dev || n1 < 2 || !zs_out) return fail(FS_INVALID_ARG, "bad arguments");
  if (dtype != FS_F32 && dtype != FS_F64) return fail(FS_INVALID_ARG, "dtype must be FS_F32 or FS_F64");
  if (n1 - 1 >= (1ull << 31) || r >= (1ull << 32)) return fail(FS_TOO_LARGE, "zoned records need R < 2^32, N < 2^31");
  if (n1 > (1ull << 24)) return fail(FS_TOO_LARGE, "zoned slot records need N+1 <= 2^24");
  // every knot costs at least 8/3 B of a slot record
  if (8 * n1 / kZonedSlots > budget_bytes) return fail(FS_TOO_LARGE, "no zoned layout fits the budget");
  std::vector<uint64_t> f;
  int rc = zoned_knot_buckets(dtype, x_dev, n1, h, f_scratch_dev, f, as_stream(stream));
  if (rc) return rc;
  // the fewest zones (32: one wavefront per warp's descriptor loads, else 64)
  int zs32 = kZonedMinZoneShift;
  while (zs32 < 31 && (r >> zs32) + 1 > 32) ++zs32;
  int best = -1;
  uint64_t best_nrec = 0, best_bytes = 0;
  for (int zs : {zs32, zs32 - 1}) {
    if (zs < kZonedMinZoneShift) continue;
    std::vector<uint32_t> desc;
    uint64_t nrec = 0;
    if (!zone_plan(f, r, zs, desc, nrec)) continue;
    const uint64_t bytes = fs_zoned_bytes(r, zs, nrec);
    if (bytes + 128 > budget_bytes) continue;
    best = zs;
    best_nrec = nrec;
    best_bytes = bytes;
    break;
  }
  if (best < 0) return fail(FS_TOO_LARGE, "no zoned layout fits the budget");
  // window of X: the densest nt consecutive knots (smallest bucket span)
  const uint64_t es = dtype == FS_F32 ? 4 : 8;
  const uint64_t room = budget_bytes - best_bytes - 128;
  const uint64_t nt = std::min<uint64_t>(n1, room / es);
  uint64_t t0 = 0;
  if (nt > 0 && nt < n1) {
    uint64_t span = ~0ull;
    for (uint64_t a = 0; a + nt <= n1; ++a)
      if (f[a + nt - 1] - f[a] < span) {
        span = f[a + nt - 1] - f[a];
        t0 = a;
      }
  }
  *zs_out = best;
  if (nrec_out) *nrec_out = best_nrec;
  if (bytes_out) *bytes_out = best_bytes;
  if (t0_out) *t0_out = t0;
  if (nt_out) *nt_out = nt;
  return FS_OK;
}

int fs_build_zoned(int32_t dtype, const void* x_dev, uint64_t n1, double h, uint64_t r, int32_t zs,
                   uint64_t* f_scratch_dev, void* buf_dev, void* stream) {
  if (!x_dev || !f_scratch_dev || !buf_dev || n1 < 2) return fail(FS_INVALID_ARG, "bad arguments");
  if (dtype != FS_F32 && dtype != FS_F64) return fail(FS_INVALID_ARG, "dtype must be FS_F32 or FS_F64");
  if (n1 - 1 >= (1ull << 31) || r >= (1ull << 32)) return fail(FS_TOO_LARGE, "zoned records need R < 2^32, N < 2^31");
  cudaStream_t s = as_stream(stream);
  std::vector<uint64_t> f;
  int rc = zoned_knot_buckets(dtype, x_dev, n1, h, f_scratch_dev, f, s);
  if (rc) return rc;
  std::vector<uint32_t> desc;
  uint64_t nrec = 0;
  if (!zone_plan(f, r, zs, desc, nrec)) return fail(FS_INVALID_ARG, "zone shift out of range for this table");
  const uint64_t nz = desc.size();
  desc.resize((nz + 3) & ~3ull, 0u);
  FS_CUDA(cudaMemcpyAsync(buf_dev, desc.data(), 4 * desc.size(), cudaMemcpyHostToDevice, s));
  if (n1 > (1ull << 24)) return fail(FS_TOO_LARGE, "zoned slot records need N+1 <= 2^24");
  auto* R = reinterpret_cast<uint2*>(static_cast<char*>(buf_dev) + 4 * desc.size());
  fill_zoned_kernel<false><<<grid_1d(nrec, 256), 256, 0, s>>>(f_scratch_dev, n1, zs, static_cast<const uint32_t*>(buf_dev),
                                                              (uint32_t)nz, R, nrec);
  FS_CUDA(cudaGetLastError());
  FS_CUDA(cudaStreamSynchronize(s));  // desc must outlive the async upload
  return FS_OK;
}

int fs_plan_zoned_rank(int32_t dtype, const void* x_dev, uint64_t n1, double h, uint64_t r, uint64_t budget_bytes,
                       uint64_t* f_scratch_dev, int32_t* zs_out, uint64_t* nrec_out, uint64_t* bytes_out,
                       uint64_t* t0_out, uint64_t* nt_out, uint64_t* xread_ppm_out, void* stream) {
  if (!x_dev || !f_scratch_dev || n1 < 2 || !zs_out) return fail(FS_INVALID_ARG, "bad arguments");
  if (dtype != FS_F32 && dtype != FS_F64) return fail(FS_INVALID_ARG, "dtype must be FS_F32 or FS_F64");
  if (n1 - 1 >= (1ull << 31) || r >= (1ull << 32)) return fail(FS_TOO_LARGE, "zoned records need R < 2^32, N < 2^31");
  // every knot needs its own mask bit
  if (n1 / 4 > budget_bytes) return fail(FS_TOO_LARGE, "no striped layout fits the budget");
  std::vector<uint64_t> f;
  int rc = zoned_knot_buckets(dtype, x_dev, n1, h, f_scratch_dev, f, as_stream(stream));
  if (rc) return rc;
  const uint64_t es = dtype == FS_F32 ? 4 : 8;
  // an eighth of the budget is kept for the window of X (the densest knots);
  // what the words leave unused goes to the window too
  const uint64_t win = std::min<uint64_t>(align128(n1 * es), (budget_bytes / 8) & ~127ull);
  if (budget_bytes < win + 256) return fail(FS_TOO_LARGE, "no striped layout fits the budget");
  const uint64_t table_budget = budget_bytes - win - 128;
  int zs32 = kZonedMinZoneShift;
  while (zs32 < 31 && (r >> zs32) + 1 > 32) ++zs32;
  int best = -1;
  uint64_t best_nrec = 0, best_bytes = 0, best_xr = ~0ull;
  // both zone counts (32: one wavefront per warp's descriptor loads; 64:
  // finer stripes): the one whose uniform queries read X least
  for (int zs : {zs32, zs32 - 1}) {
    if (zs < kZonedMinZoneShift) continue;
    std::vector<uint32_t> desc;
    uint64_t nrec = 0, xr = 0;
    if (!zone_plan_rank(f, r, zs, table_budget, desc, nrec, &xr)) continue;
    if (best < 0 || xr + (r + 1) / 64 < best_xr) {  // 64 zones must save >= 1.6% of X reads
      best = zs;
      best_nrec = nrec;
      best_bytes = fs_zoned_bytes(r, zs, nrec);
      best_xr = xr;
    }
  }
  if (best < 0) return fail(FS_TOO_LARGE, "no striped layout fits the budget");
  const uint64_t room = budget_bytes - best_bytes - 128;
  const uint64_t nt = std::min<uint64_t>(n1, room / es);
  uint64_t t0 = 0;
  if (nt > 0 && nt < n1) {
    uint64_t span = ~0ull;
    for (uint64_t a = 0; a + nt <= n1; ++a)
      if (f[a + nt - 1] - f[a] < span) {
        span = f[a + nt - 1] - f[a];
        t0 = a;
      }
  }
  *zs_out = best;
  if (nrec_out) *nrec_out = best_nrec;
  if (bytes_out) *bytes_out = best_bytes;
  if (t0_out) *t0_out = t0;
  if (nt_out) *nt_out = nt;
  if (xread_ppm_out) *xread_ppm_out = (uint64_t)((long double)best_xr * 1e6L / (long double)(r + 1));
  return FS_OK;
}

int fs_build_zoned_rank(int32_t dtype, const void* x_dev, uint64_t n1, double h, uint64_t r, int32_t zs,
                        uint64_t nrec, uint64_t* f_scratch_dev, void* buf_dev, void* stream) {
  if (!x_dev || !f_scratch_dev || !buf_dev || n1 < 2) return fail(FS_INVALID_ARG, "bad arguments");
  if (dtype != FS_F32 && dtype != FS_F64) return fail(FS_INVALID_ARG, "dtype must be FS_F32 or FS_F64");
  if (n1 - 1 >= (1ull << 31) || r >= (1ull << 32)) return fail(FS_TOO_LARGE, "zoned records need R < 2^32, N < 2^31");
  const uint64_t bytes = fs_zoned_bytes(r, zs, nrec);
  if (!bytes) return fail(FS_INVALID_ARG, "zone shift out of range for this table");
  cudaStream_t s = as_stream(stream);
  std::vector<uint64_t> f;
  int rc = zoned_knot_buckets(dtype, x_dev, n1, h, f_scratch_dev, f, s);
  if (rc) return rc;
  std::vector<uint32_t> desc;
  uint64_t got = 0;
  if (!zone_plan_rank(f, r, zs, bytes, desc, got, nullptr) || got != nrec)
    return fail(FS_INVALID_ARG, "no striped plan of this zone shift has that many words");
  const uint64_t nz = desc.size();
  desc.resize((nz + 3) & ~3ull, 0u);
  FS_CUDA(cudaMemcpyAsync(buf_dev, desc.data(), 4 * desc.size(), cudaMemcpyHostToDevice, s));
  auto* R = reinterpret_cast<uint2*>(static_cast<char*>(buf_dev) + 4 * desc.size());
  fill_zoned_kernel<true><<<grid_1d(nrec, 256), 256, 0, s>>>(f_scratch_dev, n1, zs, static_cast<const uint32_t*>(buf_dev),
                                                             (uint32_t)nz, R, nrec);
  FS_CUDA(cudaGetLastError());
  FS_CUDA(cudaStreamSynchronize(s));  // desc must outlive the async upload
  return FS_OK;
}

int fs_build_hot_window(int32_t dtype, const void* dir_dev, uint64_t r, uint64_t budget_bytes, void* ws_dev,
                        uint64_t* word0_out, uint64_t* words_out, uint64_t* knot0_out, uint64_t* knots_out,
                        uint64_t* knots_in_window_out, void* stream) {
  if (!dir_dev || !ws_dev) return fail(FS_INVALID_ARG, "NULL pointer");
  if (dtype != FS_F32 && dtype != FS_F64) return fail(FS_INVALID_ARG, "dtype must be FS_F32 or FS_F64");
  cudaStream_t s = as_stream(stream);
  const uint64_t words = (r >> 5) + 1;
  const uint32_t es = dtype == FS_F32 ? 4 : 8;
  const uint64_t budget = budget_bytes > 256 ? budget_bytes - 256 : 0;  // alignment slack
  auto* scratch = static_cast<unsigned long long*>(ws_dev);           // [0]: best key, [1..3]: window
  FS_CUDA(cudaMemsetAsync(scratch, 0, sizeof(unsigned long long), s));
  const auto* dir = static_cast<const uint2*>(dir_dev);
  hot_window_kernel<<<grid_1d(words, 256), 256, 0, s>>>(dir, words, es, budget, scratch);
  FS_CUDA(cudaGetLastError());
  unsigned long long key = 0;
  FS_CUDA(cudaMemcpyAsync(&key, scratch, sizeof(key), cudaMemcpyDeviceToHost, s));
  FS_CUDA(cudaStreamSynchronize(s));
  if (!key) {
    *word0_out = *words_out = *knot0_out = *knots_out = 0;
    if (knots_in_window_out) *knots_in_window_out = 0;
    return FS_OK;
  }
  const uint64_t a = 0xffffffffull - (key & 0xffffffffull);
  hot_window_finish<<<1, 1, 0, s>>>(dir, words, es, budget, a, reinterpret_cast<uint64_t*>(scratch) + 1);
  FS_CUDA(cudaGetLastError());
  uint64_t fin[3];
  FS_CUDA(cudaMemcpyAsync(fin, scratch + 1, sizeof(fin), cudaMemcpyDeviceToHost, s));
  FS_CUDA(cudaStreamSynchronize(s));
  *word0_out = a;
  *words_out = fin[0] - a;
  *knot0_out = fin[1];
  *knots_out = fin[2] - fin[1] + 1;
  if (knots_in_window_out) *knots_in_window_out = key >> 32;
  return FS_OK;
}

int fs_build_fused(int32_t dtype, const void* x_dev, uint64_t n1, const uint32_t* k_dev, uint64_t r, void* rec_dev,
                   void* stream) {
  if (!x_dev || !k_dev || !rec_dev || n1 < 2) return fail(FS_INVALID_ARG, "bad arguments");
  cudaStream_t s = as_stream(stream);
  const int g = grid_1d(r + 1, 256);
  if (dtype == FS_F32)
    fill_fused_f32<<<g, 256, 0, s>>>(static_cast<const float*>(x_dev), k_dev, r, static_cast<uint2*>(rec_dev));
  else if (dtype == FS_F64)
    fill_fused_f64<<<g, 256, 0, s>>>(static_cast<const double*>(x_dev), k_dev, r, static_cast<double2*>(rec_dev));
  else
    return fail(FS_INVALID_ARG, "dtype must be FS_F32 or FS_F64");
  FS_CUDA(cudaGetLastError());
  return FS_OK;
}

int fs_build_padded(int32_t dtype, const void* x_dev, uint64_t n1, int32_t pbits, void* xpad_dev, void* stream) {
  if (!x_dev || !xpad_dev || n1 < 2 || pbits < 1 || pbits > 40 || (1ull << pbits) < n1)
    return fail(FS_INVALID_ARG, "bad arguments");
  cudaStream_t s = as_stream(stream);
  const uint64_t len = 1ull << pbits;
  const int g = grid_1d(len, 256);
  if (dtype == FS_F32)
    pad_right_kernel<float><<<g, 256, 0, s>>>(static_cast<const float*>(x_dev), n1, len, static_cast<float*>(xpad_dev));
  else if (dtype == FS_F64)
    pad_right_kernel<double><<<g, 256, 0, s>>>(static_cast<const double*>(x_dev), n1, len, static_cast<double*>(xpad_dev));
  else
    return fail(FS_INVALID_ARG, "dtype must be FS_F32 or FS_F64");
  FS_CUDA(cudaGetLastError());
  return FS_OK;
}

int fs_build_eytzinger(int32_t dtype, const void* x_dev, uint64_t n1, int32_t depth, void* tree_dev, void* stream) {
  if (!x_dev || !tree_dev || n1 < 2 || depth < 1 || depth > 40 || ((1ull << depth) - 1) < n1)
    return fail(FS_INVALID_ARG, "bad arguments");
  cudaStream_t s = as_stream(stream);
  const int g = grid_1d((1ull << depth) - 1, 256);
  if (dtype == FS_F32)
    eytzinger_kernel<float><<<g, 256, 0, s>>>(static_cast<const float*>(x_dev), n1, depth, static_cast<float*>(tree_dev));
  else if (dtype == FS_F64)
    eytzinger_kernel<double><<<g, 256, 0, s>>>(static_cast<const double*>(x_dev), n1, depth, static_cast<double*>(tree_dev));
  else
    return fail(FS_INVALID_ARG, "dtype must be FS_F32 or FS_F64");
  FS_CUDA(cudaGetLastError());
  return FS_OK;
}

uint64_t fs_b2_deep_bytes(int32_t dtype, int32_t pbits, int32_t* top_bits_out, int32_t* k_out) {
  if ((dtype != FS_F32 && dtype != FS_F64) || pbits < 1 || pbits > 31) return 0;
  const int top = b2_top_bits(pbits, dtype == FS_F32 ? 4 : 8), k = b2_deep_k(dtype);
  if (top_bits_out) *top_bits_out = top;
  if (k_out) *k_out = k;
  if (pbits - top < b2_deep_min_levels(dtype)) return 0;
  return b2_deep_total_bytes(pbits, top, k);
}

int fs_build_b2_deep(int32_t dtype, const void* xpad_dev, int32_t pbits, int32_t top_bits, int32_t k,
                     void* deep_dev, void* stream) {
  if (!xpad_dev || !deep_dev || pbits < 1 || pbits > 31 || top_bits < 0 || top_bits >= pbits || k < 2 || k > 3 ||
      (dtype == FS_F64 && k > 2))
    return fail(FS_INVALID_ARG, "bad arguments");
  cudaStream_t s = as_stream(stream);
  uint64_t off = 0;
  for (int l = top_bits; pbits - l >= kB2DeepMinLevels; l += std::min<int>(k, pbits - l)) {
    const int kc = std::min<int>(k, pbits - l);
    const uint64_t nrec = 1ull << l;
    char* dst = static_cast<char*>(deep_dev) + off;
    const int g = grid_1d(nrec * 8, 256);
    if (dtype == FS_F32)
      b2_deep_kernel<float><<<g, 256, 0, s>>>(static_cast<const float*>(xpad_dev), pbits, l, kc, nrec,
                                              reinterpret_cast<float*>(dst));
    else if (dtype == FS_F64)
      b2_deep_kernel<double><<<g, 256, 0, s>>>(static_cast<const double*>(xpad_dev), pbits, l, kc, nrec,
                                               reinterpret_cast<double*>(dst));
    else
      return fail(FS_INVALID_ARG, "dtype must be FS_F32 or FS_F64");
    FS_CUDA(cudaGetLastError());
    off += nrec * 32;
  }
  return FS_OK;
}

int fs_search_device(const fs_plan* plan, const void* z_dev, uint64_t m, void* out_dev, int32_t out_bytes,
                     unsigned long long* first_bad_dev, void* stream) {
  return fs_search_device_at(plan, z_dev, m, out_dev, out_bytes, first_bad_dev, 0, stream);
}

int fs_search_device_at(const fs_plan* plan, const void* z_dev, uint64_t m, void* out_dev, int32_t out_bytes,
                        unsigned long long* first_bad_dev, uint64_t base, void* stream) {
  int rc = check_search_args(plan, z_dev, m, out_dev, out_bytes, first_bad_dev);
  if (rc) return rc;
  cudaStream_t s = as_stream(stream);
  // the kernel's last CTA writes status[0] and [3]; only an empty batch needs writes here
  if (m == 0) {
    FS_CUDA(cudaMemsetAsync(first_bad_dev, 0xff, sizeof(unsigned long long), s));
    FS_CUDA(cudaMemsetAsync(first_bad_dev + 3, 0xff, sizeof(unsigned long long), s));
    FS_CUDA(cudaMemsetAsync(reinterpret_cast<unsigned char*>(first_bad_dev + 3) + 7, 0x7f, 1, s));
    return FS_OK;
  }
  return launch_search(plan, place_for_batch(plan, m), z_dev, m, out_dev, out_bytes, first_bad_dev, base, s);
}

size_t fs_search_ws_words(void) { return FS_SEARCH_WS_WORDS; }

namespace {

}  // namespace

// One batch split into spans searched concurrently (one call per span, e.g.
// one per GPU): every span's call arrives here once its own span is known
// clean or bad, and no call writes results back until every span is clean
// -- the "nothing written on OutOfDomain" promise of batch.py:404 over the
// whole batch.  Single use.
struct fs_gate {
  std::mutex mu;
  std::condition_variable cv;
  int parties = 1, arrived = 0;
  bool bad = false;
  // true iff every party arrived with a clean span (a bad party returns at once)
  bool arrive_and_wait(bool clean) {
    std::unique_lock<std::mutex> lk(mu);
    ++arrived;
    if (!clean) bad = true;
    cv.notify_all();
    if (!clean) return false;
    cv.wait(lk, [&] { return bad || arrived >= parties; });
    return !bad;
  }
  void abort() {
    std::lock_guard<std::mutex> lk(mu);
    bad = true;
    cv.notify_all();
  }
};

namespace {

// A call's single arrival at its gate; a call that leaves early (CUDA error,
// bad argument) arrives as "bad" on the way out so no other span waits forever.
struct GateArrival {
  fs_gate* g;
  bool done = false;
  explicit GateArrival(fs_gate* gate) : g(gate) {}
  bool arrive(bool clean) {
    if (done) return clean;
    done = true;
    return g ? g->arrive_and_wait(clean) : clean;
  }
  ~GateArrival() {
    if (g && !done) g->arrive_and_wait(false);
  }
};

// Queries per staging slot of the pageable path (16 MB slots), and per chunk
// of an m-query batch: an eighth of the batch between 2 and 16 MB, so the
// host copies of one chunk overlap the DMA of the previous one even for
// mid-size batches (16 MB of queries: 4.1 -> see profiles/r02/e2e_curve.jsonl).
uint64_t staged_slot_elems(size_t es) { return ((16ull << 20) / es + 7) & ~7ull; }
uint64_t staged_chunk_elems(size_t es, uint64_t m) {
  const uint64_t lo = (2ull << 20) / es, hi = staged_slot_elems(es);
  return (std::min(hi, std::max(lo, m / 8)) + 7) & ~7ull;  // 32-B aligned on device (8-query groups)
}

// How fs_search_host splits a batch: through the library's pinned staging
// (pageable buffers of any real size) or straight from page-locked memory,
// and the queries per chunk (one search kernel per chunk).
struct HostChunking {
  bool staged;
  uint64_t chunk;
};
HostChunking host_chunking(const fs_plan* plan, const void* z_host, uint64_t m, const void* out_host, int out_bytes,
                           uint64_t chunk_elems, int flags) {
  const size_t es = plan->dtype == FS_F32 ? 4 : 8;
  HostChunking hc;
  hc.staged = m * (uint64_t)out_bytes >= (4ull << 20) && !(flags & FS_HOST_NO_STAGING) &&
              !(is_pinned(z_host) && is_pinned(out_host));
  if (hc.staged) {
    hc.chunk = staged_chunk_elems(es, m);
  } else {
    if (chunk_elems == 0) chunk_elems = (64ull << 20) / es;
    hc.chunk = (chunk_elems + 7) & ~7ull;  // keep every chunk 32-B aligned on device (8-query groups)
  }
  return hc;
}

// End-to-end search of PAGEABLE host buffers through pinned staging slots:
// phase 1 streams queries pageable -> pinned slot (host threads) -> device
// (copy engine) with the search kernel of each chunk queued behind its
// upload; after the first-bad readback (nothing is written on error), phase
// 2 drains results device -> pinned slot -> pageable out the same way.
int search_host_staged(const fs_plan* plan, Placement pl, const void* z_host, uint64_t m, void* out_host, int ob,
                       void* z_dev, void* out_dev, unsigned long long* fb, int64_t* pos_out, cudaStream_t s,
                       cudaStream_t cs, GateArrival& gate) {
  constexpr int kSlots = 3;
  const size_t es = plan->dtype == FS_F32 ? 4 : 8;
  const uint64_t chunk = staged_chunk_elems(es, m);
  const size_t slot_bytes = staged_slot_elems(es) * std::max<size_t>(es, (size_t)ob);  // one cached slot size
  void* slot[kSlots] = {nullptr, nullptr, nullptr};
  cudaEvent_t ev[kSlots] = {nullptr, nullptr, nullptr};
  int status = FS_OK;
  for (int i = 0; i < kSlots && status == FS_OK; ++i) {
    slot[i] = PinnedSlots::acquire(slot_bytes);
    if (!slot[i]) status = fail(FS_CUDA_ERROR, "pinned staging allocation failed");
    else if (cudaEventCreateWithFlags(&ev[i], cudaEventDisableTiming) != cudaSuccess)
      status = fail(FS_CUDA_ERROR, "event creation failed");
  }
  const int copy_threads = host_copy_threads();
  pl.merge = 1;
  if (status == FS_OK && cudaMemsetAsync(fb, 0xff, sizeof(unsigned long long), s) != cudaSuccess)
    status = fail(FS_CUDA_ERROR, "status reset failed");
  // phase 1: upload + search
  uint64_t c = 0;
  for (uint64_t off = 0; off < m && status == FS_OK; off += chunk, ++c) {
    const uint64_t n = std::min(chunk, m - off);
    const int k = (int)(c % kSlots);
    if (c >= kSlots && cudaEventSynchronize(ev[k]) != cudaSuccess) {
      status = fail(FS_CUDA_ERROR, "staging slot wait failed");
      break;
    }
    host_copy(slot[k], static_cast<const char*>(z_host) + off * es, n * es, copy_threads);
    char* dst = static_cast<char*>(z_dev) + off * es;
    cudaError_t e = cudaMemcpyAsync(dst, slot[k], n * es, cudaMemcpyHostToDevice, cs);
    if (e == cudaSuccess) e = cudaEventRecord(ev[k], cs);
    if (e == cudaSuccess) e = cudaStreamWaitEvent(s, ev[k], 0);
    if (e != cudaSuccess) {
      status = fail(FS_CUDA_ERROR, std::string("staged upload: ") + cudaGetErrorString(e));
      break;
    }
    status = launch_search(plan, pl, dst, n, static_cast<char*>(out_dev) + off * ob, ob, fb, off, s);
  }
  unsigned long long bad = ~0ull;
  if (status == FS_OK) {
    cudaError_t e = cudaMemcpyAsync(&bad, fb, sizeof(bad), cudaMemcpyDeviceToHost, s);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    if (e != cudaSuccess) status = fail(FS_CUDA_ERROR, std::string("first-bad readback: ") + cudaGetErrorString(e));
  }
  if (status == FS_OK && bad != ~0ull) {
    if (pos_out) *pos_out = (int64_t)bad;
    gate.arrive(false);
    status = fail(FS_OUT_OF_DOMAIN, "query outside [X0, XN)");
  }
  if (status == FS_OK && !gate.arrive(true)) status = fail(FS_ABORTED, "another span of the batch is out of domain");
  // phase 2: download (only for a clean batch)
  if (status == FS_OK) {
    const uint64_t nch = (m + chunk - 1) / chunk;
    for (uint64_t i = 0; i <= nch && status == FS_OK; ++i) {
      if (i < nch) {  // DMA of chunk i into its slot
        const uint64_t off = i * chunk, n = std::min(chunk, m - off);
        cudaError_t e = cudaMemcpyAsync(slot[i % kSlots], static_cast<const char*>(out_dev) + off * ob, n * ob,
                                        cudaMemcpyDeviceToHost, cs);
        if (e == cudaSuccess) e = cudaEventRecord(ev[i % kSlots], cs);
        if (e != cudaSuccess) status = fail(FS_CUDA_ERROR, std::string("staged download: ") + cudaGetErrorString(e));
      }
      if (i >= 1 && status == FS_OK) {  // host copy of chunk i-1 while chunk i is in flight
        const uint64_t off = (i - 1) * chunk, n = std::min(chunk, m - off);
        const int k = (int)((i - 1) % kSlots);
        if (cudaEventSynchronize(ev[k]) != cudaSuccess) status = fail(FS_CUDA_ERROR, "staging slot wait failed");
        else host_copy(static_cast<char*>(out_host) + off * ob, slot[k], n * ob, copy_threads);
      }
    }
  }
  cudaStreamSynchronize(cs);
  for (int i = 0; i < kSlots; ++i) {
    if (ev[i]) cudaEventDestroy(ev[i]);
    if (slot[i]) PinnedSlots::release(slot[i]);
  }
  return status;
}

}  // namespace

fs_gate* fs_gate_create(int32_t parties) {
  if (parties < 1) return nullptr;
  fs_gate* g = new (std::nothrow) fs_gate();
  if (g) g->parties = parties;
  return g;
}

void fs_gate_abort(fs_gate* gate) {
  if (gate) gate->abort();
}

void fs_gate_destroy(fs_gate* gate) { delete gate; }

int fs_search_host(const fs_plan* plan, const void* z_host, uint64_t m, void* out_host, int32_t out_bytes, void* z_dev,
                   void* out_dev, unsigned long long* first_bad_dev, uint64_t chunk_elems, int64_t* pos_out,
                   void* stream, void* copy_stream, int32_t flags) {
  return fs_search_host_gated(plan, z_host, m, out_host, out_bytes, z_dev, out_dev, first_bad_dev, chunk_elems,
                              pos_out, stream, copy_stream, flags, nullptr);
}

int fs_search_host_gated(const fs_plan* plan, const void* z_host, uint64_t m, void* out_host, int32_t out_bytes,
                         void* z_dev, void* out_dev, unsigned long long* first_bad_dev, uint64_t chunk_elems,
                         int64_t* pos_out, void* stream, void* copy_stream, int32_t flags, fs_gate* gate_ptr) {
  // the speculative mode promises nothing about other spans: no gate
  GateArrival gate((flags & FS_HOST_OVERLAP) ? nullptr : gate_ptr);
  int rc = check_search_args(plan, z_dev, m, out_dev, out_bytes, first_bad_dev);
  if (rc) return rc;
  if (m && (!z_host || !out_host)) return fail(FS_INVALID_ARG, "host pointer is NULL");
  cudaStream_t s = as_stream(stream), cs = as_stream(copy_stream);
  if (m && cs != s) {
    // The uploads run on the copy stream into z_dev, memory the caller's
    // allocator may have just recycled from buffers that work still queued
    // on `stream` reads or writes (e.g. an index build's scratch).  Order the
    // copy stream after everything already queued on `stream`.
    cudaEvent_t entry;
    FS_CUDA(cudaEventCreateWithFlags(&entry, cudaEventDisableTiming));
    cudaError_t e = cudaEventRecord(entry, s);
    if (e == cudaSuccess) e = cudaStreamWaitEvent(cs, entry, 0);
    cudaEventDestroy(entry);
    if (e != cudaSuccess) return fail(FS_CUDA_ERROR, std::string("stream ordering: ") + cudaGetErrorString(e));
  }
  // pageable buffers of any real size go through the library's own pinned staging
  const HostChunking hc = host_chunking(plan, z_host, m, out_host, out_bytes, chunk_elems, flags);
  if (hc.staged)
    return search_host_staged(plan, place_for_batch(plan, m), z_host, m, out_host, out_bytes, z_dev, out_dev,
                              first_bad_dev, pos_out, s, cs, gate);
  const bool overlap = (flags & FS_HOST_OVERLAP) != 0;
  const size_t es = plan->dtype == FS_F32 ? 4 : 8;
  chunk_elems = hc.chunk;
  Placement pl = place_for_batch(plan, m);
  pl.merge = 1;  // every chunk min-merges into status[0]
  // atomic mode over several chunks: host threads check the domain while the
  // chunks upload, so write-back can start before the last upload
  const uint64_t nch = (m + chunk_elems - 1) / chunk_elems;
  const bool precheck = !overlap && !(flags & FS_HOST_NO_PRECHECK) && nch >= 2;
  // Per-call resources.  On every exit the streams are drained before
  // anything is released: no copy may still read the caller's buffers or
  // write a pinned slot that is back in the process-wide cache.
  struct CallState {
    cudaStream_t s, cs, ds = nullptr;
    cudaEvent_t ev = nullptr, evk = nullptr;
    std::vector<cudaEvent_t> done;  // precheck: kernel of chunk c finished ...
    unsigned long long* prefix_bad = nullptr;  // ... with this first-bad word (pinned)
    ~CallState() {
      cudaStreamSynchronize(s);
      cudaStreamSynchronize(cs);
      if (ds) {
        cudaStreamSynchronize(ds);
        cudaStreamDestroy(ds);
      }
      for (cudaEvent_t d : done) cudaEventDestroy(d);
      if (ev) cudaEventDestroy(ev);
      if (evk) cudaEventDestroy(evk);
      if (prefix_bad) PinnedSlots::release(prefix_bad);
    }
  } st{s, cs};
  FS_CUDA(cudaMemsetAsync(first_bad_dev, 0xff, sizeof(unsigned long long), s));
  if (precheck && !(st.prefix_bad = static_cast<unsigned long long*>(PinnedSlots::acquire(nch * 8))))
    return fail(FS_CUDA_ERROR, "pinned status allocation failed");
  FS_CUDA(cudaEventCreateWithFlags(&st.ev, cudaEventDisableTiming));
  FS_CUDA(cudaEventCreateWithFlags(&st.evk, cudaEventDisableTiming));
  if (overlap || precheck) FS_CUDA(cudaStreamCreateWithFlags(&st.ds, cudaStreamNonBlocking));
  cudaEvent_t ev = st.ev, evk = st.evk;
  cudaStream_t ds = st.ds;
  std::vector<cudaEvent_t>& done = st.done;
  unsigned long long* prefix_bad = st.prefix_bad;
  int status = FS_OK;
  bool wrote = false, aborted = false;
  for (uint64_t off = 0; off < m && status == FS_OK; off += chunk_elems) {
    const uint64_t n = std::min(chunk_elems, m - off);
    const char* src = static_cast<const char*>(z_host) + off * es;
    char* dst = static_cast<char*>(z_dev) + off * es;
    char* odev = static_cast<char*>(out_dev) + off * out_bytes;
    cudaError_t e = cudaMemcpyAsync(dst, src, n * es, cudaMemcpyHostToDevice, cs);
    if (e == cudaSuccess) e = cudaEventRecord(ev, cs);
    if (e == cudaSuccess) e = cudaStreamWaitEvent(s, ev, 0);
    if (e != cudaSuccess) {
      status = fail(FS_CUDA_ERROR, std::string("chunk upload: ") + cudaGetErrorString(e));
      break;
    }
    status = launch_search(plan, pl, dst, n, odev, out_bytes, first_bad_dev, off, s);
    if (status == FS_OK && overlap) {
      // speculative write-back on a third stream: D2H of chunk c runs while
      // the H2D of chunk c+1 is in flight (the two copy engines are independent)
      e = cudaEventRecord(evk, s);
      if (e == cudaSuccess) e = cudaStreamWaitEvent(ds, evk, 0);
      if (e == cudaSuccess)
        e = cudaMemcpyAsync(static_cast<char*>(out_host) + off * out_bytes, odev, n * (uint64_t)out_bytes,
                            cudaMemcpyDeviceToHost, ds);
      if (e != cudaSuccess) status = fail(FS_CUDA_ERROR, std::string("chunk download: ") + cudaGetErrorString(e));
    }
    if (status == FS_OK && precheck) {  // the device's verdict on chunks 0..c, then done[c]
      cudaEvent_t d;
      cudaError_t e = cudaMemcpyAsync(&prefix_bad[done.size()], first_bad_dev, sizeof(unsigned long long),
                                      cudaMemcpyDeviceToHost, s);
      if (e == cudaSuccess) e = cudaEventCreateWithFlags(&d, cudaEventDisableTiming);
      if (e == cudaSuccess) {
        done.push_back(d);
        e = cudaEventRecord(d, s);
      }
      if (e != cudaSuccess) status = fail(FS_CUDA_ERROR, std::string("chunk event: ") + cudaGetErrorString(e));
    }
  }
  // every upload and search is queued: establish "no query is bad" from both
  // ends meanwhile, then queue each chunk's write-back behind its kernel
  if (status == FS_OK && precheck) {
    const int64_t nd = (int64_t)done.size();
    bool clean =
        plan->dtype == FS_F32
            ? domain_clean_two_sided<float>(static_cast<const float*>(z_host), m, chunk_elems, (float)plan->x0,
                                            (float)plan->xn, host_scan_threads(), done.data(), prefix_bad, nd)
            : domain_clean_two_sided<double>(static_cast<const double*>(z_host), m, chunk_elems, plan->x0, plan->xn,
                                             host_scan_threads(), done.data(), prefix_bad, nd);
    // every other span of a gated batch must be clean too before any write-back
    aborted = !gate.arrive(clean) && clean;
    clean = clean && !aborted;
    for (uint64_t c = 0; clean && c < done.size() && status == FS_OK; ++c) {
      const uint64_t off = c * chunk_elems, n = std::min(chunk_elems, m - off);
      cudaError_t e = cudaStreamWaitEvent(ds, done[c], 0);
      if (e == cudaSuccess)
        e = cudaMemcpyAsync(static_cast<char*>(out_host) + off * out_bytes,
                            static_cast<const char*>(out_dev) + off * out_bytes, n * (uint64_t)out_bytes,
                            cudaMemcpyDeviceToHost, ds);
      if (e != cudaSuccess) status = fail(FS_CUDA_ERROR, std::string("chunk download: ") + cudaGetErrorString(e));
      wrote = true;
    }
  }
  unsigned long long bad = ~0ull;
  if (status == FS_OK) {
    cudaError_t e = cudaMemcpyAsync(&bad, first_bad_dev, sizeof(bad), cudaMemcpyDeviceToHost, s);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    if (e == cudaSuccess && ds) e = cudaStreamSynchronize(ds);
    if (e != cudaSuccess) status = fail(FS_CUDA_ERROR, std::string("first-bad readback: ") + cudaGetErrorString(e));
  }
  if (status != FS_OK) return status;
  if (bad != ~0ull) {
    if (pos_out) *pos_out = (int64_t)bad;
    gate.arrive(false);
    if (wrote) return fail(FS_INCONSISTENT, "host and device domain checks disagree (queries modified during the call?)");
    return fail(FS_OUT_OF_DOMAIN, "query outside [X0, XN)");
  }
  if (aborted || !gate.arrive(true)) return fail(FS_ABORTED, "another span of the batch is out of domain");
  if (m && !overlap && !wrote) {
    FS_CUDA(cudaMemcpyAsync(out_host, out_dev, m * (uint64_t)out_bytes, cudaMemcpyDeviceToHost, s));
    FS_CUDA(cudaStreamSynchronize(s));
  }
  return FS_OK;
}

size_t fs_crc32_ws_bytes(uint64_t bytes) {
  const uint64_t nchunks = (bytes + kCrcChunk - 1) / kCrcChunk;
  return (size_t)std::max<uint64_t>(nchunks, 1) * sizeof(uint32_t);
}

int fs_crc32(const void* data_dev, uint64_t bytes, void* ws_dev, uint32_t* crc_out, void* stream) {
  if (!crc_out || (bytes && (!data_dev || !ws_dev))) return fail(FS_INVALID_ARG, "NULL pointer");
  if (bytes == 0) {
    *crc_out = 0;
    return FS_OK;
  }
  cudaStream_t s = as_stream(stream);
  uint32_t* c = static_cast<uint32_t*>(ws_dev);
  const uint64_t nchunks = (bytes + kCrcChunk - 1) / kCrcChunk;
  crc32_chunks_kernel<<<grid_1d(nchunks, 256), 256, 0, s>>>(static_cast<const unsigned char*>(data_dev), bytes, c,
                                                           nchunks);
  FS_CUDA(cudaGetLastError());
  for (uint64_t step = 1; step < nchunks; step *= 2) {
    const uint64_t pairs = (nchunks + 2 * step - 1) / (2 * step);
    crc32_combine_kernel<<<grid_1d(pairs, 256), 256, 0, s>>>(c, nchunks, step, bytes);
    FS_CUDA(cudaGetLastError());
  }
  FS_CUDA(cudaMemcpyAsync(crc_out, c, sizeof(uint32_t), cudaMemcpyDeviceToHost, s));
  FS_CUDA(cudaStreamSynchronize(s));
  return FS_OK;
}

int fs_plan_placement(const fs_plan* plan, int32_t* placement_out, uint64_t* smem_bytes_out) {
  int rc = validate_plan(plan);
  if (rc) return rc;
  const Placement pl = place(plan);
  if (placement_out) *placement_out = pl.flags;
  if (smem_bytes_out) *smem_bytes_out = pl.smem;
  return FS_OK;
}

int fs_search_launches(const fs_plan* plan, uint64_t m) {
  if (validate_plan(plan)) return -1;
  return m ? 1 : 0;  // launch_search: exactly one kernel; an empty batch only resets the status word
}

int64_t fs_search_host_launches(const fs_plan* plan, const void* z_host, uint64_t m, const void* out_host,
                                int32_t out_bytes, uint64_t chunk_elems, int32_t flags) {
  if (validate_plan(plan) || (out_bytes != 4 && out_bytes != 8)) return -1;
  if (m == 0) return 0;
  const HostChunking hc = host_chunking(plan, z_host, m, out_host, out_bytes, chunk_elems, flags);
  return (int64_t)((m + hc.chunk - 1) / hc.chunk);  // one search kernel per chunk (staged or pinned)
}

}  // extern "C"
