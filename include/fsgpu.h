/*
 * fsgpu.h — C-ABI of the B200 (sm_100a) sorted-interval lookup library.
 *
 * The reference (`fastsearch` 0.1.0, /root/reference/pkg) is pure Python +
 * numpy; its "FFI" for the hot path is the operator boundary in
 * pkg/src/fastsearch/batch.py (prepare / PreparedKernel.lanes / batch_search)
 * and the index builder in pkg/src/fastsearch/direct.py.  Every entry point
 * below replaces one of those functions; the reference interface it stands
 * in for is cited beside it.  A Python (ctypes) binding of exactly these
 * symbols lives in paper_1506_08620_b200/_lib.py; INTEGRATION.md shows the
 * stub a fastsearch maintainer would add.
 *
 * Conventions
 *  - Plain pointers and sizes only.  "dev" pointers are CUDA device memory;
 *    "host" pointers are host memory (pinned or pageable).
 *  - Every call is stream-ordered on the cudaStream_t passed as `void*`
 *    (NULL = legacy default stream).  Calls marked SYNC synchronise that
 *    stream before returning; all others are asynchronous.
 *  - Calls are thread-safe.  The only process-wide state is an idempotent,
 *    mutex-guarded cache of launch geometry (occupancy results and the
 *    dynamic-shared-memory attribute) per (device, kernel, smem size).
 *  - Return value: an fs_status code.  Positions (first offending element)
 *    are written through `pos_out` where the reference exception carries a
 *    `position` attribute (errors.py:28-62).
 *  - Floating point semantics are the reference's numpy semantics: IEEE-754
 *    round-to-nearest-even in the partition's own precision, subnormals kept
 *    (no FTZ), no contraction, truncation toward zero for the bucket index.
 */
#ifndef FSGPU_H
#define FSGPU_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- status codes (map 1:1 onto fastsearch.errors, errors.py:1-82) ---- */
typedef enum fs_status {
  FS_OK = 0,
  FS_NOT_DISTINGUISHABLE = 1, /* errors.NotDistinguishable(position)          */
  FS_OVERFLOW = 2,            /* errors.Overflow                              */
  FS_OUT_OF_DOMAIN = 3,       /* errors.OutOfDomain(position)                 */
  FS_INVALID_ARG = 4,         /* ValueError (qbits, q, sizes, dtype, ...)     */
  FS_CUDA_ERROR = 5,          /* CUDA runtime failure; see fs_last_error()    */
  FS_INCONSISTENT = 6,        /* build_index: "(h, r) pair is inconsistent";
                                 fs_search_host: host/device checks disagree */
  FS_TOO_LARGE = 7,           /* table/workspace does not fit the device path */
  FS_ABORTED = 8              /* fs_search_host_gated: another span of the same
                                 batch is out of domain; nothing written      */
} fs_status;

/* ---- element types ---- */
enum { FS_F32 = 0, FS_F64 = 1 };

/* ---- algorithms: the names of batch.ALGORITHMS (batch.py:35-45) ---- */
enum {
  FS_ALGO_CLASSIC = 0,      /* binsearch.classic_seq      binsearch.py:48-57   */
  FS_ALGO_BITSET1 = 1,      /* binsearch.bitset1_seq      binsearch.py:60-69   */
  FS_ALGO_BITSET2 = 2,      /* binsearch.bitset2_seq      binsearch.py:72-86   */
  FS_ALGO_BITSET3 = 3,      /* binsearch.bitset3_seq      binsearch.py:89-99   */
  FS_ALGO_OFFSET = 4,       /* binsearch.offset_seq       binsearch.py:102-114 */
  FS_ALGO_EYTZINGER = 5,    /* eytzinger.eytzinger_seq    eytzinger.py:84-89   */
  FS_ALGO_DIRECT = 6,       /* batch lanes, gap 1         batch.py:315-317     */
  FS_ALGO_DIRECT_GAP2 = 7,  /* batch lanes, gap 2         batch.py:341-343     */
  FS_ALGO_DIRECT_CACHE = 8, /* batch lanes, fused records batch.py:368-371     */
  FS_ALGO_DIRECT_GENERIC = 9 /* direct.direct_search_generic direct.py:294-300 */
};

/* ---- table placement (reported by fs_plan_placement) ---- */
enum {
  FS_PLACE_GLOBAL = 0,  /* tables gathered through L2 (ld.global.nc)               */
  FS_PLACE_SMEM_X = 1,  /* knots (or padded/tree array) staged in shared memory   */
  FS_PLACE_SMEM_K = 2,  /* bucket table / fused records staged in shared memory   */
  FS_PLACE_SMEM_TOP = 4,/* bitset2: top levels in smem, bottom levels via L2      */
  FS_PLACE_SMEM_HOT = 8,/* direct: hot window of directory + knots in smem        */
  FS_PLACE_SMEM_SPARSE = 16 /* direct: two-level sparse table in smem              */
};

/* ---- layouts of fs_plan.sparse ---- */
enum {
  FS_SPARSE_TWO_LEVEL = 0, /* C | F (| dense masks): fs_build_sparse                */
  FS_SPARSE_RECORDS = 1,   /* 16-B group records, six offsets (| F): fs_build_sparse_rec */
  FS_SPARSE_RECORDS8 = 2,  /* 8-B group records, two offsets (| F): fs_build_sparse_rec  */
  FS_SPARSE_RECORDS12 = 3, /* 16-B group records, eight 12-bit offsets (shift <= 10)      */
  FS_SPARSE_RECORDS8X3 = 4,/* 8-B group records, three 13-bit offsets (shift <= 11, N+1 <= 2^24) */
  FS_SPARSE_ZONED = 5,     /* zone descriptors | 8-B records, per-zone form: fs_build_zoned  */
  FS_SPARSE_ZONED_RANK = 6,/* zone descriptors | 8-B striped rank words: fs_build_zoned_rank */
  FS_SPARSE_COUNT = 7,     /* 8-B count words, one stripe shift for the table: fs_build_count_words */
  FS_SPARSE_KNOT_BYTES = 8,/* a byte per knot beside the rank directory (fs_plan.rank): fs_build_knot_bytes */
  FS_SPARSE_RANK_ROWS = 9  /* 16-B rank rows {mask, base, eight knot bytes} read through L2: fs_build_rank_rows */
};

/*
 * A prepared search structure resident in device memory — the device image
 * of batch.PreparedKernel.structure (batch.py:132-140).  All pointers are
 * device pointers owned by the caller.
 */
typedef struct fs_plan {
  int32_t algorithm;  /* FS_ALGO_*                                               */
  int32_t dtype;      /* FS_F32 / FS_F64                                         */
  uint64_t n1;        /* number of knots N+1 (>= 2)                              */
  const void* x;      /* knots X[0..N], n1 elements of dtype                     */
  const void* table;  /* direct/gap2/generic: K (uint32, r+1 entries);
                         direct-cache: fused records ((r+1) x 8 B f32 / 16 B f64);
                         bitset2: padded knots (2^pbits elements);
                         eytzinger: heap-order tree (2^pbits - 1 elements);
                         others: unused (NULL)                                     */
  uint64_t r;         /* direct family: bucket count R (table has R+1 entries)   */
  double h;           /* direct family: scale factor H (exact in dtype)          */
  double x0, xn;      /* domain [X0, XN) (exact in dtype)                        */
  int32_t q;          /* direct family: gap (1, 2, >2 generic)                   */
  int32_t pbits;      /* bitset family: bit_length(N); eytzinger: depth L   */
  int32_t smem_policy;/* 0 auto, 1 force global (L2) gathers                      */
  int32_t tune;       /* launch-geometry override for tuning runs, 0 = auto:
                         bits 0-11 threads per CTA, bits 12-19 max CTAs per SM   */
  const void* rank;   /* direct, optional: rank directory of K (gap 1:
                         fs_build_rank, 8-B words; generic gap q:
                         fs_build_countdir, 8-B words; gap 2: fs_build_rank2, 16-B
                         words); when set the kernel reads it instead of K.
                         NULL = read K.                                           */
  const void* records;/* direct (gap 1) only, optional: fused (K[j], X[K[j]])
                         records (fs_build_fused); used, staged in shared
                         memory, when they fit there.  NULL = unused.            */
  uint64_t hot_word0, hot_words;  /* direct over `rank`, optional: directory words
                         [hot_word0, +hot_words) staged in shared memory ...     */
  uint64_t hot_knot0, hot_knots;  /* ... with knots X[hot_knot0, +hot_knots);
                         hot_words = 0: no hot window (fs_build_hot_window).     */
  const void* sparse; /* direct (gap 1) only, optional: two-level sparse table
                         (fs_build_sparse); staged in shared memory when the
                         rank directory does not fit there.  NULL = unused.      */
  int32_t sparse_shift;/* super-bucket = 2^sparse_shift buckets (5..16);
                          zoned: zone = 2^sparse_shift buckets (10..31)         */
  uint32_t sparse_ndense; /* two-level: dense (bitmask) super-buckets in `sparse`;
                             records: overflowing records (> 0: F follows);
                             zoned: number of 8-B records                       */
  const void* b2_deep;  /* bitset2 only, optional: subtree records of the levels
                           below the shared-memory top (fs_build_b2_deep); one
                           32-B gather resolves b2_deep_k levels.  NULL = unused. */
  int32_t b2_deep_top;  /* ... built for this many staged top levels             */
  int32_t b2_deep_k;    /* ... levels per record (3 for f32, 2 for f64)           */
  int32_t sparse_format;/* layout of `sparse`: FS_SPARSE_TWO_LEVEL (fs_build_sparse)
                           or FS_SPARSE_RECORDS / FS_SPARSE_RECORDS8 /
                           FS_SPARSE_RECORDS12 / FS_SPARSE_RECORDS8X3
                           (fs_build_sparse_rec)                                  */
} fs_plan;

/* Library identification: "fsgpu <version> (sm_100a) src <16 hex>", the last
   field hashing the sources and nvcc flags the library was built from. */
const char* fs_version(void);
/* Message for the last FS_CUDA_ERROR / FS_INVALID_ARG on this thread. */
const char* fs_last_error(void);
/* Bytes of device workspace the build entry points need (status block). */
size_t fs_workspace_bytes(void);

/* ---------------------------------------------------------------------------
 * Index construction (direct.py:135-263)
 * ------------------------------------------------------------------------ */

/*
 * Certified scale factor.  Replaces direct.compute_h_r (direct.py:135-191):
 * D = RN(X - X0); collision of D[i+q] == D[i] -> FS_NOT_DISTINGUISHABLE with
 * *pos_out = first i+q; h = RN(1 / min RN(D[i+b] - D[i])), b = min(q, N);
 * FS_OVERFLOW unless RN(h * D_N) < 2^qbits; growth loop with doubling ulp
 * increments re-certifying every pair; r = floor(RN(h * D_N)).
 * h_out / h_start_out receive the values in the partition's dtype (float* or
 * double*).  SYNC (one device->host read per growth iteration).
 */
int fs_certify(int32_t dtype, const void* x_dev, uint64_t n1, int32_t qbits, int32_t q,
               void* ws_dev, void* h_out, void* h_start_out, uint64_t* r_out,
               uint32_t* increments_out, int64_t* pos_out, void* stream);

/*
 * Knot buckets f_i = floor(RN(h * RN(X_i - X0))) as uint64.  Replaces
 * direct.knot_buckets (direct.py:194-197).
 */
int fs_knot_buckets(int32_t dtype, const void* x_dev, uint64_t n1, double h, uint64_t* f_dev,
                    void* stream);

/*
 * Bucket table K.  Replaces direct.build_index (direct.py:200-243) and
 * knot_buckets (direct.py:194-197): f_i = floor(RN(h * RN(X_i - X0)));
 * FS_INCONSISTENT unless f_N == r; q == 1: K[j] = i for f_{i-1} < j <= f_i,
 * K[0] = 0; q > 1: K[j] = max{i : f_i <= j}.  k_dev holds r+1 uint32.
 * f_scratch_dev holds n1 uint64.  SYNC (reads back the consistency flag).
 */
int fs_build_table(int32_t dtype, const void* x_dev, uint64_t n1, double h, uint64_t r,
                   int32_t q, uint32_t* k_dev, uint64_t* f_scratch_dev, void* ws_dev,
                   void* stream);

/*
 * Rank directory of the gap-1 table: the same K in 2 bits per bucket.
 * For a certified gap-1 index every bucket holds at most one knot, so
 * K[j] = #{i : f_i < j} steps by 0 or 1 per bucket.  Word w (buckets
 * 32w..32w+31) is {mask_w, base_w} (8 B): bit b of mask_w is set iff some
 * f_i == 32w + b, and base_w = K[32w].  Then K[j] = base_w + popc(mask_w &
 * (2^b - 1)) exactly, and when bit b is clear the fix-up comparison of
 * batch.py:317 is known to hold (z < X[K[j]]) without reading X.
 * dir_dev holds (r >> 5) + 1 uint2 words; f_scratch_dev n1 uint64.
 */
int fs_build_rank(int32_t dtype, const void* x_dev, uint64_t n1, double h, uint64_t r,
                  uint64_t* f_scratch_dev, void* dir_dev, void* stream);

/*
 * Rank directory of the gap-2 table (a device layout of build_index with
 * q = 2, direct.py:200-243; no reference counterpart).  A gap-2 certificate
 * allows at most two knots per bucket, so each 32-bucket word is 16 B
 * {m1: buckets with a knot, m2: buckets with two, base = K-count before the
 * word, 0}; the gap-2 kernel recovers K2[j] exactly and reads X only for
 * buckets holding knots.  dir_dev holds (r >> 5) + 1 words; set it as
 * fs_plan.rank of a FS_ALGO_DIRECT_GAP2 plan.
 */
/*
 * Count directory of a gap-q table, q = 2..15 (a device layout of
 * build_index with q > 1, direct.py:200-243, searched as
 * direct_search_generic, direct.py:294-300; no reference counterpart).  A
 * gap-q certificate allows at most q knots per bucket, so a bucket's count
 * fits 2 bits (q <= 3; 16 buckets per word) or 4 bits (q <= 15; 8 per word):
 * 8-B words {counts, base = #knots before the word}.  The kernel recovers
 * K_q[j] exactly and compares z only with the knots of its own bucket.
 * This is what makes a larger gap a practical answer to an infeasible gap-1
 * layout (the minimal q that meets a memory budget).
 * dir_dev holds fs_countdir_bytes(q, r) bytes; set it as fs_plan.rank of a
 * FS_ALGO_DIRECT_GENERIC plan with the same q.
 */
uint64_t fs_countdir_bytes(int32_t q, uint64_t r);
int fs_build_countdir(int32_t dtype, const void* x_dev, uint64_t n1, double h, uint64_t r, int32_t q,
                      uint64_t* f_scratch_dev, void* dir_dev, void* stream);

int fs_build_rank2(int32_t dtype, const void* x_dev, uint64_t n1, double h, uint64_t r,
                   uint64_t* f_scratch_dev, void* dir_dev, void* stream);

/*
 * Two-level sparse encoding of the gap-1 table, for R >> N.  Super-bucket J
 * (2^shift buckets) stores C[J] = K[J 2^shift] (uint32, (r >> shift) + 2
 * entries, the last = n1); each knot i stores F[i] = f_i mod 2^shift
 * (uint16, n1 entries) after C.  Then K[j] = C[j >> shift] +
 * #{i in [C[J], C[J+1]) : F[i] < j mod 2^shift} exactly, and bucket j holds
 * knot t = K[j] iff F[t] == j mod 2^shift.  Super-buckets with more than 64
 * knots are DENSE: bit 31 of C[J] is set, F[C[J]] holds a slot, and the
 * slot's 2^shift-bit knot mask (uint32 words) and per-word prefix counts
 * (uint16) follow F -- K[j] = C[J] + prefix + popc(mask below j), as in the
 * rank directory.  Layout: C | F | pad to 4 | masks | prefixes.
 *   fs_sparse_bytes: buffer size for (shift, ndense).
 *   fs_plan_sparse: smallest shift (5..16) whose table (plus X when with_x)
 *     fits in budget_bytes -> shift, ndense, bytes; FS_TOO_LARGE if none.  SYNC.
 *   fs_build_sparse: fill the buffer for that shift.  SYNC.
 * f_scratch_dev: n1 uint64.
 */
uint64_t fs_sparse_bytes(uint64_t n1, uint64_t r, int32_t shift, uint64_t ndense);
int fs_plan_sparse(int32_t dtype, const void* x_dev, uint64_t n1, double h, uint64_t r, uint64_t budget_bytes,
                   int32_t with_x, uint64_t* f_scratch_dev, int32_t* shift_out, uint64_t* ndense_out,
                   uint64_t* bytes_out, void* stream);
int fs_build_sparse(int32_t dtype, const void* x_dev, uint64_t n1, double h, uint64_t r, int32_t shift,
                    uint64_t* f_scratch_dev, void* sparse_dev, void* stream);

/*
 * Group records of the gap-1 table (a device layout of build_index,
 * direct.py:200-243; no reference counterpart), for R >> N.  The
 * super-buckets of fs_build_sparse, each packed into one record {base |
 * overflow flag (bit 31), S uint16 knot offsets}: FS_SPARSE_RECORDS is 16 B
 * with S = 6, FS_SPARSE_RECORDS8 is 8 B with S = 2, FS_SPARSE_RECORDS12 is
 * 16 B with S = 8 offsets in 12-bit fields (0x800 | offset at bit 12k of the
 * 96 bits after base, unused 0xFFF; shift <= 10), FS_SPARSE_RECORDS8X3 is 8 B
 * with S = 3: the 64-bit word holds base (bits 0..23, so N+1 <= 2^24), the
 * overflow flag (bit 24) and fields 0x1000 | offset at bits 25 + 13k (unused
 * 0x1FFF; shift <= 11).  base = K[J 2^shift], the
 * offsets f_i mod 2^shift of the super-bucket's first min(count, S) knots in
 * ascending order, unused slots 0x7FFF.  The kernel resolves
 * K[j] = base + #{offsets < j mod 2^shift} from one shared-memory load, and
 * bucket j holds knot K[j] iff that offset slot equals j mod 2^shift.  A
 * super-bucket with more than S knots sets bit 31; its later knots are
 * searched in F (f_i mod 2^shift, uint16 per knot), which follows the
 * (r >> shift) + 2 records only when some record overflows.
 *   fs_sparse_rec_bytes: buffer size for (format, shift, novf overflowing
 *     records); 0 for an invalid format or shift.
 *   fs_plan_sparse_rec: the shift (5..14) whose layout (plus X when with_x)
 *     fits in budget_bytes and sends the fewest queries past a record's last
 *     offset (uniform queries; among shifts within 1e-3 of the best, the
 *     smallest table) -> shift, novf, bytes, and that fraction in parts per
 *     million.  FS_TOO_LARGE if none fits.  SYNC.
 *   fs_build_sparse_rec: fill the buffer (F too when novf > 0).  SYNC.
 * Set fs_plan.sparse to the buffer, sparse_shift to the shift,
 * sparse_ndense to novf and sparse_format to the format.
 * f_scratch_dev: n1 uint64.
 */
uint64_t fs_sparse_rec_bytes(int32_t format, uint64_t n1, uint64_t r, int32_t shift, uint64_t novf);
int fs_plan_sparse_rec(int32_t format, int32_t dtype, const void* x_dev, uint64_t n1, double h, uint64_t r,
                       uint64_t budget_bytes, int32_t with_x, uint64_t* f_scratch_dev, int32_t* shift_out,
                       uint64_t* novf_out, uint64_t* bytes_out, uint32_t* past_last_ppm_out, void* stream);
int fs_build_sparse_rec(int32_t format, int32_t dtype, const void* x_dev, uint64_t n1, double h, uint64_t r,
                        int32_t shift, uint64_t novf, uint64_t* f_scratch_dev, void* buf_dev, void* stream);

/*
 * Zoned records of the gap-1 table (FS_SPARSE_ZONED; a device layout of K,
 * no reference counterpart).  The buckets [0, R] are cut into nz = (R >>
 * zs) + 1 <= 64 zones of 2^zs buckets (zs >= 11), and each zone takes the
 * 8-B record form its own knot density needs: slot records (the
 * FS_SPARSE_RECORDS8X3 word: K[j0] in bits 0..23, three fields 0x1000 |
 * (f_i - j0) at bits 25 + 13k, unused 0x1FFF) per 2^s buckets (s = 6..11,
 * the largest whose records hold at most three knots), else rank records
 * {mask of the 32 buckets holding a knot, K[j0]}.  N+1 <= 2^24.
 * Buffer: nz u32 descriptors ((first record - (z << (zs - s))) << 5, as a
 * signed 27-bit value | 16 if rank | s), padded to
 * a multiple of four, then the records.  The kernel resolves K[j] from one
 * descriptor and one record load, both in shared memory, and reads X only for
 * a bucket holding a knot -- from a staged window X[t0, t0 + nt) or L2.
 *   fs_plan_zoned: the zone shift (the fewest zones, 32 or 64, whose table
 *     fits budget_bytes) -> zs, records, table bytes, and the window of X
 *     (the densest nt consecutive knots, nt = as many as the rest of the
 *     budget holds).  FS_TOO_LARGE if no zoning fits.  SYNC.
 *   fs_build_zoned: fill the buffer for that zs.  SYNC.
 * Set fs_plan.sparse to the buffer, sparse_format = FS_SPARSE_ZONED,
 * sparse_shift = zs, sparse_ndense = records, hot_knot0 = t0, hot_knots = nt
 * (hot_words = 0).  f_scratch_dev: n1 uint64.
 */
uint64_t fs_zoned_bytes(uint64_t r, int32_t zs, uint64_t nrec);
int fs_plan_zoned(int32_t dtype, const void* x_dev, uint64_t n1, double h, uint64_t r, uint64_t budget_bytes,
                  uint64_t* f_scratch_dev, int32_t* zs_out, uint64_t* nrec_out, uint64_t* bytes_out,
                  uint64_t* t0_out, uint64_t* nt_out, void* stream);
int fs_build_zoned(int32_t dtype, const void* x_dev, uint64_t n1, double h, uint64_t r, int32_t zs,
                   uint64_t* f_scratch_dev, void* buf_dev, void* stream);

/*
 * Striped rank words of the gap-1 table (FS_SPARSE_ZONED_RANK; a device
 * layout of K, no reference counterpart).  The same zones as above, every
 * zone in 8-B rank words {mask, K[j0]} whose 32 mask bits each stand for a
 * stripe of 2^k buckets (a word covers 2^(k+5) buckets from j0), k per zone
 * (0..10) and never so large that a stripe holds two knots.  For bucket j
 * of the query z, b = (j >> k) & 31 and t = K[j0] + popc(mask below bit b):
 * the knots of earlier stripes lie below z and those of later stripes above
 * it (the bucket function of direct.py:194-197 is monotone), so the answer of
 * batch.py:315-317 is t - 1 when bit b is clear and t - (z < X[t]) when it is
 * set -- X is read whenever the query's stripe holds a knot, from the staged
 * window X[t0, t0 + nt) or L2.  The decode is a mask and a popcount; tables
 * with smoothly varying gaps (cfg4's geometric knots) fit in shared memory
 * with stripes of a few buckets.
 * Buffer: nz u32 descriptors ((first word - (z << (zs - k - 5))) << 5, as a
 * signed 27-bit value | 16 | k), padded to a multiple of four, then the words.
 *   fs_plan_zoned_rank: zs, words, table bytes and the window of X for
 *     budget_bytes (an eighth of it is kept for the window; the stripes are
 *     refined, densest zone first, while the words fit the rest), plus the
 *     share of the buckets lying in knot-holding stripes in parts per million
 *     (uniform queries that read X).  FS_TOO_LARGE if nothing fits.  SYNC.
 *   fs_build_zoned_rank: fill the buffer for (zs, nrec) as planned;
 *     FS_INVALID_ARG if no plan of that zone shift has nrec words.  SYNC.
 * Set fs_plan.sparse to the buffer, sparse_format = FS_SPARSE_ZONED_RANK,
 * sparse_shift = zs, sparse_ndense = nrec, hot_knot0 = t0, hot_knots = nt
 * (hot_words = 0).  Bytes: fs_zoned_bytes.  f_scratch_dev: n1 uint64.
 */
int fs_plan_zoned_rank(int32_t dtype, const void* x_dev, uint64_t n1, double h, uint64_t r, uint64_t budget_bytes,
                       uint64_t* f_scratch_dev, int32_t* zs_out, uint64_t* nrec_out, uint64_t* bytes_out,
                       uint64_t* t0_out, uint64_t* nt_out, uint64_t* xread_ppm_out, void* stream);
int fs_build_zoned_rank(int32_t dtype, const void* x_dev, uint64_t n1, double h, uint64_t r, int32_t zs,
                        uint64_t nrec, uint64_t* f_scratch_dev, void* buf_dev, void* stream);

/*
 * Knot bytes (FS_SPARSE_KNOT_BYTES; no reference counterpart) for tables whose
 * rank directory fits in shared memory but whose X does not (the paper's
 * uniform-gap arrays at 65,535 knots): B[i] = floor(256 frac(p_i)), p_i =
 * RN(h RN(X_i - X0)) the product whose floor is knot i's bucket
 * (direct.py:194-197).  The search stages the directory and B; for a query
 * whose bucket holds knot t it compares the same byte of its own product with
 * B[t] -- RN is monotone, so a smaller byte means z < X[t] and a larger one z >
 * X[t] -- and reads X[t] (through L2) only on a tie.  Same answers as the rank
 * directory (batch.py:315-317).  Buffer: N+1 bytes padded to 16.  Async.
 * Set fs_plan.sparse to the buffer (fs_plan.rank to the directory),
 * sparse_format = FS_SPARSE_KNOT_BYTES, sparse_ndense = N+1, sparse_shift = 0.
 * Used when directory + bytes fit shared memory and directory + X do not.
 */
int fs_build_knot_bytes(int32_t dtype, const void* x_dev, uint64_t n1, double h, void* buf_dev, void* stream);

/*
 * Rank rows (FS_SPARSE_RANK_ROWS; no reference counterpart) for tables whose
 * rank directory is read through L2 (nothing fits in shared memory): row w =
 * {mask of the buckets 32w .. 32w+31 holding a knot, K[32w], the knot bytes
 * (fs_build_knot_bytes) of the row's first eight knots}, 16 B.  One gather
 * -- one 32-B sector, as for the 8-B directory word -- brings the word and
 * the bytes; X[t] is gathered only on a tie of the query's byte with its
 * knot's, or for a row's ninth and later knots.  Same answers as the rank
 * directory (batch.py:315-317).  rows_dev: ((R >> 5) + 1) * 16 bytes;
 * f_scratch_dev: n1 uint64; bytes_scratch_dev: n1 bytes padded to 16.  Async.
 * Set fs_plan.sparse to the rows, sparse_format = FS_SPARSE_RANK_ROWS
 * (sparse_shift = sparse_ndense = 0); used only when nothing is staged.
 */
int fs_build_rank_rows(int32_t dtype, const void* x_dev, uint64_t n1, double h, uint64_t r, uint64_t* f_scratch_dev,
                       void* bytes_scratch_dev, void* rows_dev, void* stream);

/*
 * Count words of the gap-1 table (FS_SPARSE_COUNT; a device layout of K, no
 * reference counterpart) for tables of few knots and many buckets (R >> N:
 * uniformly drawn knots, cfg2 and cfg5).  One stripe shift k for the whole
 * table; 8-B word g = {mask, base} covers buckets [g 2^(k+4), (g+1) 2^(k+4))
 * in 16 stripes of 2^k; bits 2b, 2b+1 of the mask hold the number of knots in
 * stripe b (saturated at 3), base = K[g 2^(k+4)] with bit 31 set when a
 * stripe of the word holds four or more knots.  For bucket j of the query z,
 * b = (j >> k) & 15 and m = mask below bit 2b: t = base + popc(m) + popc(m &
 * 0xAAAAAAAA) knots lie in earlier stripes, all below z (the bucket function
 * of direct.py:194-197 is monotone), knots of later stripes lie above z, and
 * the c = (mask >> 2b) & 3 knots of the query's own stripe are compared
 * directly: the answer of batch.py:315-317 is t - 1 + #{e : X[t+e] <= z}, one
 * predicated compare when c <= 1, a forward scan of X from t (from base for a
 * flagged word) when c >= 2.  Exact for every k; k only sets how many queries
 * take the scan.  When X is too large to stage, one byte per knot can be
 * (k <= 8): O[i] = f_i mod 2^k, knot i's bucket inside its stripe; a knot in a
 * lower bucket than the query's lies below z and one in a higher bucket above
 * it, so X is read (through L2) only for a knot in the query's own bucket.
 * Buffer: (R >> (k + 4)) + 1 words, then, if built with offsets, N+1 offset
 * bytes padded to 16 (fs_count_words_bytes(r, k, noff = N+1 or 0)).
 *   fs_plan_count_words: the finest k whose words fit budget_bytes in the
 *     given mode -- 1: beside all of X; 2: beside the knot offsets (k <= 8
 *     must fit); 0: alone, every knot read through L2 -- plus the share of
 *     buckets in knot-holding stripes (queries that read X or an offset) and
 *     in stripes of two or more knots or flagged words -- in mode 2 also the
 *     buckets that hold a lone knot themselves -- (queries that scan), in
 *     parts per million.  FS_TOO_LARGE if nothing fits or there are more
 *     knots than stripes.  SYNC.
 *   fs_build_count_words: fill the words (and the offsets) for that k.  Async.
 * Set fs_plan.sparse to the buffer, sparse_format = FS_SPARSE_COUNT,
 * sparse_shift = k, sparse_ndense = N+1 if built with offsets, else 0.  The
 * search stages X beside plain words when both fit.  f_scratch_dev: n1 uint64.
 */
uint64_t fs_count_words_bytes(uint64_t r, int32_t k, uint64_t noff);
int fs_plan_count_words(int32_t dtype, const void* x_dev, uint64_t n1, double h, uint64_t r, uint64_t budget_bytes,
                        int32_t mode, uint64_t* f_scratch_dev, int32_t* k_out, uint64_t* bytes_out,
                        uint64_t* xread_ppm_out, uint64_t* rare_ppm_out, void* stream);
int fs_build_count_words(int32_t dtype, const void* x_dev, uint64_t n1, double h, uint64_t r, int32_t k,
                         int32_t with_offsets, uint64_t* f_scratch_dev, void* buf_dev, void* stream);

/*
 * Hot window of a rank directory for shared-memory staging: among all
 * contiguous directory ranges whose words plus referenced knots fit in
 * `budget_bytes`, the one holding the most knots (ties: lowest start).
 * Queries distributed like the knots (the interpolation use of the paper)
 * then mostly hit shared memory.  dir_dev: (r >> 5) + 1 words; ws_dev:
 * fs_workspace_bytes().  Writes the window; *knots_in_window_out = knots
 * whose bucket lies inside.  SYNC.
 */
int fs_build_hot_window(int32_t dtype, const void* dir_dev, uint64_t r, uint64_t budget_bytes,
                        void* ws_dev, uint64_t* word0_out, uint64_t* words_out,
                        uint64_t* knot0_out, uint64_t* knots_out,
                        uint64_t* knots_in_window_out, void* stream);

/*
 * Cache-fused (idx, val) records.  Replaces direct.with_fused
 * (direct.py:255-263): rec[j] = {K[j], X[K[j]]}; 8 B records for f32,
 * 16 B {u32 idx, u32 pad = 0, f64 val} for f64.
 */
int fs_build_fused(int32_t dtype, const void* x_dev, uint64_t n1, const uint32_t* k_dev,
                   uint64_t r, void* rec_dev, void* stream);

/* Right padding to 2^pbits with X_N.  Replaces partition.pad_right_pow2
 * (partition.py:163-171). */
int fs_build_padded(int32_t dtype, const void* x_dev, uint64_t n1, int32_t pbits,
                    void* xpad_dev, void* stream);

/*
 * Subtree records for bitset2's global levels (a device layout of the same
 * padded array; no reference counterpart).  Below the `top_bits` levels the
 * kernel stages in shared memory, each remaining level pair (f64) / triple
 * (f32) becomes one 32-B record per node: the node's padded value and its
 * descendants' down to k levels, in BFS order.  One 256-bit gather then
 * resolves k levels with exactly the comparisons of binsearch.py:72-86; a
 * leftover single level reads xpad itself.  fs_b2_deep_bytes returns the
 * buffer size (0 = nothing to build) and the top_bits / k the search kernel
 * will use for this plan; fs_build_b2_deep fills it.
 */
uint64_t fs_b2_deep_bytes(int32_t dtype, int32_t pbits, int32_t* top_bits_out, int32_t* k_out);
int fs_build_b2_deep(int32_t dtype, const void* xpad_dev, int32_t pbits, int32_t top_bits, int32_t k,
                     void* deep_dev, void* stream);

/* Heap-order (Eytzinger) tree of depth L.  Replaces eytzinger.build_layout
 * (eytzinger.py:45-63). tree_dev holds 2^L - 1 elements. */
int fs_build_eytzinger(int32_t dtype, const void* x_dev, uint64_t n1, int32_t depth,
                       void* tree_dev, void* stream);

/* ---------------------------------------------------------------------------
 * Batch search (batch.py:399-441)
 * ------------------------------------------------------------------------ */

/*
 * Status workspace of the search calls: FS_SEARCH_WS_WORDS uint64 words of
 * device memory, ZERO-INITIALISED ONCE by its owner and then reusable by any
 * number of stream-ordered searches (not by concurrent ones).  After a
 * search, word 0 holds the first out-of-domain position or UINT64_MAX;
 * words 1-2 are the kernel's CTA ticket counter and running first-bad
 * fold, both left at 0 by every launch.
 */
#define FS_SEARCH_WS_WORDS 4
size_t fs_search_ws_words(void);

/*
 * Resolve m device-resident queries into device `out` (out_bytes = 4 for
 * int32, 8 for int64).  Replaces PreparedKernel.lanes + the domain check of
 * batch_search (batch.py:411-413): the first query with !(X0 <= z < XN)
 * (NaN included) is written to status word 0 by the kernel's last CTA (no
 * memset node).  `out` is unspecified where a query is out of domain.
 * ASYNC: exactly one kernel launch (m > 0).
 */
int fs_search_device(const fs_plan* plan, const void* z_dev, uint64_t m, void* out_dev,
                     int32_t out_bytes, unsigned long long* status_dev, void* stream);

/*
 * fs_search_device over queries base .. base + m - 1 of a larger batch (a
 * shard): status word 0 receives base + the first bad offset (UINT64_MAX when
 * clean) and word 3 the same value XOR 2^63 -- ordered as a SIGNED int64,
 * "clean" = INT64_MAX -- so shards agree on the batch's first bad position
 * with one MIN all-reduce of word 3 (dist.sharded_batch_search).  ASYNC:
 * exactly one kernel launch (m > 0).
 */
int fs_search_device_at(const fs_plan* plan, const void* z_dev, uint64_t m, void* out_dev,
                        int32_t out_bytes, unsigned long long* status_dev, uint64_t base, void* stream);

/*
 * End-to-end host-buffer search: the whole batch_search contract
 * (batch.py:399-441) on host arrays.  Copies z_host -> z_dev in chunks on
 * `copy_stream` (ordered after all work already queued on `stream`)
 * overlapped with the search kernel per chunk on `stream`;
 * then reads the first-bad word and, only if every query is in domain,
 * copies the results to out_host (nothing is written on error, as
 * batch.py:404 promises).  z_dev/out_dev are device scratch of m elements.
 * SYNC.  On FS_OUT_OF_DOMAIN *pos_out is the first offending position.
 *
 * flags & FS_HOST_OVERLAP: speculative write-back -- each chunk's results
 * are copied to out_host as soon as its kernel finishes, so the D2H stream
 * overlaps the H2D stream (PCIe is full duplex: ~2x end to end).  On
 * FS_OUT_OF_DOMAIN the error and position are the same, but out_host may
 * hold results for some chunks (opt-in relaxation of batch.py:404).
 */
#define FS_HOST_OVERLAP 1
/*
 * Pageable (not page-locked) host buffers of 4 MB or more are staged by the
 * library through a cached ring of pinned slots filled and drained by a pool
 * of host threads (parallel memcpy overlapped with the DMA); the contract is
 * the same.  flags & FS_HOST_NO_STAGING: hand pageable buffers to the
 * driver's bounce buffer instead.
 */
#define FS_HOST_NO_STAGING 2
/*
 * Default (atomic) mode over two or more chunks of page-locked (or small)
 * buffers: while the uploads run, "no query is bad" is established from both
 * ends -- the device's per-chunk verdicts cover a growing prefix, host
 * threads scan chunks from the end; once they meet, each chunk's results are
 * copied back as soon as its kernel finishes, overlapping the remaining
 * uploads (nothing is written if a query is bad -- the contract is
 * unchanged).  flags & FS_HOST_NO_PRECHECK:
 * wait for the device's first-bad word before any write-back instead.
 * FS_INCONSISTENT if the two checks disagree (z_host modified during the call).
 */
#define FS_HOST_NO_PRECHECK 4
int fs_search_host(const fs_plan* plan, const void* z_host, uint64_t m, void* out_host,
                   int32_t out_bytes, void* z_dev, void* out_dev,
                   unsigned long long* status_dev, uint64_t chunk_elems,
                   int64_t* pos_out, void* stream, void* copy_stream, int32_t flags);

/*
 * One host batch split into contiguous spans searched concurrently -- one
 * fs_search_host_gated call per span, e.g. one per GPU, each with its own
 * plan, scratch and streams on its device (the reference's thread spans,
 * batch.py:385-396 and 428-440, with devices for threads).  The calls share
 * a gate created for `parties` spans: a call writes results back only once
 * every span is known to be in domain, so the batch keeps batch.py:404's
 * "nothing written on OutOfDomain" as a whole.  A span with a bad query
 * returns FS_OUT_OF_DOMAIN with its span-local position (the caller
 * min-merges span offset + position); the others return FS_ABORTED and
 * write nothing.  A caller that cannot make its call must fs_gate_abort()
 * the gate, or the other calls wait for it.  FS_HOST_OVERLAP calls ignore
 * the gate.  Destroy the gate after every call has returned.
 */
typedef struct fs_gate fs_gate;
fs_gate* fs_gate_create(int32_t parties);
void fs_gate_abort(fs_gate* gate);
void fs_gate_destroy(fs_gate* gate);
int fs_search_host_gated(const fs_plan* plan, const void* z_host, uint64_t m, void* out_host,
                         int32_t out_bytes, void* z_dev, void* out_dev,
                         unsigned long long* status_dev, uint64_t chunk_elems,
                         int64_t* pos_out, void* stream, void* copy_stream, int32_t flags,
                         fs_gate* gate);

/* ---------------------------------------------------------------------------
 * Index persistence (bench/persist.py:1-112)
 * ------------------------------------------------------------------------ */

/*
 * zlib-compatible CRC-32 of `bytes` bytes of device memory: the K-payload
 * checksum of the FBSIDX1 index file (persist.py:63, 91), computed on the
 * GPU (chunked slice-by-4 + GF(2) combine tree) so a loaded payload is
 * verified where it lands.  ws_dev: fs_crc32_ws_bytes(bytes) bytes.  SYNC.
 */
size_t fs_crc32_ws_bytes(uint64_t bytes);
int fs_crc32(const void* data_dev, uint64_t bytes, void* ws_dev, uint32_t* crc_out, void* stream);

/* Placement the search kernel will use for this plan (FS_PLACE_* bit set),
 * plus the dynamic shared memory bytes per CTA it stages. */
int fs_plan_placement(const fs_plan* plan, int32_t* placement_out, uint64_t* smem_bytes_out);

/* Number of kernel launches fs_search_device issues for this plan and batch
 * (1, or 0 for an empty batch; -1 for an invalid plan). */
int fs_search_launches(const fs_plan* plan, uint64_t m);

/* Number of search kernels fs_search_host issues for the same arguments: one
 * per chunk -- 16 MB of queries per staging slot for pageable buffers, else
 * chunk_elems (default 64 MB of queries).  -1 for an invalid plan. */
int64_t fs_search_host_launches(const fs_plan* plan, const void* z_host, uint64_t m, const void* out_host,
                                int32_t out_bytes, uint64_t chunk_elems, int32_t flags);

#ifdef __cplusplus
}
#endif

#endif /* FSGPU_H */
