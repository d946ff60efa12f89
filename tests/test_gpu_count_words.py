"""GPU tests of the count words of the gap-1 table (fs_plan_count_words /
fs_build_count_words + CountWordProbe): the planner's stripe shift and
statistics and the device buffer against a numpy construction from the
oracle's knot buckets (bit for bit), and every answer against the oracle
(batch.py:315-317 semantics) on tables of uniformly drawn knots (cfg2, cfg5),
stripes holding one, two, three and more knots (flagged words), every knot
and its neighbours, word / stripe edges, X staged, read through L2 and replaced by staged knot offsets, f32
and f64 with int32 and int64 outputs, the last bucket R and out-of-domain
lanes."""

import ctypes

import numpy as np
import pytest

from oracle import fs_oracle as orc

pytestmark = pytest.mark.gpu

WORD_SHIFT, MAX_SHIFT, MAX_OFFSET_SHIFT, FLAG = 4, 27, 8, 0x80000000


def _fs():
    import paper_1506_08620_b200 as fs

    return fs


def words_bytes(r, k, noff=0):
    return 8 * ((r >> (k + WORD_SHIFT)) + 1) + (noff + 15) // 16 * 16


def expected_plan(f, r, n1, es, budget, mode):
    """(k, xread_ppm, rare_ppm) as fs_plan_count_words picks them for ``mode`` (1: beside
    all of X; 2: beside a byte per knot, k <= 8; 0: words alone), or None."""
    beside = {0: 0, 1: (n1 * es + 127) // 128 * 128, 2: (n1 + 15) // 16 * 16}[mode]
    if budget < beside + 128 + 8:
        return None
    k = 0
    while k <= MAX_SHIFT and words_bytes(r, k) > budget - beside - 128:
        k += 1
    if k > MAX_SHIFT or (mode == 2 and k > MAX_OFFSET_SHIFT) or n1 > (r >> k) + 1:
        return None
    stripe, cnt = np.unique(f >> k, return_counts=True)
    width = np.minimum(1 << k, r + 1 - (stripe << k))
    xread = int(width.sum())
    rare = int(width[cnt >= 2].sum())
    if mode == 2:
        rare += int((cnt == 1).sum())  # a lone knot's own bucket: X decides it on the scan path
    ws = k + WORD_SHIFT
    rare += int(np.minimum(1 << ws, r + 1 - ((stripe[cnt >= 4] >> WORD_SHIFT) << ws)).sum())
    rare = min(rare, r + 1)
    return k, xread * 10**6 // (r + 1), rare * 10**6 // (r + 1)


def _same_plan(got, exp):
    """k exactly; the ppm statistics to one part (the library rounds in long double)."""
    return got[0] == exp[0] and all(abs(int(a) - int(b)) <= 1 for a, b in zip(got[1:], exp[1:]))


def expected_words(f, r, k):
    """uint32[nwords, 2] = {2-bit counts saturated at 3, base | flag}, the largest
    stripe count met and the number of flagged words."""
    n = (r >> (k + WORD_SHIFT)) + 1
    s = k + WORD_SHIFT
    j0 = np.arange(n, dtype=np.int64) << s
    lo = np.searchsorted(f, j0, side="left")
    hi = np.searchsorted(f, j0 + (1 << s), side="left")
    out = np.zeros((n, 2), dtype=np.uint64)
    out[:, 1] = lo
    top = flagged = 0
    for g in np.flatnonzero(hi > lo):
        c = np.bincount((f[lo[g]:hi[g]] - j0[g]) >> k, minlength=16)
        top = max(top, int(c.max()))
        out[g, 0] = sum(int(min(v, 3)) << (2 * b) for b, v in enumerate(c))
        if c.max() >= 4:
            out[g, 1] |= FLAG
            flagged += 1
    return out.astype(np.uint32), top, flagged


def with_count_words(fs, p, prep, budget, k=None, offsets=False, mode=None):
    """Plan for ``mode`` (or take ``k`` and ``offsets``) and build count words on
    prep's table and set them on its plan.  Returns (buffer, k, xread_ppm,
    rare_ppm) or None."""
    from paper_1506_08620_b200 import _device, _lib

    idx = prep.structure
    lib = _lib.load()
    dt = _lib.FS_F32 if p.precision == "single" else _lib.FS_F64
    n1 = len(p.values)
    f_dev = _device.empty(n1, np.uint64)
    kk = ctypes.c_int32(-1)
    nbytes, xread, rare = (ctypes.c_uint64(0) for _ in range(3))
    x = p.device_values()
    if k is None:
        rc = lib.fs_plan_count_words(dt, x.data_ptr(), n1, float(idx.h), idx.r, budget, mode, f_dev.data_ptr(),
                                     ctypes.byref(kk), ctypes.byref(nbytes), ctypes.byref(xread), ctypes.byref(rare),
                                     _device.stream_ptr())
        if rc == _lib.FS_TOO_LARGE:
            return None
        _lib.check(rc)
        k, offsets = kk.value, mode == 2
        assert nbytes.value == lib.fs_count_words_bytes(idx.r, k, n1 if offsets else 0)
        assert nbytes.value == words_bytes(idx.r, k, n1 if offsets else 0)
    buf = _device.empty(words_bytes(idx.r, k, n1 if offsets else 0), np.uint8)
    _lib.check(lib.fs_build_count_words(dt, x.data_ptr(), n1, float(idx.h), idx.r, k, int(offsets), f_dev.data_ptr(),
                                        buf.data_ptr(), _device.stream_ptr()))
    plan = prep.plan
    plan.records = None
    plan.rank = None  # placement must not prefer a rank directory that happens to fit
    plan.sparse = buf.data_ptr()
    plan.sparse_format = _lib.SPARSE_COUNT
    plan.sparse_shift = k
    plan.sparse_ndense = n1 if offsets else 0
    plan.hot_word0 = plan.hot_words = plan.hot_knot0 = plan.hot_knots = 0
    return buf, k, xread.value, rare.value


def _check_buffer(buf, f, r, k, offsets):
    """Words (and offset bytes) bit for bit; returns (largest stripe count, flagged words)."""
    want_words, top, flagged = expected_words(f, r, k)
    got = buf.cpu().numpy()
    assert np.array_equal(got[: want_words.nbytes].view(np.uint32).reshape(-1, 2), want_words), k
    if offsets:
        assert np.array_equal(got[want_words.nbytes: want_words.nbytes + len(f)], (f & ((1 << k) - 1)).astype(np.uint8)), k
        assert len(got) == want_words.nbytes + (len(f) + 15) // 16 * 16 and not got[want_words.nbytes + len(f):].any()
    else:
        assert len(got) == want_words.nbytes
    return top, flagged


def _buffer_of(prep, ptr):
    return next(b for b in prep.buffers if b.data_ptr() == ptr)


def _all_knots(xs):
    """Every knot and the values one ulp either side: each compare of a stripe's
    knots decided on both sides."""
    z = np.concatenate([xs, np.nextafter(xs, -np.inf), np.nextafter(xs, np.inf)]).astype(xs.dtype)
    return z[(z >= xs[0]) & (z < xs[-1])]


def _edge_queries(xs, h, r, k):
    """Queries at the edges of the first, last and some random words and stripes."""
    t = xs.dtype.type
    rng = np.random.default_rng(k)
    s = k + WORD_SHIFT
    nw = (r >> s) + 1
    words = np.unique(np.concatenate([[0, 1, nw - 1, max(nw - 2, 0)], rng.integers(0, nw, 200)]))
    buckets = np.concatenate([(words << s) + (b << k) + d for b in (0, 1, 15) for d in (-1, 0, 1)] + [[r - 1, r]])
    buckets = buckets[(buckets >= 0) & (buckets <= r)]
    v = (xs[0] + buckets.astype(xs.dtype) / t(h)).astype(xs.dtype)
    z = np.concatenate([np.nextafter(v, t(-np.inf)), v, np.nextafter(v, t(np.inf))]).astype(xs.dtype)
    return z[(z >= xs[0]) & (z < xs[-1])]


@pytest.mark.parametrize("label", ["cfg2_s0", "cfg2_s1", "cfg2_s2"])
def test_count_words_chosen_for_cfg2(cuda, label):
    """cfg2 (f64, 10,001 uniform knots; R = 25 M / 399 M / 202 M): prepare()
    stages count words beside all of X; plan and buffer bit-exact against
    numpy; answers equal the oracle at every knot and its neighbours (stripes
    of two knots included), word and stripe edges, bucket edges and the
    config's own stream with its exact-knot queries; int32 and int64 outputs."""
    fs = _fs()
    from paper_1506_08620_b200 import batch, workloads

    p = workloads.knots("cfg2", seed=int(label[-1]))
    prep = fs.prepare("direct", p)
    pl = prep.placement()
    assert pl["smem_sparse"] and pl["sparse_format"] == "count-words" and pl["smem_x"], pl
    xs = p.values
    idx = prep.structure
    f = orc.knot_buckets(xs, idx.h).astype(np.int64)
    budget = min(batch._smem_budget() - 512, batch.COUNT_WORDS_BUDGET_BYTES)
    k, xread, rare = expected_plan(f, idx.r, len(xs), xs.itemsize, budget, 1)
    assert (prep.plan.sparse_shift, prep.plan.sparse_ndense) == (k, 0)
    assert rare <= batch.COUNT_WORDS_MAX_RARE_PPM and xread <= batch.COUNT_WORDS_MAX_XREAD_PPM
    assert pl["smem_bytes"] <= 196 * 1024  # under the carve-out step that leaves L1 only 28 KB
    top, flagged = _check_buffer(_buffer_of(prep, prep.plan.sparse), f, idx.r, k, False)
    assert top >= 2  # uniform draws: some stripes hold two knots (seed 2: one holds four, a flagged word)
    z = np.concatenate([
        workloads.queries_host("cfg2", p, 300_000, seed=5), _all_knots(xs), _edge_queries(xs, idx.h, idx.r, k),
        orc.boundary_probes(xs), orc.bucket_edge_probes(xs, idx.h, idx.r, 100_000, seed=4),
    ]).astype(xs.dtype)
    z = z[(z >= xs[0]) & (z < xs[-1])]
    want = orc.rank_oracle(xs, z)
    assert np.array_equal(fs.run_batch(prep, z), want)
    out32 = np.empty(len(z), dtype=np.int32)
    fs.batch_search(fs.LaneConfig(1, "direct", prep), z, out32)
    assert np.array_equal(out32, want)


@pytest.mark.parametrize("size", [32769, 65537])
def test_count_words_with_offsets_for_cfg5(cuda, size):
    """cfg5 N+1 = 32769 (and 65537, where no group record layout fits and the
    count words replace the two-level table): X cannot be staged, a byte per knot can:
    prepare() stages count words (k = 5) and the knots' in-stripe buckets, and
    reads X through L2 only for a knot in the query's own bucket.  Plan, words
    and offsets bit-exact; answers equal the oracle at every knot and its
    neighbours, layout and bucket edges and uniform queries.  With the
    offsets switched off the planner keeps the group records (9% of the
    buckets lie in knot-holding stripes: too many L2 reads); forced, the
    plain words give the same answers."""
    fs = _fs()
    from paper_1506_08620_b200 import batch, workloads

    p = workloads.knots("cfg5", n1=size)
    xs = p.values
    prep = fs.prepare("direct", p)
    pl = prep.placement()
    assert pl["smem_sparse"] and pl["sparse_format"] == "count-words" and not pl["smem_x"], pl
    idx = prep.structure
    f = orc.knot_buckets(xs, idx.h).astype(np.int64)
    # 32769: tried before the 16-B group records, within the carve-out budget; 65537: the late
    # stage (nothing but the two-level table left), with all of shared memory
    budget = batch._smem_budget() - 512
    if size == 32769:
        budget = min(budget, batch.COUNT_WORDS_BUDGET_BYTES)
    assert expected_plan(f, idx.r, len(xs), xs.itemsize, budget, 1) is None  # X does not fit beside any words
    k, xread, rare = expected_plan(f, idx.r, len(xs), xs.itemsize, budget, 2)
    assert (prep.plan.sparse_shift, prep.plan.sparse_ndense) == (k, len(xs)) and k <= MAX_OFFSET_SHIFT
    top, _ = _check_buffer(_buffer_of(prep, prep.plan.sparse), f, idx.r, k, True)
    assert top >= 2
    z = np.concatenate([workloads.queries_host("cfg5", p, 300_000, seed=5), _all_knots(xs),
                        _edge_queries(xs, idx.h, idx.r, k), orc.boundary_probes(xs),
                        orc.bucket_edge_probes(xs, idx.h, idx.r, 100_000, seed=4)]).astype(xs.dtype)
    z = z[(z >= xs[0]) & (z < xs[-1])]
    want = orc.rank_oracle(xs, z)
    assert np.array_equal(fs.run_batch(prep, z), want)
    out32 = np.empty(len(z), dtype=np.int32)
    fs.batch_search(fs.LaneConfig(1, "direct", prep), z, out32)
    assert np.array_equal(out32, want)
    saved = batch.COUNT_WORDS_OFFSETS
    try:
        batch.COUNT_WORDS_OFFSETS = False
        prep = fs.prepare("direct", p)
    finally:
        batch.COUNT_WORDS_OFFSETS = saved
    assert prep.placement()["sparse_format"] != "count-words"  # group records (32769) / the two-level table
    buf, k0, *_ = with_count_words(fs, p, prep, 0, k=5)
    pl = prep.placement()
    assert pl["sparse_format"] == "count-words" and not pl["smem_x"] and prep.plan.sparse_ndense == 0, pl
    _check_buffer(buf, f, idx.r, 5, False)
    assert np.array_equal(fs.run_batch(prep, z), want)


def _clumped(n, dtype, seed, clump=(0, 3)):
    """Knots in clumps of neighbours a few buckets apart between wide gaps:
    stripes of every count; clumps of five and more give flagged words."""
    rng = np.random.default_rng(seed)
    x = [0.0]
    while len(x) < n:
        x.append(x[-1] + rng.uniform(50.0, 400.0))
        for _ in range(int(rng.integers(clump[0], clump[1]))):
            x.append(x[-1] + rng.uniform(1.0, 3.0))
    return np.array(x[:n], dtype=np.float64).astype(dtype)


@pytest.mark.parametrize("dtype", [np.float32, np.float64])
@pytest.mark.parametrize("clump", [(0, 3), (2, 9)])
def test_count_words_every_shift(cuda, dtype, clump):
    """Clumped knots at every stripe shift from one bucket to a handful of
    words for the table: counts of 1, 2, 3 and saturated stripes (flagged
    words, scanned from their base), buffer bit for bit, X staged; answers
    equal the oracle at every knot, its neighbours and the layout's edges.
    Correctness must not depend on k."""
    fs = _fs()
    xs = _clumped(5000, dtype, seed=7, clump=clump)
    p = fs.validate_partition(xs, "single" if dtype == np.float32 else "double")
    xs = p.values
    prep = fs.prepare("direct", p)
    idx = prep.structure
    f = orc.knot_buckets(xs, idx.h).astype(np.int64)
    base = np.concatenate([_all_knots(xs), orc.random_queries(xs, 100_000, seed=2), orc.boundary_probes(xs)])
    seen_top = seen_flagged = 0
    kmax = max(0, int(idx.r).bit_length() - WORD_SHIFT - 2)
    for k in range(0, kmax + 1):
        if words_bytes(idx.r, k) + len(xs) * xs.itemsize + 256 > 220_000:
            continue
        z = np.concatenate([base, _edge_queries(xs, idx.h, idx.r, k)]).astype(dtype)
        z = z[(z >= xs[0]) & (z < xs[-1])]
        want = orc.rank_oracle(xs, z)
        for offsets in (False, True) if k <= MAX_OFFSET_SHIFT else (False,):
            buf, *_ = with_count_words(fs, p, prep, 0, k=k, offsets=offsets)
            pl = prep.placement()
            # plain words sit beside X; words built with offsets are the layout without it
            assert pl["sparse_format"] == "count-words" and pl["smem_x"] == (not offsets), (k, offsets, pl)
            top, flagged = _check_buffer(buf, f, idx.r, k, offsets)
            seen_top, seen_flagged = max(seen_top, top), max(seen_flagged, flagged)
            assert np.array_equal(fs.run_batch(prep, z), want), (k, offsets)
            out32 = np.empty(len(z), dtype=np.int32)
            fs.batch_search(fs.LaneConfig(1, "direct", prep), z, out32)
            assert np.array_equal(out32, want), (k, offsets)
    assert seen_top >= 4 and seen_flagged > 0  # coarse stripes saturate: the flagged-word scan ran


def test_count_words_planner_budgets(cuda):
    """fs_plan_count_words over budgets and modes (words alone, beside all of
    X, beside the knot offsets with k <= 8): k and both statistics equal the
    numpy plan; FS_TOO_LARGE when nothing fits; answers equal the oracle either way."""
    fs = _fs()
    xs = _clumped(4000, np.float64, seed=3)
    p = fs.validate_partition(xs, "double")
    xs = p.values
    prep = fs.prepare("direct", p)
    idx = prep.structure
    f = orc.knot_buckets(xs, idx.h).astype(np.int64)
    z = np.concatenate([_all_knots(xs), orc.random_queries(xs, 50_000, seed=1)])
    want = orc.rank_oracle(xs, z)
    fitted = set()
    for budget in (100, 3000, 6000, 20_000, 50_000, 70_000, 150_000, 225_000):
        for mode in (0, 1, 2):
            exp = expected_plan(f, idx.r, len(xs), xs.itemsize, budget, mode)
            got = with_count_words(fs, p, prep, budget, mode=mode)
            if exp is None:
                assert got is None, (budget, mode)
                continue
            assert got is not None and _same_plan(got[1:], exp), (budget, mode, got[1:], exp)
            fitted.add(mode)
            pl = prep.placement()
            assert pl["sparse_format"] == "count-words" and pl["smem_x"] == (mode != 2), (budget, mode, pl)
            assert np.array_equal(fs.run_batch(prep, z), want), (budget, mode)
    assert fitted == {0, 1, 2}  # words alone (placement adds X when it fits), beside X, beside the knot offsets


def test_count_words_out_of_domain_and_last_bucket(cuda):
    """Out-of-domain lanes (NaN, +-inf, below X0, at and above XN) beside valid
    ones report the first bad position and fault nothing -- also in the scan
    path of a stripe holding the last knots; the last bucket R resolves."""
    fs = _fs()
    xs = _clumped(3000, np.float64, seed=11, clump=(2, 6))
    p = fs.validate_partition(xs, "double")
    xs = p.values
    prep = fs.prepare("direct", p)
    idx = prep.structure
    for k, offsets in ((2, False), (9, False), (3, True), (8, True)):
        with_count_words(fs, p, prep, 0, k=k, offsets=offsets)
        assert prep.placement()["sparse_format"] == "count-words"
        tail = np.concatenate([xs[-8:-1], np.nextafter(xs[-8:], -np.inf), orc.random_queries(xs, 5000, seed=3)])
        tail = tail[(tail >= xs[0]) & (tail < xs[-1])]
        assert np.array_equal(fs.run_batch(prep, tail), orc.rank_oracle(xs, tail))
        for bad in (np.nan, np.inf, -np.inf, xs[0] - 1.0, xs[-1], xs[-1] * 2):
            z = orc.random_queries(xs, 10_000, seed=5)
            z[4321] = bad
            z[7777] = bad
            with pytest.raises(fs.OutOfDomain) as ei:
                fs.run_batch(prep, z)
            assert ei.value.position == 4321


def test_count_words_switch(cuda):
    """The planner knobs: count words excluded (or their thresholds at 0) give
    the group records back, with the same answers."""
    fs = _fs()
    from paper_1506_08620_b200 import batch, workloads

    p = workloads.knots("cfg2", seed=1)
    z = np.concatenate([workloads.queries_host("cfg2", p, 200_000, seed=9), _all_knots(p.values)])
    want = orc.rank_oracle(p.values, z)
    saved = batch.SPARSE_FORMATS, batch.COUNT_WORDS_MAX_RARE_PPM
    try:
        batch.SPARSE_FORMATS = tuple(n for n in saved[0] if n != "count-words")
        prep = fs.prepare("direct", p)
        assert prep.placement()["sparse_format"].startswith("records")
        assert np.array_equal(fs.run_batch(prep, z), want)
        batch.SPARSE_FORMATS = saved[0]
        batch.COUNT_WORDS_MAX_RARE_PPM = 0
        assert fs.prepare("direct", p).placement()["sparse_format"].startswith("records")
        batch.COUNT_WORDS_MAX_RARE_PPM = saved[1]
        prep = fs.prepare("direct", p)
        assert prep.placement()["sparse_format"] == "count-words"
        assert np.array_equal(fs.run_batch(prep, z), want)
    finally:
        batch.SPARSE_FORMATS, batch.COUNT_WORDS_MAX_RARE_PPM = saved


def test_count_words_abi_validation(cuda):
    """C-ABI argument checks: null pointers, bad dtype, stripe shifts out of
    range, budgets nothing fits, and validate_plan on a count-word plan with an
    out-of-range shift."""
    fs = _fs()
    from paper_1506_08620_b200 import _device, _lib

    xs = _clumped(3000, np.float32, seed=1)
    p = fs.validate_partition(xs, "single")
    prep = fs.prepare("direct", p)
    idx = prep.structure
    lib = _lib.load()
    n1 = len(p.values)
    x = p.device_values()
    f_dev = _device.empty(n1, np.uint64)
    k = ctypes.c_int32(-1)
    outs = [ctypes.c_uint64(0) for _ in range(3)]
    st = _device.stream_ptr()

    def plan(dt, xp, budget, fp=f_dev.data_ptr(), mode=1):
        return lib.fs_plan_count_words(dt, xp, n1, float(idx.h), idx.r, budget, mode, fp, ctypes.byref(k),
                                       ctypes.byref(outs[0]), ctypes.byref(outs[1]), ctypes.byref(outs[2]), st)

    assert plan(_lib.FS_F32, None, 100_000) == _lib.FS_INVALID_ARG
    assert plan(_lib.FS_F32, x.data_ptr(), 100_000, None) == _lib.FS_INVALID_ARG
    assert plan(7, x.data_ptr(), 100_000) == _lib.FS_INVALID_ARG
    assert plan(_lib.FS_F32, x.data_ptr(), 100_000, mode=3) == _lib.FS_INVALID_ARG
    assert plan(_lib.FS_F32, x.data_ptr(), 100) == _lib.FS_TOO_LARGE
    assert plan(_lib.FS_F32, x.data_ptr(), 4000, mode=2) == _lib.FS_TOO_LARGE  # offsets need k <= 8
    assert plan(_lib.FS_F32, x.data_ptr(), 100_000) == _lib.FS_OK
    assert lib.fs_count_words_bytes(idx.r, -1, 0) == 0 and lib.fs_count_words_bytes(idx.r, MAX_SHIFT + 1, 0) == 0
    assert lib.fs_count_words_bytes(1 << 32, 3, 0) == 0 and lib.fs_count_words_bytes(idx.r, MAX_OFFSET_SHIFT + 1, n1) == 0
    buf = _device.empty(words_bytes(idx.r, k.value), np.uint8)
    for bad_k, off in ((-1, 0), (MAX_SHIFT + 1, 0), (MAX_OFFSET_SHIFT + 1, 1)):
        assert lib.fs_build_count_words(_lib.FS_F32, x.data_ptr(), n1, float(idx.h), idx.r, bad_k, off,
                                        f_dev.data_ptr(), buf.data_ptr(), st) == _lib.FS_INVALID_ARG
    assert lib.fs_build_count_words(_lib.FS_F32, x.data_ptr(), n1, float(idx.h), idx.r, k.value, 0, f_dev.data_ptr(),
                                    None, st) == _lib.FS_INVALID_ARG
    with_count_words(fs, p, prep, 100_000, mode=1)
    z = orc.random_queries(p.values, 1000, seed=1)
    assert np.array_equal(fs.run_batch(prep, z), orc.rank_oracle(p.values, z))
    for bad_k in (-1, MAX_SHIFT + 1):
        prep.plan.sparse_shift = bad_k
        with pytest.raises(ValueError):
            fs.run_batch(prep, z)
    prep.plan.sparse_shift, prep.plan.sparse_ndense = 3, n1 - 1  # offsets come for every knot or none
    with pytest.raises(ValueError):
        fs.run_batch(prep, z)
