"""GPU tests of the count words of the gap-1 table (fs_plan_count_words /
fs_build_count_words + CountWordProbe): the planner's stripe shift and
statistics and the device buffer against a numpy construction from the
oracle's knot buckets (bit for bit), and every answer against the oracle
(batch.py:315-317 semantics) on tables of uniformly drawn knots (cfg2, cfg5),
stripes holding one, two, three and more knots (flagged words), every knot
and its neighbours, word / stripe edges, X staged and read through L2, f32
and f64 with int32 and int64 outputs, the last bucket R and out-of-domain
lanes."""

import ctypes

import numpy as np
import pytest

from oracle import fs_oracle as orc

pytestmark = pytest.mark.gpu

WORD_SHIFT, MAX_SHIFT, FLAG = 4, 27, 0x80000000


def _fs():
    import paper_1506_08620_b200 as fs

    return fs


def words_bytes(r, k):
    return 8 * ((r >> (k + WORD_SHIFT)) + 1)


def expected_plan(f, r, n1, es, budget):
    """(k, with_x, xread_ppm, rare_ppm) as fs_plan_count_words picks them, or None."""
    xb = (n1 * es + 127) // 128 * 128
    xb = xb if xb <= budget // 2 else 0
    if budget < xb + 128 + 8:
        return None
    tb = budget - xb - 128
    k = 0
    while k <= MAX_SHIFT and words_bytes(r, k) > tb:
        k += 1
    if k > MAX_SHIFT or n1 > (r >> k) + 1:
        return None
    stripe, cnt = np.unique(f >> k, return_counts=True)
    width = np.minimum(1 << k, r + 1 - (stripe << k))
    xread = int(width.sum())
    rare = int(width[cnt >= 2].sum())
    ws = k + WORD_SHIFT
    rare += int(np.minimum(1 << ws, r + 1 - ((stripe[cnt >= 4] >> WORD_SHIFT) << ws)).sum())
    rare = min(rare, r + 1)
    return k, int(xb != 0), xread * 10**6 // (r + 1), rare * 10**6 // (r + 1)


def _same_plan(got, exp):
    """k and the X rule exactly; the ppm statistics to one part (the library rounds in long double)."""
    return tuple(got[:2]) == tuple(exp[:2]) and all(abs(int(a) - int(b)) <= 1 for a, b in zip(got[2:], exp[2:]))


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


def with_count_words(fs, p, prep, budget, k=None):
    """Plan (or take ``k``) and build count words on prep's table and set them
    on its plan.  Returns (buffer, k, with_x, xread_ppm, rare_ppm) or None."""
    from paper_1506_08620_b200 import _device, _lib

    idx = prep.structure
    lib = _lib.load()
    dt = _lib.FS_F32 if p.precision == "single" else _lib.FS_F64
    n1 = len(p.values)
    f_dev = _device.empty(n1, np.uint64)
    kk, wx = ctypes.c_int32(-1), ctypes.c_int32(0)
    nbytes, xread, rare = (ctypes.c_uint64(0) for _ in range(3))
    x = p.device_values()
    if k is None:
        rc = lib.fs_plan_count_words(dt, x.data_ptr(), n1, float(idx.h), idx.r, budget, f_dev.data_ptr(),
                                     ctypes.byref(kk), ctypes.byref(nbytes), ctypes.byref(wx), ctypes.byref(xread),
                                     ctypes.byref(rare), _device.stream_ptr())
        if rc == _lib.FS_TOO_LARGE:
            return None
        _lib.check(rc)
        k = kk.value
        assert nbytes.value == lib.fs_count_words_bytes(idx.r, k) == words_bytes(idx.r, k)
    buf = _device.empty(words_bytes(idx.r, k), np.uint8)
    _lib.check(lib.fs_build_count_words(dt, x.data_ptr(), n1, float(idx.h), idx.r, k, f_dev.data_ptr(),
                                        buf.data_ptr(), _device.stream_ptr()))
    plan = prep.plan
    plan.records = None
    plan.rank = None  # placement must not prefer a rank directory that happens to fit
    plan.sparse = buf.data_ptr()
    plan.sparse_format = _lib.SPARSE_COUNT
    plan.sparse_shift = k
    plan.sparse_ndense = 0
    plan.hot_word0 = plan.hot_words = plan.hot_knot0 = plan.hot_knots = 0
    return buf, k, wx.value, xread.value, rare.value


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
    budget = batch._smem_budget() - 512
    k, with_x, xread, rare = expected_plan(f, idx.r, len(xs), xs.itemsize, budget)
    assert (prep.plan.sparse_shift, with_x) == (k, 1) and rare <= batch.COUNT_WORDS_MAX_RARE_PPM
    want_words, top, flagged = expected_words(f, idx.r, k)
    got = _buffer_of(prep, prep.plan.sparse).cpu().numpy().view(np.uint32).reshape(-1, 2)
    assert np.array_equal(got, want_words)
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


def test_count_words_rule_keeps_records_without_x(cuda):
    """cfg5 N+1 = 32769: X (256 KB) cannot be staged and 9% of the buckets lie
    in knot-holding stripes, so the planner keeps the group records; forced,
    the count words (every knot read through L2) give the same answers."""
    fs = _fs()
    from paper_1506_08620_b200 import batch, workloads

    p = workloads.knots("cfg5", n1=32769)
    prep = fs.prepare("direct", p)
    assert prep.placement()["sparse_format"].startswith("records")
    xs = p.values
    idx = prep.structure
    f = orc.knot_buckets(xs, idx.h).astype(np.int64)
    got = with_count_words(fs, p, prep, batch._smem_budget() - 512)
    assert got is not None
    buf, k, with_x, xread, rare = got
    assert _same_plan((k, with_x, xread, rare), expected_plan(f, idx.r, len(xs), xs.itemsize, batch._smem_budget() - 512))
    assert with_x == 0 and xread > batch.COUNT_WORDS_MAX_L2_XREAD_PPM
    pl = prep.placement()
    assert pl["sparse_format"] == "count-words" and not pl["smem_x"], pl
    want_words, top, _ = expected_words(f, idx.r, k)
    assert np.array_equal(buf.cpu().numpy().view(np.uint32).reshape(-1, 2), want_words) and top >= 2
    z = np.concatenate([workloads.queries_host("cfg5", p, 300_000, seed=5), _all_knots(xs),
                        _edge_queries(xs, idx.h, idx.r, k)]).astype(xs.dtype)
    z = z[(z >= xs[0]) & (z < xs[-1])]
    assert np.array_equal(fs.run_batch(prep, z), orc.rank_oracle(xs, z))


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
        buf, *_ = with_count_words(fs, p, prep, 0, k=k)
        pl = prep.placement()
        assert pl["sparse_format"] == "count-words" and pl["smem_x"], (k, pl)
        want_words, top, flagged = expected_words(f, idx.r, k)
        assert np.array_equal(buf.cpu().numpy().view(np.uint32).reshape(-1, 2), want_words), k
        seen_top, seen_flagged = max(seen_top, top), max(seen_flagged, flagged)
        z = np.concatenate([base, _edge_queries(xs, idx.h, idx.r, k)]).astype(dtype)
        z = z[(z >= xs[0]) & (z < xs[-1])]
        want = orc.rank_oracle(xs, z)
        assert np.array_equal(fs.run_batch(prep, z), want), k
        out32 = np.empty(len(z), dtype=np.int32)
        fs.batch_search(fs.LaneConfig(1, "direct", prep), z, out32)
        assert np.array_equal(out32, want), k
    assert seen_top >= 4 and seen_flagged > 0  # coarse stripes saturate: the flagged-word scan ran


def test_count_words_planner_budgets(cuda):
    """fs_plan_count_words over budgets: k, the X rule (all of X when it takes
    at most half the budget, else none) and both statistics equal the numpy
    plan; FS_TOO_LARGE when nothing fits; answers equal the oracle either way."""
    fs = _fs()
    xs = _clumped(4000, np.float64, seed=3)
    p = fs.validate_partition(xs, "double")
    xs = p.values
    prep = fs.prepare("direct", p)
    idx = prep.structure
    f = orc.knot_buckets(xs, idx.h).astype(np.int64)
    z = np.concatenate([_all_knots(xs), orc.random_queries(xs, 50_000, seed=1)])
    want = orc.rank_oracle(xs, z)
    staged = set()
    for budget in (100, 3000, 20_000, 50_000, 70_000, 150_000, 225_000):
        exp = expected_plan(f, idx.r, len(xs), xs.itemsize, budget)
        got = with_count_words(fs, p, prep, budget)
        if exp is None:
            assert got is None, budget
            continue
        assert got is not None and _same_plan(got[1:], exp), (budget, got[1:], exp)
        staged.add(exp[1])
        assert np.array_equal(fs.run_batch(prep, z), want), budget
    assert staged == {0, 1}


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
    for k in (2, 9):
        with_count_words(fs, p, prep, 0, k=k)
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
    k, wx = ctypes.c_int32(-1), ctypes.c_int32(0)
    outs = [ctypes.c_uint64(0) for _ in range(3)]
    st = _device.stream_ptr()

    def plan(dt, xp, budget, fp=f_dev.data_ptr()):
        return lib.fs_plan_count_words(dt, xp, n1, float(idx.h), idx.r, budget, fp, ctypes.byref(k),
                                       ctypes.byref(outs[0]), ctypes.byref(wx), ctypes.byref(outs[1]),
                                       ctypes.byref(outs[2]), st)

    assert plan(_lib.FS_F32, None, 100_000) == _lib.FS_INVALID_ARG
    assert plan(_lib.FS_F32, x.data_ptr(), 100_000, None) == _lib.FS_INVALID_ARG
    assert plan(7, x.data_ptr(), 100_000) == _lib.FS_INVALID_ARG
    assert plan(_lib.FS_F32, x.data_ptr(), 100) == _lib.FS_TOO_LARGE
    assert plan(_lib.FS_F32, x.data_ptr(), 100_000) == _lib.FS_OK
    assert lib.fs_count_words_bytes(idx.r, -1) == 0 and lib.fs_count_words_bytes(idx.r, MAX_SHIFT + 1) == 0
    assert lib.fs_count_words_bytes(1 << 32, 3) == 0
    buf = _device.empty(words_bytes(idx.r, k.value), np.uint8)
    for bad_k in (-1, MAX_SHIFT + 1):
        assert lib.fs_build_count_words(_lib.FS_F32, x.data_ptr(), n1, float(idx.h), idx.r, bad_k, f_dev.data_ptr(),
                                        buf.data_ptr(), st) == _lib.FS_INVALID_ARG
    assert lib.fs_build_count_words(_lib.FS_F32, x.data_ptr(), n1, float(idx.h), idx.r, k.value, f_dev.data_ptr(),
                                    None, st) == _lib.FS_INVALID_ARG
    with_count_words(fs, p, prep, 100_000)
    z = orc.random_queries(p.values, 1000, seed=1)
    assert np.array_equal(fs.run_batch(prep, z), orc.rank_oracle(p.values, z))
    for bad_k in (-1, MAX_SHIFT + 1):
        prep.plan.sparse_shift = bad_k
        with pytest.raises(ValueError):
            fs.run_batch(prep, z)
