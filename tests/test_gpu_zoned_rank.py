"""GPU tests of the striped rank words of the gap-1 table (fs_plan_zoned_rank /
fs_build_zoned_rank + ZonedProbe<STRIPED>): the planner's stripe shifts and the
device buffer against a numpy construction from the oracle's knot buckets (bit
for bit), and every answer against the oracle (batch.py:315-317 semantics) at
zone, word and stripe edges, exact knots and their neighbours, both sides of
the staged X window, the last bucket R and out-of-domain lanes."""

import ctypes

import numpy as np
import pytest

from oracle import fs_oracle as orc

pytestmark = pytest.mark.gpu

RANK_SHIFT, RANK_FLAG, MAX_STRIPE, MIN_ZONE_SHIFT = 5, 16, 10, 11


def _fs():
    import paper_1506_08620_b200 as fs

    return fs


def expected_plan(f, r, zs, table_budget):
    """Stripe shift per zone as zone_plan_rank picks it: the largest k whose
    stripes hold at most one knot, then refined (k - 1) zone by zone -- most
    buckets inside knot-holding stripes first -- while the words fit."""
    nz = (r >> zs) + 1
    kcap = min(MAX_STRIPE, zs - RANK_SHIFT)
    zb = [min(1 << zs, r + 1 - (z << zs)) for z in range(nz)]
    zone = f >> zs
    cnt = np.bincount(zone, minlength=nz).tolist()
    k = [kcap] * nz
    same = zone[1:] == zone[:-1]
    hb = np.floor(np.log2((f[1:] ^ f[:-1]).astype(np.float64))).astype(np.int64)  # buckets < 2^32: exact
    for z, b in zip(zone[:-1][same].tolist(), hb[same].tolist()):
        k[z] = min(k[z], b)

    def words(z, kz):
        return (zb[z] + (1 << (kz + RANK_SHIFT)) - 1) >> (kz + RANK_SHIFT)

    head = 4 * ((nz + 3) // 4 * 4)
    total = sum(words(z, k[z]) for z in range(nz))
    if head + 8 * total > table_budget:
        return None
    while True:
        order = sorted((z for z in range(nz) if k[z] > 0 and cnt[z] > 0), key=lambda z: -(cnt[z] << k[z]))
        for z in order:
            t2 = total - words(z, k[z]) + words(z, k[z] - 1)
            if head + 8 * t2 <= table_budget:
                k[z] -= 1
                total = t2
                break
        else:
            break
    xread = sum(min(cnt[z] << k[z], zb[z]) for z in range(nz))
    return k, total, xread


def expected_buffer(f, r, zs, k):
    """(desc uint32[nz], words uint32[nrec, 2] = {mask, base}) for stripe shifts k."""
    nz = (r >> zs) + 1
    desc, recs = [], []
    nrec = 0
    for z in range(nz):
        zlo = z << zs
        zb = min(1 << zs, r + 1 - zlo)
        s = k[z] + RANK_SHIFT
        n = (zb + (1 << s) - 1) >> s
        rel = nrec - (z << (zs - s))
        desc.append(((rel << 5) & 0xFFFFFFFF) | RANK_FLAG | k[z])
        j0 = zlo + (np.arange(n, dtype=np.int64) << s)
        lo = np.searchsorted(f, j0, side="left")
        hi = np.searchsorted(f, j0 + (1 << s), side="left")
        for g in range(n):
            bits = ((f[lo[g]:hi[g]] - j0[g]) >> k[z]).tolist()
            assert len(set(bits)) == len(bits), "two knots in one stripe"
            recs.append([sum(1 << b for b in bits), int(lo[g])])
        nrec += n
    return np.array(desc, dtype=np.uint32), np.array(recs, dtype=np.uint64).astype(np.uint32)


def _buffer_of(prep, ptr):
    return next(b for b in prep.buffers if b.data_ptr() == ptr)


def _edge_queries(xs, h, buckets):
    t = xs.dtype.type
    out = []
    for j in buckets:
        for jj in (j - 1, j, j + 1):
            if jj < 0:
                continue
            v = t(xs[0] + t(jj) / t(h))
            out += [np.nextafter(v, t(-np.inf)), v, np.nextafter(v, t(np.inf))]
    z = np.array(out, dtype=xs.dtype)
    return z[(z >= xs[0]) & (z < xs[-1])]


def _layout_edges(k, r, zs):
    """Buckets at zone edges, the first words' edges and the first stripes' edges of every zone."""
    edges = []
    for z, kz in enumerate(k):
        zlo = z << zs
        s = kz + RANK_SHIFT
        edges += [zlo, zlo + (1 << zs) - 1]
        edges += [zlo + (g << s) for g in range(0, min(1 << (zs - s), 4))]
        edges += [zlo + (g << kz) for g in range(1, 6)]
        edges += [zlo + 31 * (1 << kz), zlo + 32 * (1 << kz) - 1]
    return [e for e in edges if 0 <= e <= r] + [r]


def _knot_neighbours(xs, count, seed):
    """Exact knots and the values one ulp either side (the z < X[t] compare)."""
    rng = np.random.default_rng(seed)
    pick = xs[rng.integers(0, len(xs) - 1, count)]
    z = np.concatenate([pick, np.nextafter(pick, -np.inf), np.nextafter(pick, np.inf)]).astype(xs.dtype)
    return z[(z >= xs[0]) & (z < xs[-1])]


def _geometric(n, ratio, dtype):
    gaps = 1e-4 * ratio ** np.arange(n, dtype=np.float64)
    return np.unique(np.concatenate([[0.0], np.cumsum(gaps)]).astype(dtype))


def with_zoned_rank(fs, p, prep, budget, window=None):
    """Plan and build striped rank words for `budget` bytes on prep's table;
    `window` = (t0, nt) overrides the planner's X window.  Returns (buffer, zs,
    k, nrec) or None when nothing fits."""
    from paper_1506_08620_b200 import _device, _lib

    idx = prep.structure
    lib = _lib.load()
    dt = _lib.FS_F32 if p.precision == "single" else _lib.FS_F64
    n1 = len(p.values)
    f_dev = _device.empty(n1, np.uint64)
    zs = ctypes.c_int32(-1)
    nrec, nbytes, t0, nt, ppm = (ctypes.c_uint64(0) for _ in range(5))
    rc = lib.fs_plan_zoned_rank(dt, p.device_values().data_ptr(), n1, float(idx.h), idx.r, budget, f_dev.data_ptr(),
                                ctypes.byref(zs), ctypes.byref(nrec), ctypes.byref(nbytes), ctypes.byref(t0),
                                ctypes.byref(nt), ctypes.byref(ppm), _device.stream_ptr())
    if rc == _lib.FS_TOO_LARGE:
        return None
    _lib.check(rc)
    assert nbytes.value == lib.fs_zoned_bytes(idx.r, zs.value, nrec.value)
    assert nbytes.value + 128 + nt.value * p.values.itemsize <= budget
    buf = _device.empty(int(nbytes.value), np.uint8)
    rc = lib.fs_build_zoned_rank(dt, p.device_values().data_ptr(), n1, float(idx.h), idx.r, zs.value, nrec.value,
                                 f_dev.data_ptr(), buf.data_ptr(), _device.stream_ptr())
    _lib.check(rc)
    plan = prep.plan
    plan.records = None
    plan.sparse = buf.data_ptr()
    plan.sparse_format = _lib.SPARSE_ZONED_RANK
    plan.sparse_shift = zs.value
    plan.sparse_ndense = nrec.value
    plan.hot_word0 = plan.hot_words = 0
    plan.hot_knot0, plan.hot_knots = window if window is not None else (t0.value, nt.value)
    return buf, zs.value, nrec.value, ppm.value


def _check_against_numpy(buf, f, r, zs, nrec, table_budget, ppm=None):
    """The planner's stripes for this zone shift and the buffer, bit for bit."""
    # the build re-plans with the budget set to the table's own size: same plan
    nz = (r >> zs) + 1
    k, total, xread = expected_plan(f, r, zs, table_budget)
    assert total == nrec
    k2, total2, _ = expected_plan(f, r, zs, 4 * ((nz + 3) // 4 * 4) + 8 * nrec)
    assert (k2, total2) == (k, total)
    desc, rec = expected_buffer(f, r, zs, k)
    got = buf.cpu().numpy()
    nzp = (nz + 3) // 4 * 4
    assert np.array_equal(got[: 4 * nz].view(np.uint32), desc)
    assert np.array_equal(got[4 * nzp: 4 * nzp + rec.nbytes].view(np.uint32).reshape(rec.shape), rec)
    if ppm is not None:
        assert ppm == int(xread * 10**6 // (r + 1)) or abs(ppm - xread * 1e6 / (r + 1)) <= 1
    return k


def _table_budget(budget, n1, es):
    win = min((n1 * es + 127) // 128 * 128, (budget // 8) // 128 * 128)
    return budget - win - 128


def test_zoned_rank_chosen_for_cfg4(cuda):
    """cfg4 (geometric knots, R = 7.0 M): prepare() stages striped rank words
    (stripes of one bucket at the dense start, growing behind) plus the densest
    knots; planner and buffer bit-exact; answers equal the oracle for both
    halves of the query mix, layout edges, knots and window edges, int32 and
    int64 outputs."""
    fs = _fs()
    from paper_1506_08620_b200 import batch, workloads

    p = workloads.knots("cfg4")
    prep = fs.prepare("direct", p)
    pl = prep.placement()
    assert pl["smem_sparse"] and pl["sparse_format"] == "zoned-rank" and not pl["smem_hot"], pl
    xs = p.values
    idx = prep.structure
    zs, nrec = prep.plan.sparse_shift, prep.plan.sparse_ndense
    f = orc.knot_buckets(xs, idx.h).astype(np.int64)
    budget = batch._smem_budget() - 512
    k = _check_against_numpy(_buffer_of(prep, prep.plan.sparse), f, idx.r, zs, nrec,
                             _table_budget(budget, len(xs), xs.itemsize))
    assert k[0] == 0 and max(k) >= 4  # the dense start needs one-bucket stripes, the tail takes coarse ones
    t0, nt = prep.plan.hot_knot0, prep.plan.hot_knots
    assert nt > 0 and pl["smem_x"]
    if nt < len(xs):
        span = f[nt - 1:] - f[: len(f) - nt + 1]
        assert t0 == int(np.argmin(span))
    z = np.concatenate([
        workloads.queries_host("cfg4", p, 400_000, seed=5),
        _edge_queries(xs, idx.h, _layout_edges(k, idx.r, zs)),
        _knot_neighbours(xs, 20_000, seed=3),
        xs[max(0, t0 - 3): t0 + 3], xs[max(0, t0 + nt - 3): t0 + nt + 3],
        np.nextafter(xs[max(0, t0 + nt - 3): t0 + nt + 3], -np.inf),
        orc.boundary_probes(xs), orc.bucket_edge_probes(xs, idx.h, idx.r, 100_000, seed=4),
    ]).astype(xs.dtype)
    z = z[(z >= xs[0]) & (z < xs[-1])]
    want = orc.rank_oracle(xs, z)
    assert np.array_equal(fs.run_batch(prep, z), want)
    out32 = np.empty(len(z), dtype=np.int32)
    fs.batch_search(fs.LaneConfig(1, "direct", prep), z, out32)
    assert np.array_equal(out32, want)


@pytest.mark.parametrize("dtype", [np.float32, np.float64])
def test_zoned_rank_budgets_and_windows(cuda, dtype):
    """A skewed table under striped rank words at several budgets (coarse
    stripes that read X often ... fine stripes) and X windows (none, the head,
    the middle, the tail): planner and buffer bit-exact, answers equal the
    oracle."""
    fs = _fs()
    from paper_1506_08620_b200 import batch

    xs = _geometric(20_000, 1.0003, dtype)
    p = fs.validate_partition(xs)
    prep = fs.prepare("direct", p)
    idx = prep.structure
    f = orc.knot_buckets(xs, idx.h).astype(np.int64)
    rng = np.random.default_rng(8)
    dense_top = xs[min(len(xs) - 1, 3000)]
    zbase = np.concatenate([orc.random_queries(xs, 150_000, seed=1),
                            rng.uniform(xs[0], dense_top, 150_000).astype(dtype),
                            _knot_neighbours(xs, 20_000, seed=2),
                            orc.boundary_probes(xs)]).astype(dtype)
    n1 = len(xs)
    full = batch._smem_budget() - 512
    seen = set()
    for budget in (24 * 1024, 64 * 1024, 128 * 1024, full):
        for window in (None, (0, 0), (0, 1500), (7000, 1200), (n1 - 700, 700)):
            made = with_zoned_rank(fs, p, prep, budget, window)
            if made is None:
                continue
            buf, zs, nrec, ppm = made
            k = _check_against_numpy(buf, f, idx.r, zs, nrec, _table_budget(budget, n1, xs.itemsize), ppm)
            seen.add(tuple(k))
            pl = prep.placement()
            assert pl["sparse_format"] == "zoned-rank", (budget, window, pl)
            t0, nt = prep.plan.hot_knot0, prep.plan.hot_knots
            assert pl["smem_x"] == (nt > 0)
            z = np.concatenate([zbase, _edge_queries(xs, idx.h, _layout_edges(k, idx.r, zs)),
                                xs[max(0, t0 - 2): t0 + 2], xs[max(0, t0 + nt - 2): t0 + nt + 2]]).astype(dtype)
            z = z[(z >= xs[0]) & (z < xs[-1])]
            assert np.array_equal(fs.run_batch(prep, z), orc.rank_oracle(xs, z)), (budget, window)
            del buf
    assert len(seen) >= 2  # the budgets really gave different stripes
    assert f[-1] == idx.r


def test_zoned_rank_irregular_table_falls_back(cuda):
    """A skewed table with close pairs scattered through its sparse tail needs
    one-bucket stripes everywhere: the striped words do not fit (or read X too
    often) and prepare() keeps the mixed slot/rank records; answers equal."""
    fs = _fs()

    xs = _geometric(60_000, 1.0001, np.float32).astype(np.float64)
    rng = np.random.default_rng(5)
    pairs = rng.choice(xs[30_000:], 400, replace=False) + 1.05e-4  # a knot one bucket behind another, all along the tail
    xs = np.unique(np.concatenate([xs, pairs])).astype(np.float32)
    xs = xs[np.concatenate([[True], np.diff(xs.astype(np.float64)) >= 9e-5])]
    p = fs.validate_partition(xs)
    prep = fs.prepare("direct", p)
    pl = prep.placement()
    assert pl["sparse_format"] != "zoned-rank", pl
    z = np.concatenate([orc.random_queries(xs, 200_000, seed=1), _knot_neighbours(xs, 5000, seed=2)])
    z = z[(z >= xs[0]) & (z < xs[-1])]
    assert np.array_equal(fs.run_batch(prep, z), orc.rank_oracle(xs, z))


def test_zoned_rank_threshold_and_switch(cuda):
    """ZONED_RANK_MAX_XREAD_PPM: 0 skips the striped words (cfg4 takes the
    mixed records), a threshold below the plan's X-read share does too."""
    fs = _fs()
    from paper_1506_08620_b200 import batch, workloads

    p = workloads.knots("cfg4")
    keep = batch.ZONED_RANK_MAX_XREAD_PPM
    try:
        for ppm in (0, 1000):
            batch.ZONED_RANK_MAX_XREAD_PPM = ppm
            assert fs.prepare("direct", p).placement()["sparse_format"] == "zoned", ppm
    finally:
        batch.ZONED_RANK_MAX_XREAD_PPM = keep


def test_zoned_rank_out_of_domain_and_last_bucket(cuda):
    """Out-of-domain lanes (NaN, +-inf, below X0, at XN) report the first bad
    position and write nothing; the last bucket R answers N - 1."""
    fs = _fs()
    from paper_1506_08620_b200 import workloads

    p = workloads.knots("cfg4")
    prep = fs.prepare("direct", p)
    assert prep.placement()["sparse_format"] == "zoned-rank"
    xs = p.values
    top = np.nextafter(xs[-1], -np.inf)
    z = np.array([xs[0], top, xs[-2], np.nextafter(xs[-2], -np.inf)], dtype=xs.dtype)
    assert fs.run_batch(prep, z).tolist() == orc.rank_oracle(xs, z).tolist()
    zq = workloads.queries_host("cfg4", p, 200_003, seed=2)
    for bad in (np.nan, np.inf, -np.inf, xs[-1], np.float32(-1.0)):
        zb = zq.copy()
        zb[123_457] = bad
        out = np.full(len(zb), -5, dtype=np.int32)
        with pytest.raises(fs.OutOfDomain) as e:
            fs.batch_search(fs.LaneConfig(1, "direct", prep), zb, out)
        assert e.value.position == 123_457
        assert (out == -5).all()


def test_zoned_rank_abi_validation(cuda):
    """fs_plan_zoned_rank: FS_TOO_LARGE for a budget nothing fits;
    fs_build_zoned_rank: FS_INVALID_ARG for zone shifts out of range and for a
    word count no plan of that zone shift has; validate_plan rejects bad zone
    shifts and knot windows for the format."""
    fs = _fs()
    from paper_1506_08620_b200 import _device, _lib, workloads

    p = workloads.knots("cfg4")
    prep = fs.prepare("direct", p)
    plan = prep.plan
    assert plan.sparse_format == _lib.SPARSE_ZONED_RANK
    lib = _lib.load()
    r = prep.structure.r
    n1 = len(p.values)
    f = _device.empty(n1, np.uint64)
    zs = ctypes.c_int32(0)
    outs = [ctypes.c_uint64(0) for _ in range(5)]
    for budget in (100, 1000, 20_000):
        rc = lib.fs_plan_zoned_rank(_lib.FS_F32, p.device_values().data_ptr(), n1, float(prep.structure.h), r, budget,
                                    f.data_ptr(), ctypes.byref(zs), *[ctypes.byref(o) for o in outs], None)
        assert rc == _lib.FS_TOO_LARGE, budget
    buf = _device.empty(int(lib.fs_zoned_bytes(r, plan.sparse_shift, plan.sparse_ndense)), np.uint8)
    for bad_zs in (5, 12, 40):
        rc = lib.fs_build_zoned_rank(_lib.FS_F32, p.device_values().data_ptr(), n1, float(prep.structure.h), r,
                                     bad_zs, plan.sparse_ndense, f.data_ptr(), buf.data_ptr(), None)
        assert rc == _lib.FS_INVALID_ARG, bad_zs
    for bad_nrec in (1, plan.sparse_ndense - 1):
        rc = lib.fs_build_zoned_rank(_lib.FS_F32, p.device_values().data_ptr(), n1, float(prep.structure.h), r,
                                     plan.sparse_shift, bad_nrec, f.data_ptr(), buf.data_ptr(), None)
        assert rc == _lib.FS_INVALID_ARG, bad_nrec
    z = workloads.queries_host("cfg4", p, 10_000, seed=1)
    for field, value in (("sparse_shift", 10), ("sparse_shift", 12), ("hot_knots", n1 + 1)):
        keep = getattr(plan, field)
        setattr(plan, field, value)
        with pytest.raises(ValueError):
            fs.run_batch(prep, z)
        setattr(plan, field, keep)
    assert np.array_equal(fs.run_batch(prep, z), orc.rank_oracle(p.values, z))
