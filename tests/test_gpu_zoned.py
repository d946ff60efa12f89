"""GPU tests of the zoned-record layout of the gap-1 table (fs_plan_zoned /
fs_build_zoned + ZonedProbe): the device buffer against a numpy
construction from the oracle's knot buckets (bit for bit), and every answer
against the oracle (batch.py:315-317 semantics) at zone edges, record edges,
exact knots, both sides of the staged X window, the last bucket R, and
out-of-domain lanes."""

import ctypes

import numpy as np
import pytest

from oracle import fs_oracle as orc

pytestmark = pytest.mark.gpu

MIN_SHIFT, MAX_SHIFT, SLOTS, RANK_SHIFT, RANK_FLAG = 6, 11, 3, 5, 16


@pytest.fixture(autouse=True)
def mixed_records_only():
    """These tests cover the mixed slot/rank records; the striped rank words
    that prepare() tries first (tests/test_gpu_zoned_rank.py) are switched off."""
    from paper_1506_08620_b200 import batch

    keep = batch.ZONED_RANK_MAX_XREAD_PPM
    batch.ZONED_RANK_MAX_XREAD_PPM = 0
    yield
    batch.ZONED_RANK_MAX_XREAD_PPM = keep


def _fs():
    import paper_1506_08620_b200 as fs

    return fs


def expected_zoned(xs, h, r, zs):
    """(desc uint32[nz], records uint32[nrec, 2]) as fs_build_zoned lays them
    out: per zone the largest shift 6..min(11, zs) whose records hold <= 3
    knots (slot records: base | fields 0x1000 | offset at bits 25 + 13k,
    unused 0x1FFF), else 32-bucket rank records {mask, base}."""
    f = orc.knot_buckets(xs, h).astype(np.int64)
    nz = (r >> zs) + 1
    desc, recs = [], []
    nrec = 0
    for z in range(nz):
        zlo = z << zs
        zb = min(1 << zs, r + 1 - zlo)
        fz = f[(f >= zlo) & (f < zlo + zb)] - zlo
        s = -1
        for sh in range(min(MAX_SHIFT, zs), MIN_SHIFT - 1, -1):
            if len(fz) == 0 or np.bincount(fz >> sh).max() <= SLOTS:
                s = sh
                break
        rank = s < 0
        if rank:
            s = RANK_SHIFT
        n = (zb + (1 << s) - 1) >> s
        rel = nrec - (z << (zs - s))  # zone-relative first record (signed 27 bits)
        desc.append(((rel << 5) & 0xFFFFFFFF) | (RANK_FLAG if rank else 0) | s)
        j0 = zlo + (np.arange(n, dtype=np.int64) << s)
        lo = np.searchsorted(f, j0, side="left")
        hi = np.searchsorted(f, j0 + (1 << s), side="left")
        for g in range(n):
            inr = [int(v) for v in f[lo[g]:hi[g]] - j0[g]]
            if rank:
                recs.append([sum(1 << o for o in inr), int(lo[g])])
            else:
                assert len(inr) <= SLOTS
                w = int(lo[g])
                for k, o in enumerate(inr + [0xFFF] * (SLOTS - len(inr))):
                    w |= (0x1000 | o) << (25 + 13 * k)
                recs.append([w & 0xFFFFFFFF, w >> 32])
        nrec += n
    return np.array(desc, dtype=np.uint32), np.array(recs, dtype=np.uint64).astype(np.uint32)


def _buffer_of(prep, ptr):
    return next(b for b in prep.buffers if b.data_ptr() == ptr)


def _check_buffer(prep, p):
    idx = prep.structure
    zs = prep.plan.sparse_shift
    desc, rec = expected_zoned(p.values, idx.h, idx.r, zs)
    buf = _buffer_of(prep, prep.plan.sparse).cpu().numpy()
    nzp = (len(desc) + 3) // 4 * 4
    got_desc = buf[: 4 * len(desc)].view(np.uint32)
    assert np.array_equal(got_desc, desc)
    got_rec = buf[4 * nzp: 4 * nzp + rec.nbytes].view(np.uint32).reshape(rec.shape)
    assert np.array_equal(got_rec, rec)
    assert prep.plan.sparse_ndense == len(rec)
    return desc, rec


def with_zoned(fs, p, prep, zs, t0, nt):
    """Rebuild prep's table as zoned records with zone shift zs and the knot
    window X[t0, t0 + nt) (the caller keeps the returned buffer alive)."""
    from paper_1506_08620_b200 import _device, _lib

    idx = prep.structure
    desc, rec = expected_zoned(p.values, idx.h, idx.r, zs)
    lib = _lib.load()
    nbytes = int(lib.fs_zoned_bytes(idx.r, zs, len(rec)))
    assert nbytes == 4 * ((len(desc) + 3) // 4 * 4) + rec.nbytes
    buf = _device.empty(nbytes, np.uint8)
    f = _device.empty(len(p.values), np.uint64)
    rc = lib.fs_build_zoned(_lib.FS_F32 if p.precision == "single" else _lib.FS_F64, p.device_values().data_ptr(),
                            len(p.values), float(idx.h), idx.r, zs, f.data_ptr(), buf.data_ptr(),
                            _device.stream_ptr())
    _lib.check(rc)
    plan = prep.plan
    plan.records = None
    plan.sparse = buf.data_ptr()
    plan.sparse_format = _lib.SPARSE_ZONED
    plan.sparse_shift = zs
    plan.sparse_ndense = len(rec)
    plan.hot_word0 = plan.hot_words = 0
    plan.hot_knot0, plan.hot_knots = t0, nt
    return buf, desc, rec


def _edge_queries(xs, h, buckets):
    """Queries at the first/last bucket of each given bucket index, +-1 ulp."""
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


def _zone_and_record_edges(desc, r, zs):
    edges = []
    for z, d in enumerate(desc):
        zlo = z << zs
        s = int(d) & 15
        edges += [zlo, zlo + (1 << zs) - 1]
        edges += [zlo + (g << s) for g in range(0, min(1 << (zs - s), 6))]
        edges += [zlo + (g << s) - 1 for g in range(1, min(1 << (zs - s), 6))]
    return [e for e in edges if 0 <= e <= r] + [r]


def _geometric(n, ratio, dtype):
    gaps = 1e-4 * ratio ** np.arange(n, dtype=np.float64)
    return np.unique(np.concatenate([[0.0], np.cumsum(gaps)]).astype(dtype))


def test_zoned_chosen_for_cfg4(cuda):
    """cfg4 (geometric knots, R = 7.0 M, directory 1.75 MB): the planner
    stages zoned records (rank records at the dense start, slot records of
    growing shift behind) plus the densest knots; buffer bit-exact, answers
    equal the oracle for both halves of the query mix, zone and record edges,
    knots and window edges, int32 and int64 outputs."""
    fs = _fs()
    from paper_1506_08620_b200 import workloads

    p = workloads.knots("cfg4")
    prep = fs.prepare("direct", p)
    pl = prep.placement()
    assert pl["smem_sparse"] and pl["sparse_format"] == "zoned" and not pl["smem_hot"], pl
    desc, rec = _check_buffer(prep, p)
    assert any(int(d) & RANK_FLAG for d in desc) and any(not int(d) & RANK_FLAG for d in desc)
    xs = p.values
    idx = prep.structure
    t0, nt = prep.plan.hot_knot0, prep.plan.hot_knots
    assert nt > 0 and pl["smem_x"]
    f = orc.knot_buckets(xs, idx.h).astype(np.int64)
    if nt < len(xs):  # the window is the first of the densest nt-knot spans
        span = f[nt - 1:] - f[: len(f) - nt + 1]
        assert t0 == int(np.argmin(span))
    z = np.concatenate([
        workloads.queries_host("cfg4", p, 400_000, seed=5),
        _edge_queries(xs, idx.h, _zone_and_record_edges(desc, idx.r, prep.plan.sparse_shift)),
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
def test_zoned_every_window_and_zone_shift(cuda, dtype):
    """A skewed table (dense start, sparse tail) under zoned records at both
    zone shifts the planner considers and at several X windows (none, the
    head, the middle, all of X when it fits): buffer bit-exact, answers equal
    the oracle."""
    fs = _fs()
    from paper_1506_08620_b200 import batch

    xs = _geometric(20_000, 1.0003, dtype)
    p = fs.validate_partition(xs)
    prep = fs.prepare("direct", p)
    idx = prep.structure
    zs32 = 11
    while (idx.r >> zs32) + 1 > 32:
        zs32 += 1
    f = orc.knot_buckets(xs, idx.h).astype(np.int64)
    rng = np.random.default_rng(8)
    dense_top = xs[min(len(xs) - 1, 3000)]
    zbase = np.concatenate([orc.random_queries(xs, 150_000, seed=1),
                            rng.uniform(xs[0], dense_top, 150_000).astype(dtype),
                            orc.boundary_probes(xs)]).astype(dtype)
    n1 = len(xs)
    budget = batch._smem_budget() - 512
    for zs in (zs32, zs32 - 1):
        if zs < 11:
            continue
        for t0, nt in ((0, 0), (0, 4000), (7000, 2500), (n1 - 1000, 1000)):
            buf, desc, rec = with_zoned(fs, p, prep, zs, t0, nt)
            if 4 * len(desc) + rec.nbytes + 128 + nt * xs.itemsize > budget:
                continue
            pl = prep.placement()
            assert pl["sparse_format"] == "zoned" and pl["smem_x"] == (nt > 0), (zs, t0, nt, pl)
            got = _buffer_of_ptr(buf)
            nzp = (len(desc) + 3) // 4 * 4
            assert np.array_equal(got[: 4 * len(desc)].view(np.uint32), desc)
            assert np.array_equal(got[4 * nzp:].view(np.uint32).reshape(rec.shape), rec)
            z = np.concatenate([zbase,
                                _edge_queries(xs, idx.h, _zone_and_record_edges(desc, idx.r, zs)),
                                xs[max(0, t0 - 2): t0 + 2], xs[max(0, t0 + nt - 2): t0 + nt + 2]]).astype(dtype)
            z = z[(z >= xs[0]) & (z < xs[-1])]
            assert np.array_equal(fs.run_batch(prep, z), orc.rank_oracle(xs, z)), (zs, t0, nt)
            del buf
    assert f[-1] == idx.r


def _buffer_of_ptr(buf):
    return buf.cpu().numpy()


def test_zoned_out_of_domain_and_last_bucket(cuda):
    """cfg4 zoned: out-of-domain lanes (NaN, +-inf, below X0, at XN) report
    the first bad position and write nothing; the last bucket R answers N-1."""
    fs = _fs()
    from paper_1506_08620_b200 import workloads

    p = workloads.knots("cfg4")
    prep = fs.prepare("direct", p)
    assert prep.placement()["sparse_format"] == "zoned"
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


def test_zoned_not_used_when_directory_fits(cuda):
    """Tables whose rank directory (+ X) fits in shared memory, or that a
    sparse layout serves, keep those layouts (cfg3, cfg5 N+1 = 1025); a table
    no zoning fits keeps the L2 directory (cfg5 N+1 = 2^20 + 1); with zoning
    off, cfg4 takes its hot window."""
    fs = _fs()
    from paper_1506_08620_b200 import batch, workloads

    for name, kw in (("cfg3", {}), ("cfg5", {"n1": 1025}), ("cfg5", {"n1": 1_048_577})):
        prep = fs.prepare("direct", workloads.knots(name, **kw))
        assert prep.placement()["sparse_format"] != "zoned", (name, kw)
    keep = batch.ZONED
    batch.ZONED = False
    try:
        pl = fs.prepare("direct", workloads.knots("cfg4")).placement()
    finally:
        batch.ZONED = keep
    assert pl["smem_hot"] and pl["sparse_format"] != "zoned", pl


def test_zoned_abi_validation(cuda):
    """validate_plan: zone shifts giving > 64 zones or < 2^11 buckets, and a
    knot window outside X, are rejected; fs_zoned_bytes reports 0 for them."""
    fs = _fs()
    from paper_1506_08620_b200 import _lib, workloads

    p = workloads.knots("cfg4")
    prep = fs.prepare("direct", p)
    z = workloads.queries_host("cfg4", p, 10_000, seed=1)
    plan = prep.plan
    lib = _lib.load()
    r = prep.structure.r
    assert lib.fs_zoned_bytes(r, 10, 100) == 0
    assert lib.fs_zoned_bytes(r, 12, 100) == 0  # 1711 zones
    assert lib.fs_zoned_bytes(r, plan.sparse_shift, 100) == 4 * (((r >> plan.sparse_shift) + 4) // 4 * 4) + 800
    for field, value in (("sparse_shift", 10), ("sparse_shift", 12), ("hot_knots", len(p.values) + 1)):
        keep = getattr(plan, field)
        setattr(plan, field, value)
        with pytest.raises(ValueError):
            fs.run_batch(prep, z)
        setattr(plan, field, keep)
    assert np.array_equal(fs.run_batch(prep, z), orc.rank_oracle(p.values, z))
    f = _device_f(len(p.values))
    zs = ctypes.c_int32(0)
    outs = [ctypes.c_uint64(0) for _ in range(4)]
    rc = lib.fs_plan_zoned(_lib.FS_F32, p.device_values().data_ptr(), len(p.values), float(prep.structure.h), r,
                           1000, f.data_ptr(), ctypes.byref(zs), *[ctypes.byref(o) for o in outs], None)
    assert rc == _lib.FS_TOO_LARGE
    buf = _device_f(4096)
    for bad_zs in (5, 12, 40):  # below the minimum zone, > 64 zones, beyond 31
        rc = lib.fs_build_zoned(_lib.FS_F32, p.device_values().data_ptr(), len(p.values), float(prep.structure.h), r,
                                bad_zs, f.data_ptr(), buf.data_ptr(), None)
        assert rc == _lib.FS_INVALID_ARG, bad_zs


def _device_f(n):
    from paper_1506_08620_b200 import _device

    return _device.empty(n, np.uint64)
