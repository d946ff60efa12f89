"""GPU tests of the group-record layout of the gap-1 table
(fs_build_sparse_rec): the device buffer against a numpy construction from
the oracle's knot buckets (bit for bit), and every answer against the
oracle (batch.py:315-317 semantics) for every super-bucket shift, for
super-buckets holding 0..6 knots (resolved inside the record) and more
(the overflow path past the sixth knot), at bucket edges, exact knots and
the last bucket R."""

import ctypes

import numpy as np
import pytest

from oracle import fs_oracle as orc

pytestmark = pytest.mark.gpu

SENTINEL = 0x7FFF
FORMATS = {"records": 6, "records8": 2, "records12": 8, "records8x3": 3}  # offset slots per record
MAX_SHIFT = {"records": 14, "records8": 14, "records12": 10, "records8x3": 11}


def _fs():
    import paper_1506_08620_b200 as fs

    return fs


def _fmt_code(name):
    from paper_1506_08620_b200 import _lib

    return {"records": _lib.SPARSE_RECORDS, "records8": _lib.SPARSE_RECORDS8, "records12": _lib.SPARSE_RECORDS12,
            "records8x3": _lib.SPARSE_RECORDS8X3}[name]


def expected_records(xs, h, r, s, slots=6):
    """uint32 (ng, words): {base | overflow << 31, off0 | off1 << 16, ...};
    for 8 slots, 96 bits of 12-bit fields 0x800 | offset (unused 0xFFF)."""
    f = orc.knot_buckets(xs, h).astype(np.uint64)
    ng = (r >> s) + 2
    base = np.searchsorted(f, np.arange(ng, dtype=np.uint64) << np.uint64(s), side="left").astype(np.int64)
    rec = np.zeros((ng, {8: 4, 3: 2}.get(slots, 1 + slots // 2)), dtype=np.uint32)
    mask = (1 << s) - 1
    for J in range(ng):
        lo = int(base[J])
        hi = int(base[J + 1]) if J + 1 < ng else lo
        offs = [int(f[i]) & mask for i in range(lo, min(hi, lo + slots))]
        offs += [{8: 0x7FF, 3: 0xFFF}.get(slots, SENTINEL)] * (slots - len(offs))
        rec[J, 0] = lo | ((hi - lo > slots) << 31)
        if slots == 3:
            w = lo | ((hi - lo > slots) << 24)
            w |= sum((0x1000 | o) << (25 + 13 * e) for e, o in enumerate(offs))
            rec[J, 0], rec[J, 1] = w & 0xFFFFFFFF, w >> 32
        elif slots == 8:
            bits = sum((0x800 | o) << (12 * e) for e, o in enumerate(offs))
            for w in range(3):
                rec[J, 1 + w] = (bits >> (32 * w)) & 0xFFFFFFFF
        else:
            for w in range(slots // 2):
                rec[J, 1 + w] = offs[2 * w] | (offs[2 * w + 1] << 16)
    return rec, f & np.uint64(mask)


def _buffer_of(prep, ptr):
    return next(b for b in prep.buffers if b.data_ptr() == ptr)


def with_records(fs, p, prep, s, fmt="records"):
    """Rebuild prep's sparse table as group records (format fmt) with
    super-bucket shift s (the caller keeps the returned buffer alive while the
    plan uses it)."""
    from paper_1506_08620_b200 import _device, _lib

    idx = prep.structure
    rec, _ = expected_records(p.values, idx.h, idx.r, s, FORMATS[fmt])
    novf = int(np.count_nonzero((rec[:, 0] >> 24) & 1 if fmt == "records8x3" else rec[:, 0] >> 31))
    lib = _lib.load()
    code = _fmt_code(fmt)
    nbytes = int(lib.fs_sparse_rec_bytes(code, len(p.values), idx.r, s, novf))
    buf = _device.empty(nbytes, np.uint8)
    f = _device.empty(len(p.values), np.uint64)
    rc = lib.fs_build_sparse_rec(code, _lib.FS_F32 if p.precision == "single" else _lib.FS_F64,
                                 p.device_values().data_ptr(), len(p.values), float(idx.h), idx.r, s, novf,
                                 f.data_ptr(), buf.data_ptr(), _device.stream_ptr())
    _lib.check(rc)
    prep.plan.records = None
    prep.plan.rank = None  # records are used whenever they fit (a fitting directory would win otherwise)
    prep.plan.sparse = buf.data_ptr()
    prep.plan.sparse_shift = s
    prep.plan.sparse_ndense = novf
    prep.plan.sparse_format = code
    return buf, rec, novf


def _probe_set(xs, h, r, m, seed):
    z = np.concatenate([orc.random_queries(xs, m, seed=seed), orc.boundary_probes(xs),
                        orc.bucket_edge_probes(xs, h, r, 50_000, seed=seed + 1)])
    return z[(z >= xs[0]) & (z < xs[-1])]


def clustered_partition(seed, dtype=np.float64):
    """Mostly sparse knots plus clusters of 1..12 knots at the minimum gap:
    super-buckets holding 0..12 knots at every shift, knots in the first and
    last bucket of super-buckets."""
    rng = np.random.default_rng(seed)
    base = np.sort(rng.uniform(0.0, 1.0, 600))
    g = 5e-6 if dtype == np.float64 else 2e-5  # R <= 2e5: records fit in smem at every shift
    parts = [base]
    for k, c in enumerate(rng.uniform(0.05, 0.95, 40)):
        parts.append(c + g * np.arange(1 + k % 12))
    xs = np.unique(np.concatenate(parts + [[0.0, 1.0]])).astype(dtype)
    keep = np.concatenate([[True], np.diff(xs) >= 0.99 * g])
    xs = np.unique(xs[keep])
    return xs


def _records_forced(fs, p, fmt="records"):
    from paper_1506_08620_b200 import batch

    old = batch.SPARSE_FORMATS, batch.SPARSE_RECORDS_MAX_PAST_SIXTH_PPM, batch.SPARSE_RECORDS8_MAX_PAST_PPM
    try:
        batch.SPARSE_FORMATS = (fmt,)
        batch.SPARSE_RECORDS_MAX_PAST_SIXTH_PPM = batch.SPARSE_RECORDS8_MAX_PAST_PPM = 10**6
        return fs.prepare("direct", p)
    finally:
        batch.SPARSE_FORMATS, batch.SPARSE_RECORDS_MAX_PAST_SIXTH_PPM, batch.SPARSE_RECORDS8_MAX_PAST_PPM = old


def test_records_chosen_for_sparse_configs(cuda, monkeypatch):
    """The planner's picks (profiles/r01/tune_sparse_records.txt): cfg2 seed 0
    16-B records with X staged; cfg2 seed 1 (R = 398.6 M) 8-B records, X via
    L2; cfg5 N+1 = 1025 8-B records with X; cfg5 N+1 = 32769 overflowing 16-B
    records, X via L2.  The buffer equals the numpy construction, answers
    equal the oracle."""
    fs = _fs()
    from paper_1506_08620_b200 import workloads

    from paper_1506_08620_b200 import batch

    # the picks among the record layouts (count words, tried first, are tested in test_gpu_count_words.py)
    monkeypatch.setattr(batch, "SPARSE_FORMATS", tuple(n for n in batch.SPARSE_FORMATS if n != "count-words"))
    for name, kw, fmts, sx in (("cfg2", {}, ("records", "records8x3"), True), ("cfg2", {"seed": 1}, ("records8",), False),
                               ("cfg5", {"n1": 1025}, ("records8",), True),
                               ("cfg5", {"n1": 32769}, ("records", "records12"), False)):
        p = workloads.knots(name, **kw)
        prep = fs.prepare("direct", p)
        pl = prep.placement()
        fmt = pl["sparse_format"]
        assert pl["smem_sparse"] and fmt in fmts and pl["smem_x"] == sx, (name, kw, pl)
        idx = prep.structure
        s = prep.plan.sparse_shift
        rec, fmod = expected_records(p.values, idx.h, idx.r, s, FORMATS[fmt])
        buf = _buffer_of(prep, prep.plan.sparse).cpu().numpy()
        assert np.array_equal(buf[: rec.nbytes].view(np.uint32).reshape(rec.shape), rec), name
        novf = int(np.count_nonzero((rec[:, 0] >> 24) & 1 if fmt == "records8x3" else rec[:, 0] >> 31))
        assert prep.plan.sparse_ndense == novf
        if novf:
            assert np.array_equal(buf[rec.nbytes: rec.nbytes + 2 * len(fmod)].view(np.uint16), fmod.astype(np.uint16))
        z = np.concatenate([_probe_set(p.values, idx.h, idx.r, 400_000, seed=3),
                            workloads.queries_host(name, p, 200_000, seed=5)])
        want = orc.rank_oracle(p.values, z)
        assert np.array_equal(fs.run_batch(prep, z), want), (name, kw)
        out32 = np.empty(len(z), dtype=np.int32)
        fs.batch_search(fs.LaneConfig(1, "direct", prep), z, out32)
        assert np.array_equal(out32, want), (name, kw)
        del prep


@pytest.mark.parametrize("fmt", sorted(FORMATS))
@pytest.mark.parametrize("dtype", [np.float64, np.float32])
def test_records_every_shift_with_overflow(cuda, dtype, fmt):
    """Clusters of 1..12 knots: records holding 0..slots knots and
    overflowing records at every shift 5..14; buffer bit-exact, answers exact."""
    fs = _fs()
    xs = clustered_partition(7, dtype)
    p = fs.validate_partition(xs)
    prep = fs.prepare("direct", p)
    idx = prep.structure
    z = _probe_set(xs, idx.h, idx.r, 200_000, seed=11)
    # queries inside every cluster (the overflow path) and at each knot's neighbours
    near = np.concatenate([np.nextafter(xs, -np.inf), xs, np.nextafter(xs, np.inf),
                           (xs[:-1] + (xs[1:] - xs[:-1]) * 0.5).astype(xs.dtype)])
    z = np.concatenate([z, near[(near >= xs[0]) & (near < xs[-1])]]).astype(xs.dtype)
    want = orc.rank_oracle(xs, z)
    assert idx.r < 230_000
    seen_ovf = False
    for s in range(5, MAX_SHIFT[fmt] + 1):
        buf, rec, novf = with_records(fs, p, prep, s, fmt)
        seen_ovf |= novf > 0
        got = buf.cpu().numpy()[: rec.nbytes].view(np.uint32).reshape(rec.shape)
        assert np.array_equal(got, rec), s
        assert prep.placement()["sparse_format"] == fmt
        assert np.array_equal(fs.run_batch(prep, z), want), s
    assert seen_ovf


def test_records_overflow_chosen_by_planner(cuda):
    """A tight 200-knot cluster in a sparse layout: group records of either
    width (forced) with overflowing records, and the layout the planner picks,
    give the oracle's answers."""
    fs = _fs()

    rng = np.random.default_rng(17)
    base = np.sort(rng.uniform(0.0, 1.0, 1000))
    base = base[np.concatenate([[True], np.diff(base) > 1e-5])]
    cluster = 0.5 + 1e-7 * np.arange(1, 201)
    xs = np.unique(np.concatenate([base[(base < 0.5) | (base > 0.5 + 1e-4)], cluster, [0.0, 1.0]]))
    p = fs.validate_partition(xs)
    z = np.concatenate([orc.random_queries(xs, 300_000, seed=2), orc.boundary_probes(xs),
                        np.random.default_rng(3).uniform(0.5, 0.5 + 2.1e-5, 100_000)])
    z = z[(z >= xs[0]) & (z < xs[-1])]
    want = orc.rank_oracle(xs, z)
    for fmt in FORMATS:
        prep = _records_forced(fs, p, fmt)
        assert prep.placement()["sparse_format"] == fmt and prep.plan.sparse_ndense > 0
        assert np.array_equal(fs.run_batch(prep, z), want), fmt
    prep2 = fs.prepare("direct", p)
    assert prep2.placement()["smem_sparse"]
    assert np.array_equal(fs.run_batch(prep2, z), want)


@pytest.mark.parametrize("fmt", sorted(FORMATS))
def test_records_out_of_domain_and_last_bucket(cuda, fmt):
    """Out-of-domain lanes (NaN, +-inf, below X0, at XN) clamp inside the
    records; the first bad position is reported; the last bucket R (the
    sentinel record after it is read by the overflow path) answers N-1."""
    fs = _fs()
    from paper_1506_08620_b200 import workloads

    p = workloads.knots("cfg5", n1=1025)
    prep = _records_forced(fs, p, fmt)
    assert prep.placement()["sparse_format"] == fmt
    xs = p.values
    top = np.nextafter(xs[-1], -np.inf)
    z = np.array([xs[0], top, xs[-2], np.nextafter(xs[-2], -np.inf)], dtype=xs.dtype)
    assert fs.run_batch(prep, z).tolist() == orc.rank_oracle(xs, z).tolist()
    for bad in (np.nan, np.inf, -np.inf, xs[-1], np.nextafter(xs[0], -np.inf)):
        zb = np.concatenate([orc.random_queries(xs, 1001, seed=4), [bad], orc.random_queries(xs, 77, seed=5)])
        out = np.full(len(zb), -7, dtype=np.int64)
        with pytest.raises(fs.OutOfDomain) as e:
            fs.batch_search(fs.LaneConfig(1, "direct", prep), zb.astype(xs.dtype), out)
        assert e.value.position == 1001
        assert (out == -7).all()


def test_records_abi_validation(cuda):
    """validate_plan: unknown formats and shifts above 14 are rejected."""
    fs = _fs()
    from paper_1506_08620_b200 import _lib, workloads

    p = workloads.knots("cfg5", n1=1025)
    prep = _records_forced(fs, p)
    z = orc.random_queries(p.values, 1000, seed=1)
    for fmt, shift in ((5, prep.plan.sparse_shift), (_lib.SPARSE_RECORDS, 15), (_lib.SPARSE_RECORDS12, 11),
                       (_lib.SPARSE_RECORDS8X3, 12)):
        keep = (prep.plan.sparse_format, prep.plan.sparse_shift)
        prep.plan.sparse_format, prep.plan.sparse_shift = fmt, shift
        with pytest.raises(ValueError):
            fs.run_batch(prep, z)
        prep.plan.sparse_format, prep.plan.sparse_shift = keep
    assert np.array_equal(fs.run_batch(prep, z), orc.rank_oracle(p.values, z))
    lib = _lib.load()
    rb = lib.fs_sparse_rec_bytes
    assert rb(_lib.SPARSE_RECORDS, 1025, 1 << 20, 15, 0) == 0
    assert rb(_lib.SPARSE_RECORDS, 1025, 1 << 20, 10, 0) == 16 * ((1 << 10) + 2)
    assert rb(_lib.SPARSE_RECORDS, 1025, 1 << 20, 10, 3) == (16 * ((1 << 10) + 2) + 2 * 1025 + 15) // 16 * 16
    assert rb(_lib.SPARSE_RECORDS8, 1025, 1 << 20, 10, 3) == (8 * ((1 << 10) + 2) + 2 * 1025 + 15) // 16 * 16
