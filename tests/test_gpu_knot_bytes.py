"""GPU tests of the knot bytes beside the rank directory (fs_build_knot_bytes +
RankBytesProbe): the bytes against a numpy construction that repeats the
reference's product op for op (direct.py:194-197: p = RN(h RN(X - X0)); byte =
floor(256 frac(p))), the placement rule (directory + bytes staged when
directory + X do not fit), and every answer against the oracle
(batch.py:315-317 semantics): every knot and its neighbours, queries whose
byte ties with their bucket's knot (the X read through L2), bucket edges, f32
and f64, int32 and int64 outputs, out-of-domain lanes."""

import numpy as np
import pytest

from oracle import fs_oracle as orc

pytestmark = pytest.mark.gpu


def _fs():
    import paper_1506_08620_b200 as fs

    return fs


def expected_bytes(xs, h):
    """floor(256 frac(p)) with p = RN(h * RN(X - X0)) in X's precision."""
    t = xs.dtype.type
    p = (t(h) * (xs - xs[0]).astype(xs.dtype)).astype(xs.dtype)
    return np.floor((p - np.floor(p)).astype(xs.dtype) * t(256)).astype(np.uint8)


def _buffer_of(prep, ptr):
    return next(b for b in prep.buffers if b.data_ptr() == ptr)


def _probe_queries(xs, h, r, seed):
    """Every knot, its neighbours by one and a few ulps, values sharing a knot's
    bucket on both sides of it and tied with its byte, bucket edges, random queries."""
    t = xs.dtype.type
    rng = np.random.default_rng(seed)
    near = [xs]
    for steps in (1, 2, 3, 7):
        lo, hi = xs.copy(), xs.copy()
        for _ in range(steps):
            lo, hi = np.nextafter(lo, t(-np.inf)), np.nextafter(hi, t(np.inf))
        near += [lo, hi]
    # inside the knot's bucket: offsets of a fraction of a bucket either side of the knot
    width = t(1) / t(h)
    for frac in (1 / 512, 1 / 300, 1 / 256, 1 / 200, 1 / 64, 1 / 3):
        near += [(xs - t(frac) * width).astype(xs.dtype), (xs + t(frac) * width).astype(xs.dtype)]
    z = np.concatenate(near + [orc.random_queries(xs, 300_000, seed=seed), orc.boundary_probes(xs),
                               orc.bucket_edge_probes(xs, h, r, 100_000, seed=seed + 1)]).astype(xs.dtype)
    return z[(z >= xs[0]) & (z < xs[-1])]


@pytest.mark.parametrize("precision,size", [("single", 65535), ("double", 65535), ("double", 32767), ("single", 131071)])
def test_knot_bytes_for_uniform_gap_tables(cuda, precision, size):
    """The paper's arrays (gaps U[1, 5]): the directory fits in shared memory,
    X does not; prepare() stages the directory and the knot bytes.  Bytes bit
    for bit against numpy; ties between a query's byte and its knot's exist in
    the probe set and resolve through X; answers equal the oracle."""
    fs = _fs()
    from paper_1506_08620_b200 import _lib

    p = fs.gen_uniform_gap_partition(size, 1.0, 5.0, 42, precision)
    prep = fs.prepare("direct", p)
    pl = prep.placement()
    assert pl["sparse_format"] == "knot-bytes" and pl["smem_table"] and pl["smem_sparse"] and not pl["smem_hot"], pl
    xs = p.values
    idx = prep.structure
    assert prep.plan.sparse_format == _lib.SPARSE_KNOT_BYTES and prep.plan.sparse_ndense == len(xs)
    want_bytes = expected_bytes(xs, idx.h)
    got = _buffer_of(prep, prep.plan.sparse).cpu().numpy()
    assert np.array_equal(got[: len(xs)], want_bytes) and not got[len(xs):].any()
    assert len(got) == (len(xs) + 15) // 16 * 16
    z = _probe_queries(xs, idx.h, idx.r, seed=3)
    # the probe set holds queries tied with their bucket's knot in (bucket, byte), on both sides of it
    t = xs.dtype.type
    pz = (t(idx.h) * (z - xs[0]).astype(xs.dtype)).astype(xs.dtype)
    jz = np.floor(pz).astype(np.int64)
    qz = np.floor((pz - np.floor(pz)).astype(xs.dtype) * t(256)).astype(np.int64)
    f = orc.knot_buckets(xs, idx.h).astype(np.int64)
    pos = np.searchsorted(f, jz)
    has = (pos < len(f)) & (f[np.minimum(pos, len(f) - 1)] == jz)
    tie = has & (want_bytes[np.minimum(pos, len(f) - 1)] == qz)
    assert np.count_nonzero(tie & (z < xs[np.minimum(pos, len(f) - 1)])) > 100
    assert np.count_nonzero(tie & (z >= xs[np.minimum(pos, len(f) - 1)])) > 100
    want = orc.rank_oracle(xs, z)
    assert np.array_equal(fs.run_batch(prep, z), want)
    out32 = np.empty(len(z), dtype=np.int32)
    fs.batch_search(fs.LaneConfig(1, "direct", prep), z, out32)
    assert np.array_equal(out32, want)


def test_knot_bytes_rule_and_switch(cuda):
    """Not used when X fits beside the directory (cfg1, uniform-gap 4095), when
    the directory itself does not fit (cfg4, cfg5 N+1 = 32769), or with the knob
    off (same answers from the directory alone)."""
    fs = _fs()
    from paper_1506_08620_b200 import batch, workloads

    for p in (workloads.knots("cfg1"), fs.gen_uniform_gap_partition(4095, 1.0, 5.0, 42, "double"),
              workloads.knots("cfg4"), workloads.knots("cfg5", n1=32769)):
        assert fs.prepare("direct", p).placement()["sparse_format"] != "knot-bytes"
    p = fs.gen_uniform_gap_partition(65535, 1.0, 5.0, 7, "single")
    z = _probe_queries(p.values, fs.prepare("direct", p).structure.h, fs.prepare("direct", p).structure.r, seed=5)
    want = orc.rank_oracle(p.values, z)
    saved = batch.KNOT_BYTES
    try:
        batch.KNOT_BYTES = False
        prep = fs.prepare("direct", p)
        assert prep.placement()["sparse_format"] is None and prep.placement()["smem_table"]
        assert np.array_equal(fs.run_batch(prep, z), want)
    finally:
        batch.KNOT_BYTES = saved
    prep = fs.prepare("direct", p)
    assert prep.placement()["sparse_format"] == "knot-bytes"
    assert np.array_equal(fs.run_batch(prep, z), want)


def test_knot_bytes_out_of_domain(cuda):
    """Out-of-domain lanes (NaN, +-inf, below X0, at and above XN) beside valid
    ones report the first bad position and fault nothing; the last bucket resolves."""
    fs = _fs()
    p = fs.gen_uniform_gap_partition(65535, 1.0, 5.0, 11, "double")
    xs = p.values
    prep = fs.prepare("direct", p)
    assert prep.placement()["sparse_format"] == "knot-bytes"
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


def test_knot_bytes_abi_validation(cuda):
    """fs_build_knot_bytes argument checks, and validate_plan on a knot-byte plan
    without its directory or with a byte count that is not one per knot."""
    fs = _fs()
    from paper_1506_08620_b200 import _device, _lib

    p = fs.gen_uniform_gap_partition(65535, 1.0, 5.0, 3, "single")
    prep = fs.prepare("direct", p)
    lib = _lib.load()
    n1 = len(p.values)
    x = p.device_values()
    buf = _device.empty((n1 + 15) // 16 * 16, np.uint8)
    st = _device.stream_ptr()
    h = float(prep.structure.h)
    assert lib.fs_build_knot_bytes(_lib.FS_F32, None, n1, h, buf.data_ptr(), st) == _lib.FS_INVALID_ARG
    assert lib.fs_build_knot_bytes(_lib.FS_F32, x.data_ptr(), n1, h, None, st) == _lib.FS_INVALID_ARG
    assert lib.fs_build_knot_bytes(_lib.FS_F32, x.data_ptr(), 1, h, buf.data_ptr(), st) == _lib.FS_INVALID_ARG
    assert lib.fs_build_knot_bytes(9, x.data_ptr(), n1, h, buf.data_ptr(), st) == _lib.FS_INVALID_ARG
    assert lib.fs_build_knot_bytes(_lib.FS_F32, x.data_ptr(), n1, h, buf.data_ptr(), st) == _lib.FS_OK
    z = orc.random_queries(p.values, 1000, seed=1)
    assert np.array_equal(fs.run_batch(prep, z), orc.rank_oracle(p.values, z))
    keep = prep.plan.sparse_ndense
    prep.plan.sparse_ndense = n1 - 1
    with pytest.raises(ValueError):
        fs.run_batch(prep, z)
    prep.plan.sparse_ndense = keep
    rank = prep.plan.rank
    prep.plan.rank = None
    with pytest.raises(ValueError):
        fs.run_batch(prep, z)
    prep.plan.rank = rank
    assert np.array_equal(fs.run_batch(prep, z), orc.rank_oracle(p.values, z))
