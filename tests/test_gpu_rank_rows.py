"""GPU tests of the 16-B rank rows (fs_build_rank_rows + RankRowsProbe), the
directory layout of tables searched through L2: rows bit for bit against a
numpy construction (mask and base from the oracle's knot buckets, the knot
bytes from the reference's product repeated op for op, direct.py:194-197),
and every answer against the oracle (batch.py:315-317 semantics) on cfg5 N+1 =
2^20 + 1 (rows of ~3 knots) and the paper's uniform-gap arrays at 2^20 - 1
knots (rows of ~11 knots: the ninth and later knots read X), ties of the
bytes, exact knots and their neighbours, f32 and f64, int32 and int64
outputs, out-of-domain lanes."""

import numpy as np
import pytest

from oracle import fs_oracle as orc

pytestmark = pytest.mark.gpu


def _fs():
    import paper_1506_08620_b200 as fs

    return fs


def expected_rows(xs, h, r):
    """uint32[(r >> 5) + 1, 4] = {mask, base, bytes 0-3, bytes 4-7} and the knots per row."""
    t = xs.dtype.type
    p = (t(h) * (xs - xs[0]).astype(xs.dtype)).astype(xs.dtype)
    f = np.floor(p).astype(np.int64)
    assert np.array_equal(f, orc.knot_buckets(xs, h).astype(np.int64))
    byte = np.floor((p - np.floor(p)).astype(xs.dtype) * t(256)).astype(np.uint64)
    words = (r >> 5) + 1
    rows = np.zeros((words, 4), dtype=np.uint64)
    w = f >> 5
    np.bitwise_or.at(rows[:, 0], w, np.uint64(1) << (f & 31).astype(np.uint64))
    base = np.searchsorted(f, np.arange(words, dtype=np.int64) << 5, side="left")
    rows[:, 1] = base
    rank_in_row = np.arange(len(f)) - base[w]
    for col, lo in ((2, 0), (3, 4)):
        sel = (rank_in_row >= lo) & (rank_in_row < lo + 4)
        np.bitwise_or.at(rows[:, col], w[sel], byte[sel] << (8 * (rank_in_row[sel] - lo)).astype(np.uint64))
    return rows.astype(np.uint32), np.bincount(w, minlength=words)


def _buffer_of(prep, ptr):
    return next(b for b in prep.buffers if b.data_ptr() == ptr)


def _queries(xs, h, r, seed, count=400_000):
    t = xs.dtype.type
    rng = np.random.default_rng(seed)
    pick = xs[rng.integers(0, len(xs) - 1, 200_000)]
    near = [pick, np.nextafter(pick, t(-np.inf)), np.nextafter(pick, t(np.inf))]
    width = t(1) / t(h)
    for frac in (1 / 512, 1 / 256, 1 / 100, 1 / 3):
        near += [(pick - t(frac) * width).astype(xs.dtype), (pick + t(frac) * width).astype(xs.dtype)]
    z = np.concatenate(near + [orc.random_queries(xs, count, seed=seed), orc.boundary_probes(xs)[:200_000],
                               orc.bucket_edge_probes(xs, h, r, 100_000, seed=seed + 1)]).astype(xs.dtype)
    return z[(z >= xs[0]) & (z < xs[-1])]


def _partition(fs, name):
    from paper_1506_08620_b200 import workloads

    if name == "cfg5":
        return workloads.knots("cfg5", n1=1_048_577)
    return fs.gen_uniform_gap_partition(1_048_575, 1.0, 5.0, 42, "single" if name == "unif32" else "double")


@pytest.mark.parametrize("name", ["cfg5", "unif32", "unif64"])
def test_rank_rows_for_l2_tables(cuda, name):
    """Neither the directory nor X fits in shared memory: prepare() builds rank
    rows and the search stages nothing.  Rows bit for bit against numpy; the
    uniform-gap arrays put nine and more knots in most rows (X read for those),
    cfg5 about three; answers equal the oracle."""
    fs = _fs()
    from paper_1506_08620_b200 import _lib

    p = _partition(fs, name)
    prep = fs.prepare("direct", p)
    xs = p.values
    idx = prep.structure
    assert prep.plan.sparse_format == _lib.SPARSE_RANK_ROWS and prep.plan.sparse
    pl = prep.placement()
    assert pl["smem_bytes"] == 0 and not pl["smem_sparse"] and not pl["smem_hot"] and pl["l2_directory"] == "rank-rows", pl
    want_rows, per_row = expected_rows(xs, idx.h, idx.r)
    got = _buffer_of(prep, prep.plan.sparse).cpu().numpy().view(np.uint32).reshape(-1, 4)
    assert np.array_equal(got, want_rows)
    if name == "cfg5":
        assert 2.5 < per_row.mean() < 4.5
    else:
        assert per_row.max() > 8 and np.count_nonzero(per_row > 8) > len(per_row) // 2
    z = _queries(xs, idx.h, idx.r, seed=3)
    want = orc.rank_oracle(xs, z)
    assert np.array_equal(fs.run_batch(prep, z), want)
    out32 = np.empty(len(z), dtype=np.int32)
    fs.batch_search(fs.LaneConfig(1, "direct", prep), z, out32)
    assert np.array_equal(out32, want)


def test_rank_rows_rule_switch_and_out_of_domain(cuda):
    """Rows only for tables searched through L2 with enough knot-holding
    buckets; with the knob at 0 the 8-B directory answers the same; out-of-domain
    lanes report the first bad position and fault nothing."""
    fs = _fs()
    from paper_1506_08620_b200 import _lib, batch, workloads

    for p in (workloads.knots("cfg3"), workloads.knots("cfg4"), workloads.knots("cfg5", n1=32769),
              fs.gen_uniform_gap_partition(65535, 1.0, 5.0, 42, "double")):
        assert fs.prepare("direct", p).plan.sparse_format != _lib.SPARSE_RANK_ROWS
    p = fs.gen_uniform_gap_partition(1_048_575, 1.0, 5.0, 7, "double")
    xs = p.values
    prep = fs.prepare("direct", p)
    assert prep.plan.sparse_format == _lib.SPARSE_RANK_ROWS
    z = _queries(xs, prep.structure.h, prep.structure.r, seed=9, count=200_000)
    want = orc.rank_oracle(xs, z)
    assert np.array_equal(fs.run_batch(prep, z), want)
    saved = batch.RANK_ROWS_MIN_KNOT_SHARE
    try:
        batch.RANK_ROWS_MIN_KNOT_SHARE = 0
        plain = fs.prepare("direct", p)
    finally:
        batch.RANK_ROWS_MIN_KNOT_SHARE = saved
    assert not plain.plan.sparse and plain.placement()["smem_bytes"] == 0 and plain.placement()["l2_directory"] == "rank"
    assert np.array_equal(fs.run_batch(plain, z), want)
    tail = np.concatenate([xs[-8:-1], np.nextafter(xs[-8:], -np.inf)])
    tail = tail[(tail >= xs[0]) & (tail < xs[-1])]
    assert np.array_equal(fs.run_batch(prep, tail), orc.rank_oracle(xs, tail))
    for bad in (np.nan, np.inf, -np.inf, xs[0] - 1.0, xs[-1], xs[-1] * 2):
        zz = orc.random_queries(xs, 10_000, seed=5)
        zz[4321] = bad
        zz[7777] = bad
        with pytest.raises(fs.OutOfDomain) as ei:
            fs.run_batch(prep, zz)
        assert ei.value.position == 4321


def test_rank_rows_abi_validation(cuda):
    """fs_build_rank_rows argument checks and validate_plan on a rows plan of the wrong gap."""
    fs = _fs()
    from paper_1506_08620_b200 import _device, _lib

    p = fs.gen_uniform_gap_partition(1_048_575, 1.0, 5.0, 3, "single")
    prep = fs.prepare("direct", p)
    lib = _lib.load()
    n1 = len(p.values)
    x = p.device_values()
    r = prep.structure.r
    h = float(prep.structure.h)
    f = _device.empty(n1, np.uint64)
    scratch = _device.empty((n1 + 15) // 16 * 16, np.uint8)
    rows = _device.empty(16 * ((r >> 5) + 1), np.uint8)
    st = _device.stream_ptr()
    args = (f.data_ptr(), scratch.data_ptr(), rows.data_ptr(), st)
    assert lib.fs_build_rank_rows(_lib.FS_F32, None, n1, h, r, *args) == _lib.FS_INVALID_ARG
    assert lib.fs_build_rank_rows(_lib.FS_F32, x.data_ptr(), n1, h, r, None, scratch.data_ptr(), rows.data_ptr(),
                                  st) == _lib.FS_INVALID_ARG
    assert lib.fs_build_rank_rows(_lib.FS_F32, x.data_ptr(), n1, h, r, f.data_ptr(), None, rows.data_ptr(),
                                  st) == _lib.FS_INVALID_ARG
    assert lib.fs_build_rank_rows(_lib.FS_F32, x.data_ptr(), n1, h, r, f.data_ptr(), scratch.data_ptr(), None,
                                  st) == _lib.FS_INVALID_ARG
    assert lib.fs_build_rank_rows(_lib.FS_F32, x.data_ptr(), n1, h, 1 << 32, *args) == _lib.FS_TOO_LARGE
    assert lib.fs_build_rank_rows(7, x.data_ptr(), n1, h, r, *args) == _lib.FS_INVALID_ARG
    assert lib.fs_build_rank_rows(_lib.FS_F32, x.data_ptr(), n1, h, r, *args) == _lib.FS_OK
    z = orc.random_queries(p.values, 1000, seed=1)
    assert np.array_equal(fs.run_batch(prep, z), orc.rank_oracle(p.values, z))
    prep.plan.q = 2
    with pytest.raises(ValueError):
        fs.run_batch(prep, z)
