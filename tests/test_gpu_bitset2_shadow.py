"""GPU tests of bitset2's f32 shadow keys for f64 partitions (Bitset2Probe::
kShadow: staged levels compared on RN(key) / RN(z), every right turn
validated by one exact f64 compare, an exact re-descent when it fails).
Answers must equal the oracle (binsearch.py:72-86 semantics) where the
shadow keys tie: queries at and one ulp around every knot, and knots closer
than the f32 resolution (whole runs of equal shadow keys)."""

import numpy as np
import pytest

from oracle import fs_oracle as orc

pytestmark = pytest.mark.gpu


def _fs():
    import paper_1506_08620_b200 as fs

    return fs


def _around_knots(xs):
    z = np.concatenate([xs, np.nextafter(xs, -np.inf), np.nextafter(xs, np.inf),
                        np.nextafter(np.nextafter(xs, -np.inf), -np.inf)])
    return z[(z >= xs[0]) & (z < xs[-1])]


@pytest.mark.parametrize("n1", [8193, 32769, 1 << 18])
def test_shadow_ties_at_knots(cuda, n1):
    """Sorted U[0, 1) knots (p = 13, 15, 18: shadow levels in smem, global
    levels below for the larger two): queries at and around every knot --
    each ties with its knot's shadow key -- plus random ones."""
    fs = _fs()
    rng = np.random.default_rng(n1)
    xs = np.unique(rng.uniform(0.0, 1.0, n1 + n1 // 4))[:n1]
    p = fs.validate_partition(xs)
    prep = fs.prepare("bitset2", p)
    assert prep.placement()["smem_top"] or prep.placement()["smem_x"]
    z = np.concatenate([_around_knots(xs), orc.random_queries(xs, 200_000, seed=1)])
    assert np.array_equal(fs.run_batch(prep, z), orc.rank_oracle(xs, z))


def test_shadow_keys_below_f32_resolution(cuda):
    """Knots spaced 1e-12 around 1.0 (every shadow key rounds to 1.0f) and
    spaced 1e-3 elsewhere: runs of equal shadow keys, ties at every level."""
    fs = _fs()
    dense = 1.0 + 1e-12 * np.arange(9000)
    sparse = np.linspace(-5.0, 0.99, 4000)
    tail = np.linspace(1.5, 9.0, 4000)
    xs = np.unique(np.concatenate([sparse, dense, tail]))
    p = fs.validate_partition(xs)
    assert p.n_intervals.bit_length() >= 13
    prep = fs.prepare("bitset2", p)
    rng = np.random.default_rng(2)
    z = np.concatenate([_around_knots(xs), rng.uniform(1.0, 1.0 + 9e-9, 100_000),
                        orc.random_queries(xs, 100_000, seed=3), [-0.0, 0.0]])
    z = z[(z >= xs[0]) & (z < xs[-1])]
    want = orc.rank_oracle(xs, z)
    for odt in (np.int32, np.int64):
        out = np.empty(len(z), dtype=odt)
        fs.batch_search(fs.LaneConfig(1, "bitset2", prep), z, out)
        assert np.array_equal(out, want), odt


def test_shadow_signed_zero_and_negative_knots(cuda):
    """Negative knots, -0.0 as a knot, and +0.0 / -0.0 queries: the shadow
    compare and the exact check agree with IEEE (-0.0 == +0.0)."""
    fs = _fs()
    xs = np.concatenate([np.linspace(-1.0, -1e-9, 6000), [-0.0], np.linspace(1e-9, 1.0, 6000)])
    p = fs.validate_partition(xs)
    prep = fs.prepare("bitset2", p)
    z = np.concatenate([_around_knots(xs), [0.0, -0.0, 5e-324, -5e-324]])
    z = z[(z >= xs[0]) & (z < xs[-1])]
    assert np.array_equal(fs.run_batch(prep, z), orc.rank_oracle(xs, z))
