"""GPU tests of the rank-directory hot window (fs_build_hot_window +
HotRankProbe): for a skewed table too large for shared memory, the
knot-densest directory window and its knots are staged in shared memory and
every other query gathers through L2.  Answers must equal the oracle
(batch.py:315-317) on both sides of every window edge."""

import numpy as np
import pytest

from oracle import fs_oracle as orc

pytestmark = pytest.mark.gpu


def _fs():
    import paper_1506_08620_b200 as fs

    return fs


@pytest.fixture(autouse=True)
def _no_zoned():
    """These skewed tables take zoned records by default
    (tests/test_gpu_zoned.py); the hot window is tested with zoning off."""
    from paper_1506_08620_b200 import batch

    keep = batch.ZONED
    batch.ZONED = False
    yield
    batch.ZONED = keep



def _edge_queries(xs, h, words):
    """Queries in the buckets around directory words `words` (32 buckets
    each): first and last bucket of each word, +-1 ulp around them."""
    t = xs.dtype.type
    out = []
    for w in words:
        for j in (32 * w - 1, 32 * w, 32 * w + 1, 32 * w + 31, 32 * w + 32):
            if j < 0:
                continue
            v = t(xs[0] + t(j) / t(h))
            out += [np.nextafter(v, t(-np.inf)), v, np.nextafter(v, t(np.inf))]
    z = np.array(out, dtype=xs.dtype)
    return z[(z >= xs[0]) & (z < xs[-1])]


@pytest.mark.parametrize("dtype", [np.float32, np.float64])
def test_hot_window_skewed_table(cuda, dtype):
    """cfg4-like geometric knots (dense start, sparse tail; directory larger
    than shared memory): the window is chosen, and answers equal the oracle
    and the L2-only plan for uniform, clustered, window-edge and knot-edge
    queries."""
    fs = _fs()
    gaps = 1e-4 * 1.00012 ** np.arange(60_000, dtype=np.float64)  # R ~ 11 M: directory > smem, skewed
    xs = np.concatenate([[0.0], np.cumsum(gaps)]).astype(dtype)
    xs = np.unique(xs)
    p = fs.validate_partition(xs)
    hot = fs.prepare("direct", p)
    cold = fs.prepare("direct", p, hot_window=False)
    assert hot.placement()["smem_hot"], (hot.placement(), hot.structure.r)
    assert not cold.placement()["smem_hot"]
    plan = hot.plan
    assert plan.hot_words > 0 and plan.hot_knots > 0
    idx = hot.structure
    w0, nw, t0, nt = plan.hot_word0, plan.hot_words, plan.hot_knot0, plan.hot_knots
    rng = np.random.default_rng(3)
    dense_top = xs[min(len(xs) - 1, t0 + nt)]
    z = np.concatenate([
        orc.random_queries(xs, 300_000, seed=1),
        rng.uniform(xs[0], dense_top, 300_000).astype(dtype),
        _edge_queries(xs, idx.h, [w0 - 1, w0, w0 + 1, w0 + nw - 1, w0 + nw, w0 + nw + 1]),
        xs[max(0, t0 - 2): t0 + 2], xs[t0 + nt - 2: t0 + nt + 2],
        orc.boundary_probes(xs),
    ]).astype(dtype)
    z = z[(z >= xs[0]) & (z < xs[-1])]
    want = orc.rank_oracle(xs, z)
    got = fs.run_batch(hot, z)
    assert np.array_equal(got, want)
    assert np.array_equal(fs.run_batch(cold, z), want)
    out32 = np.empty(len(z), dtype=np.int32)
    fs.batch_search(fs.LaneConfig(1, "direct", hot), z, out32)
    assert np.array_equal(out32, want)


def test_hot_window_rejected_for_uniform_tables(cuda):
    """A uniform table (cfg5 N+1 = 2^20 + 1) gains nothing from a window:
    the density rule keeps the whole directory in L2."""
    fs = _fs()
    from paper_1506_08620_b200 import workloads

    p = workloads.knots("cfg5", n1=1_048_577)
    prep = fs.prepare("direct", p)
    assert not prep.placement()["smem_hot"]
    z = workloads.queries_host("cfg5", p, 500_000, seed=9)
    assert np.array_equal(fs.run_batch(prep, z), orc.rank_oracle(p.values, z))


def test_hot_window_cfg4_out_of_domain(cuda):
    """cfg4 with its window: first bad position reported, nothing written."""
    fs = _fs()
    from paper_1506_08620_b200 import workloads

    p = workloads.knots("cfg4")
    prep = fs.prepare("direct", p)
    assert prep.placement()["smem_hot"]
    z = workloads.queries_host("cfg4", p, 200_003, seed=2)
    want = orc.rank_oracle(p.values, z)
    assert np.array_equal(fs.run_batch(prep, z), want)
    for bad in (np.nan, np.inf, p.values[-1], np.float32(-1.0)):
        zb = z.copy()
        zb[123_457] = bad
        out = np.full(len(zb), -5, dtype=np.int32)
        with pytest.raises(fs.OutOfDomain) as e:
            fs.batch_search(fs.LaneConfig(1, "direct", prep), zb, out)
        assert e.value.position == 123_457
        assert (out == -5).all()
