"""Property-based parity on adversarial partitions (hypothesis).

CPU: the oracle restatement equals the REFERENCE itself (run from
/root/reference/pkg/src when present in the build container; skipped
elsewhere) for compute_h_r (raw bits of h, r, growth increments, error kind
and position) and the K table -- including layouts that drive the H growth
loop, near-collisions, subnormal gaps and Overflow.
GPU: the CUDA build and all nine search kernels equal the oracle bit for bit.
"""

import sys
from pathlib import Path

import numpy as np
import pytest
from hypothesis import HealthCheck, given, settings
from hypothesis import strategies as st

from oracle import fs_oracle as orc
from strategies import big_partitions, partitions

REF = Path("/root/reference/pkg/src")


def _bits(v):
    v = np.asarray(v)
    return int(v.view(np.uint32 if v.dtype == np.float32 else np.uint64))


def _oracle_build(xs, q):
    try:
        h, r, inc, h0 = orc.compute_h_r(xs, 32, q)
        return ("ok", _bits(h), r, inc, _bits(h0))
    except orc.OracleError as e:
        return (e.kind, e.position if e.kind == "not_distinguishable" else None)


@pytest.fixture(scope="module")
def reference():
    if not REF.exists():
        pytest.skip("reference package not present (only in the build container)")
    sys.path.insert(0, str(REF))
    from fastsearch import direct, errors, partition

    return direct, errors, partition


@settings(max_examples=300, deadline=None, suppress_health_check=[HealthCheck.too_slow])
@given(xs=partitions(), q=st.sampled_from([1, 2]))
def test_oracle_build_equals_reference(reference, xs, q):
    direct, errors, partition = reference
    p = partition.validate_partition(xs)
    try:
        h, r, stats = direct.compute_h_r(p, q=q)
        want = ("ok", _bits(h), r, stats.increments)
    except errors.NotDistinguishable as e:
        want = ("not_distinguishable", e.position)
    except errors.Overflow:
        want = ("overflow", None)
    got = _oracle_build(xs, q)
    assert got[: len(want)] == want
    if want[0] == "ok" and r < 200_000:
        k_ref = direct.build_index(p, h, r, q=q).k
        assert np.array_equal(orc.build_table(xs, h, r, q), k_ref)


@pytest.mark.gpu
@settings(max_examples=int(__import__("os").environ.get("FSG_SMALL_EXAMPLES", "400")), deadline=None, suppress_health_check=[HealthCheck.too_slow,
                                                                   HealthCheck.function_scoped_fixture])
@given(xs=partitions())
def test_gpu_equals_oracle(cuda, xs):
    import paper_1506_08620_b200 as fs

    p = fs.validate_partition(xs)
    z = np.unique(np.concatenate([orc.boundary_probes(xs), orc.random_queries(xs, 4000, seed=len(xs))]))
    want = orc.rank_oracle(xs, z)
    for q in (1, 2):
        ob = _oracle_build(xs, q)
        if ob[0] == "ok":
            h, r, st = fs.compute_h_r(p, q=q)
            assert (_bits(h), r, st.increments) == ob[1:4]
        elif ob[0] == "not_distinguishable":
            with pytest.raises(fs.NotDistinguishable) as e:
                fs.compute_h_r(p, q=q)
            assert e.value.position == ob[1]
        else:
            with pytest.raises(fs.Overflow):
                fs.compute_h_r(p, q=q)
    for algo in fs.ALGORITHMS:
        try:
            prep = fs.prepare(algo, p)
        except fs.InfeasibleError:
            continue
        if algo.startswith("direct") and prep.structure.r > 50_000_000:
            continue
        got = fs.run_batch(prep, z)
        assert np.array_equal(got, want), algo


@pytest.mark.gpu
@settings(max_examples=int(__import__("os").environ.get("FSG_BIG_EXAMPLES", "24")), deadline=None, suppress_health_check=[HealthCheck.too_slow,
                                                                  HealthCheck.function_scoped_fixture])
@given(xs=big_partitions())
def test_gpu_big_tables_equal_oracle(cuda, xs):
    """Large partitions and batches (4M queries + knot neighbourhoods): the
    big-table layouts of direct, direct-cache, direct-gap2 and bitset2 equal
    the oracle."""
    import paper_1506_08620_b200 as fs

    p = fs.validate_partition(xs)
    rng = np.random.default_rng(len(xs))
    pick = xs[rng.integers(0, len(xs) - 1, 20_000)]
    t = xs.dtype.type
    near = np.concatenate([pick, np.nextafter(pick, t(np.inf)), np.nextafter(pick, t(-np.inf))])
    near = near[(near >= xs[0]) & (near < xs[-1])]
    z = np.concatenate([orc.random_queries(xs, 1 << 22, seed=len(xs) + 1), near])
    want = orc.rank_oracle(xs, z)
    for algo in ("direct", "direct-cache", "direct-gap2", "bitset2"):
        try:
            prep = fs.prepare(algo, p)
        except fs.InfeasibleError:
            continue
        got = fs.run_batch(prep, z)
        bad = np.flatnonzero(got != want)
        assert len(bad) == 0, (algo, len(xs), xs.dtype.name, int(len(bad)), int(bad[0]), float(z[bad[0]]),
                               int(got[bad[0]]), int(want[bad[0]]), prep.placement(), int(getattr(prep.structure, "r", 0)))
    # each sparse layout forced on its own (group records also past the
    # planner's slow-path bound): the same answers whenever it fits
    from paper_1506_08620_b200 import batch

    keep = batch.SPARSE_FORMATS, batch.SPARSE_RECORDS_MAX_PAST_SIXTH_PPM, batch.SPARSE_RECORDS8_MAX_PAST_PPM
    keep_cw = batch.COUNT_WORDS_MAX_RARE_PPM, batch.COUNT_WORDS_MAX_L2_XREAD_PPM, batch.COUNT_WORDS_MAX_XREAD_PPM
    try:
        for fmt in (("count-words",), ("records",), ("records8",), ("records12",), ("records8x3",), ("two-level",)):
            batch.SPARSE_FORMATS = fmt
            batch.SPARSE_RECORDS_MAX_PAST_SIXTH_PPM = batch.SPARSE_RECORDS8_MAX_PAST_PPM = 10**6
            batch.COUNT_WORDS_MAX_RARE_PPM = batch.COUNT_WORDS_MAX_L2_XREAD_PPM = 10**6  # past the scan-path bound too
            batch.COUNT_WORDS_MAX_XREAD_PPM = 10**6
            try:
                prep = fs.prepare("direct", p)
            except fs.InfeasibleError:
                break
            if prep.placement()["sparse_format"] != fmt[0]:
                continue
            got = fs.run_batch(prep, z)
            bad = np.flatnonzero(got != want)
            assert len(bad) == 0, (fmt, len(xs), xs.dtype.name, int(len(bad)), int(bad[0]), prep.placement(),
                                   prep.plan.sparse_shift, prep.plan.sparse_ndense)
    finally:
        batch.SPARSE_FORMATS, batch.SPARSE_RECORDS_MAX_PAST_SIXTH_PPM, batch.SPARSE_RECORDS8_MAX_PAST_PPM = keep
        batch.COUNT_WORDS_MAX_RARE_PPM, batch.COUNT_WORDS_MAX_L2_XREAD_PPM, batch.COUNT_WORDS_MAX_XREAD_PPM = keep_cw
    # zoned records and the hot window are alternatives for skewed tables: when
    # the planner took one, the other (zoning off) must answer the same
    if fs.prepare("direct", p).placement()["sparse_format"] == "zoned":
        keep_z = batch.ZONED
        batch.ZONED = False
        try:
            prep = fs.prepare("direct", p)
        finally:
            batch.ZONED = keep_z
        assert prep.placement()["sparse_format"] != "zoned"
        assert np.array_equal(fs.run_batch(prep, z), want), ("zoning off", len(xs), prep.placement())
