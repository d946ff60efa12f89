"""Host-side logic of the drop-in API, CPU only: type validation and error
positions (reference pkg/tests/test_partition.py), constants
(test_binsearch.py), advisory estimates (test_direct.py), batch contract
validation (test_batch.py), query coercion, sharding spans, workloads."""

import numpy as np
import pytest

import golden_data as gd
import paper_1506_08620_b200 as fs
from oracle import fs_oracle as orc
from paper_1506_08620_b200 import dist, workloads
from paper_1506_08620_b200.direct import feasibility_threshold
from paper_1506_08620_b200.partition import coerce_queries

# fastsearch/__init__.py:77-123, minus the oracle (linear_scan_oracle*), which
# lives in oracle/ as test infrastructure
REFERENCE_ALL = [
    "ALGORITHMS", "BadMagic", "ChecksumMismatch", "DirectIndex", "EytzingerLayout", "FeasibilityReport",
    "HGrowthStats", "IndexFileError", "InfeasibleError", "LaneConfig", "NonFinite", "NotDistinguishable",
    "NotStrictlyIncreasing", "OffsetConstants", "OutOfDomain", "Overflow", "PartitionError", "PaddedPartition",
    "PreparedKernel", "QueryBatch", "SortedPartition", "TooShort", "TruncatedFile", "VersionMismatch",
    "batch_search", "bitset_search_v1", "bitset_search_v2", "bitset_search_v3", "build", "build_index",
    "classic_search", "closed_form_h_r", "compute_h_r", "direct_search", "direct_search_cache",
    "direct_search_gap2", "direct_search_generic", "eytzinger_search", "feasibility_estimate", "gen_queries",
    "gen_uniform_gap_partition", "memory_cost_estimate", "minimal_index_bytes", "offset_constants",
    "offset_search", "pad_right_pow2", "prepare", "probe_constant", "run_batch", "validate_partition", "with_fused",
]


def test_public_surface_covers_reference():
    missing = [n for n in REFERENCE_ALL if not hasattr(fs, n)]
    assert not missing, missing
    assert fs.ALGORITHMS == ("classic", "bitset1", "bitset2", "bitset3", "offset", "eytzinger", "direct",
                             "direct-gap2", "direct-cache")


class TestValidate:
    def test_accepts_sorted(self):
        p = fs.validate_partition([0, 1, 2, 3])
        assert p.n_intervals == 3 and p.precision == "double"

    @pytest.mark.parametrize("raw,pos", [([0, 1, 1, 3], 2), ([0, 2, 1, 3], 2)])
    def test_not_increasing_position(self, raw, pos):
        with pytest.raises(fs.NotStrictlyIncreasing) as e:
            fs.validate_partition(raw)
        assert e.value.position == pos

    @pytest.mark.parametrize("raw,pos", [([0, np.nan], 1), ([0, 1, np.inf], 2)])
    def test_non_finite_position(self, raw, pos):
        with pytest.raises(fs.NonFinite) as e:
            fs.validate_partition(raw)
        assert e.value.position == pos

    def test_too_short(self):
        with pytest.raises(fs.TooShort):
            fs.validate_partition([1.0])

    def test_precision_inferred_frozen_and_copied(self):
        raw = np.array([0, 1], dtype=np.float32)
        p = fs.validate_partition(raw)
        assert p.precision == "single" and p.values.dtype == np.float32
        with pytest.raises(ValueError):
            p.values[0] = 5.0
        raw[0] = -1.0
        assert p.values[0] == 0.0

    def test_error_hierarchy(self):
        assert issubclass(fs.TooShort, fs.PartitionError) and issubclass(fs.PartitionError, ValueError)
        assert issubclass(fs.NotDistinguishable, fs.InfeasibleError) and issubclass(fs.Overflow, fs.InfeasibleError)
        assert issubclass(fs.OutOfDomain, ValueError)
        assert fs.OutOfDomain(position=3).position == 3


class TestGenerators:
    def test_uniform_gap_matches_oracle_recipe(self):
        for prec, dt in (("single", np.float32), ("double", np.float64)):
            p = fs.gen_uniform_gap_partition(255, 1, 5, seed=7, precision=prec)
            assert np.array_equal(p.values, orc.gen_uniform_gap(255, 1, 5, 7, dt))

    def test_queries_in_domain_and_reproducible(self):
        p = fs.gen_uniform_gap_partition(64, 1, 5, seed=5, precision="single")
        a = fs.gen_queries(p, 1000, seed=6)
        b = fs.gen_queries(p, 1000, seed=6)
        assert np.array_equal(a.values, b.values)
        assert ((a.values >= p.x0) & (a.values < p.xn)).all()
        assert np.array_equal(a.values, orc.random_queries(p.values, 1000, 6))
        with pytest.raises(ValueError):
            fs.gen_queries(p, 0, seed=1)

    def test_generator_validation(self):
        with pytest.raises(ValueError):
            fs.gen_uniform_gap_partition(1, 1, 5, seed=0)
        with pytest.raises(ValueError):
            fs.gen_uniform_gap_partition(10, 5, 1, seed=0)


class TestConstants:
    @pytest.mark.parametrize("n,f,s,j", [(7, 4, 4, 3), (1, 1, 1, 1), (14, 7, 8, 3)])
    def test_offset_constants(self, n, f, s, j):
        c = fs.offset_constants(n)
        assert (c.F, c.S, c.J) == (f, s, j)

    def test_offset_invariants(self):
        for n in range(1, 200):
            c = fs.offset_constants(n)
            assert c.F + c.S == n + 1 and 2 ** c.J <= n + 1 < 2 ** (c.J + 1)

    def test_probe_constant(self):
        assert fs.probe_constant(8) == 8 and fs.probe_constant(9) == 8 and fs.probe_constant(1) == 1
        with pytest.raises(ValueError):
            fs.probe_constant(0)


class TestAdvisory:
    """test_direct.py:132-136, 281-316 (host float64 planning arithmetic)."""

    def test_thresholds(self):
        assert feasibility_threshold("single", 32) == 2.0 ** -23
        assert feasibility_threshold("double", 32) == 2.0 ** -32
        assert feasibility_threshold("double", 64) == 2.0 ** -51

    def test_margin_and_collision_advice(self):
        rep = fs.feasibility_estimate(fs.validate_partition(np.array([0, 1, 2, 3], dtype=np.float32)))
        assert rep.feasible and rep.margin == pytest.approx((1 / 3) / 2 ** -23)
        p = fs.validate_partition(np.array([-1e9, 0.0, 1.0], dtype=np.float32))
        assert not fs.feasibility_estimate(p).feasible and fs.feasibility_estimate(p, q=2).feasible

    def test_closed_form_and_memory(self):
        p = fs.validate_partition([0.0, 0.5, 0.7, 1.1])
        h, r = fs.closed_form_h_r(p)
        assert r == 7 and h == pytest.approx(6.36, abs=0.01)
        assert fs.memory_cost_estimate(p, 4) == 24
        assert fs.minimal_index_bytes(200) == 1 and fs.minimal_index_bytes(70_000) == 4
        assert fs.minimal_index_bytes(65_536) == 2 and fs.minimal_index_bytes(2 ** 40) == 8


class TestBatchContract:
    def test_lane_width_validated(self):
        with pytest.raises(ValueError):
            fs.LaneConfig(d=0, kernel="direct", structure=None)

    def test_unknown_algorithm(self):
        with pytest.raises(ValueError):
            fs.prepare("fibonacci", fs.validate_partition([0.0, 1.0]))

    def test_threads(self, monkeypatch):
        monkeypatch.setenv("FASTSEARCH_THREADS", "3")
        assert fs.resolve_threads(None) == 3 and fs.resolve_threads(2) == 2
        monkeypatch.delenv("FASTSEARCH_THREADS")
        assert fs.resolve_threads(None) == 1
        with pytest.raises(ValueError):
            fs.resolve_threads(0)


class TestCoercion:
    def test_same_dtype_is_untouched(self):
        z = np.array([0.5, 1.5], dtype=np.float32)
        assert coerce_queries(z, np.dtype(np.float32)) is z

    def test_wider_queries_keep_exact_answers(self):
        """float64 queries on a float32 partition: rounding toward -inf keeps
        max{i : X_i <= z} exact (and the domain test) for every query."""
        xs = orc.gen_uniform_gap(300, 1, 5, 3, np.float32)
        rng = np.random.default_rng(0)
        z64 = rng.uniform(float(xs[0]), float(xs[-1]), 200_000)
        z64 = np.concatenate([z64, xs[:-1].astype(np.float64), np.nextafter(xs[1:].astype(np.float64), -np.inf)])
        zc = coerce_queries(z64, np.dtype(np.float32))
        assert zc.dtype == np.float32
        exact = np.searchsorted(xs.astype(np.float64), z64, side="right") - 1
        assert np.array_equal(orc.rank_oracle(xs, zc), exact)

    def test_longdouble_and_large_integers_round_down(self):
        """Inputs more precise than the partition (longdouble, integers above
        2^53) round toward -inf too: a value just above a knot's predecessor
        never rounds up across the knot (exact answers, no false
        OutOfDomain just below X_N)."""
        one = np.longdouble(1)
        eps = np.longdouble(2) ** -60
        z = np.array([one - eps, one + eps, np.longdouble(2) - eps], dtype=np.longdouble)
        zc = coerce_queries(z, np.dtype(np.float64))
        assert zc[0] < 1.0 and zc[1] == 1.0 and zc[2] < 2.0
        xs = np.array([0.0, 1.0, 2.0])
        assert orc.first_bad(xs, zc) is None
        assert orc.rank_oracle(xs, zc).tolist() == [0, 1, 1]
        big = np.array([2**53 + 1, 2**62 + 1, -(2**53) - 1, 7], dtype=np.int64)
        zb = coerce_queries(big, np.dtype(np.float64))
        assert [int(v) for v in zb] == [2**53, 2**62, -(2**53) - 2, 7]
        z32 = coerce_queries(np.array([16777217, 3], dtype=np.int64), np.dtype(np.float32))
        assert z32.tolist() == [16777216.0, 3.0]

    def test_narrower_float_is_exact(self):
        z = np.array([0.5, 65504.0], dtype=np.float16)
        assert coerce_queries(z, np.dtype(np.float32)).tolist() == [0.5, 65504.0]

    def test_domain_preserved(self):
        xs = np.array([0.0, 1.0, 2.0], dtype=np.float32)
        z = np.array([np.nextafter(2.0, -np.inf), 2.0, -1e-300, np.nan])
        zc = coerce_queries(z, np.dtype(np.float32))
        assert orc.first_bad(xs, zc[:1]) is None
        assert orc.first_bad(xs, zc) == 1
        assert orc.first_bad(xs, zc[2:]) == 0


class TestShardSpans:
    @pytest.mark.parametrize("m", [0, 1, 3, 4, 17, 4001, 1 << 20])
    @pytest.mark.parametrize("world", [1, 2, 3, 4, 8])
    def test_spans_partition_the_batch(self, m, world):
        spans = [dist.shard_span(m, r, world) for r in range(world)]
        assert spans[0][0] == 0 and spans[-1][1] == m
        for (a, b), (c, _) in zip(spans, spans[1:]):
            assert b == c and a <= b
        for a, _ in spans:
            assert a % 4 == 0

    def test_invalid(self):
        with pytest.raises(ValueError):
            dist.shard_span(10, 2, 2)


class TestWorkloads:
    def test_config_facts(self):
        """R and h of the configs (pinned by golden)."""
        b = {c["name"]: c for c in gd.build_cases(lambda c: c["name"].startswith("cfg"))}
        assert b["cfg3_s0"]["r"] == 8159 and b["cfg4"]["r"] == 7_005_360
        assert [b[f"cfg1_s{s}"]["r"] for s in range(3)] == [485_920, 457_601, 837_857]
        assert b["cfg2_s0"]["r"] == 24_753_039
        assert b["cfg5_1048577_unfiltered"]["error"] == "overflow"

    def test_cfg2_exact_knot_queries(self):
        p = workloads.knots("cfg2", seed=0)
        z = workloads.queries_host("cfg2", p, 100_000, seed=3)
        hits = np.isin(z, p.values[:-1]).sum()
        assert hits >= 1000

    def test_cfg4_clustered_half(self):
        p = workloads.knots("cfg4")
        z = workloads.queries_host("cfg4", p, 200_000, seed=3)
        dense = (z < workloads.cfg4_dense_top(p)).mean()
        assert 0.49 < dense < 0.52
        assert ((z >= p.x0) & (z < p.xn)).all()

    def test_cfg5_min_gap(self):
        p = workloads.knots("cfg5", n1=32769)
        assert np.diff(p.values).min() >= 1e-7 and len(p.values) == 32769


def test_eytzinger_in_order_host_helper():
    from paper_1506_08620_b200.eytzinger import EytzingerLayout, in_order

    xs = orc.gen_uniform_gap(20, 1, 5, 20, np.float64)
    tree, depth = orc.eytzinger_layout(xs)
    lay = EytzingerLayout(tree_dev=None, L=depth, source=None, _host={"tree": tree})
    flat = in_order(lay)
    assert np.array_equal(flat[:20], xs) and (flat[20:] == xs[-1]).all()
