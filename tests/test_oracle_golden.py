"""Pin the CPU oracle (oracle/fs_oracle.py) to the reference's own outputs.

Every vector in tests/golden was produced by running the unmodified
reference (tests/golden/make_golden.py); these tests prove the numpy
restatement reproduces them bit for bit, which is what lets the GPU parity
tests use the oracle as their checker.  CPU only.
"""

import numpy as np
import pytest

import golden_data as gd
from oracle import fs_oracle as orc

BUILD = gd.build_cases()
QUERY = gd.query_cases()


def _bits(v):
    v = np.asarray(v)
    return int(v.view(np.uint32 if v.dtype == np.float32 else np.uint64))


@pytest.mark.parametrize("case", BUILD, ids=[c["name"] for c in BUILD])
def test_oracle_build_matches_reference(case):
    xs = gd.knots_for(case)
    if "error" in case:
        with pytest.raises(orc.OracleError) as e:
            orc.compute_h_r(xs, case["qbits"], case["q"])
        assert e.value.kind == case["error"]
        if case["error"] == "not_distinguishable":
            assert e.value.position == case["position"]
        return
    h, r, inc, h0 = orc.compute_h_r(xs, case["qbits"], case["q"])
    assert _bits(h) == case["h_bits"]
    assert r == case["r"]
    assert inc == case["increments"]
    assert _bits(h0) == case["h_start_bits"]
    assert gd.sha(orc.knot_buckets(xs, h)) == case["f_sha"]
    k = orc.build_table(xs, h, r, case["q"])
    assert len(k) == case["k_len"] and k.dtype == np.uint32
    a = gd.arrays()
    assert np.array_equal(k[a[f"{case['name']}/k_sample_pos"]], a[f"{case['name']}/k_sample"])
    if f"{case['name']}/k" in a:
        assert np.array_equal(k, a[f"{case['name']}/k"])
    assert gd.sha(k) == case["k_sha"]
    if "fused_sha" in case:
        assert gd.sha(orc.fused_records(xs, k)) == case["fused_sha"]


@pytest.mark.parametrize("case", QUERY, ids=[c["name"] for c in QUERY])
def test_oracle_answers_match_reference(case):
    xs = gd.knots_for(case)
    z = gd.queries_for(case, xs)
    want = orc.rank_oracle(xs, z)
    gd.check_answers(case, want)
    if len(z) <= 5000:
        gd.check_answers(case, orc.linear_scan_batch(xs, z))


def test_lane_restatements_match_reference_sweeps():
    """Each lane kernel of the restatement equals the reference answers on
    the 1e5-query sweeps (test_acceptance.py:56-63 pins them to the oracle)."""
    for case in gd.query_cases(lambda c: c["name"].startswith("sweep_")):
        xs = gd.knots_for(case)
        z = gd.queries_for(case, xs)
        h, r, _, _ = orc.compute_h_r(xs)
        k = orc.build_table(xs, h, r)
        padded, _, probe = orc.pad_right_pow2(xs)
        tree, depth = orc.eytzinger_layout(xs)
        h2, r2, _, _ = orc.compute_h_r(xs, 32, 2)
        k2 = orc.build_table(xs, h2, r2, 2)
        for got in (
            orc.direct_lanes(xs, h, k, z),
            orc.cache_lanes(xs, h, orc.fused_records(xs, k), z),
            orc.gap2_lanes(xs, h2, k2, z),
            orc.bitset2_lanes(padded, probe, z),
            orc.bitset1_lanes(xs, probe, z),
            orc.bitset3_lanes(xs, probe, z),
            orc.offset_lanes(xs, z),
            orc.eytzinger_lanes(tree, depth, z),
        ):
            gd.check_answers(case, got)


def test_out_of_domain_positions_match_reference():
    a = gd.arrays()
    ood = {c["name"]: c["position"] for c in gd.meta()["out_of_domain"]}
    xs = a["ood/right_endpoint/x"]
    assert orc.first_bad(xs, a["ood/right_endpoint/z"]) == ood["right_endpoint"] == 3
    assert orc.first_bad(xs, a["ood/nan/z"]) == ood["nan"] == 5


def test_batch_port_equals_reference():
    """The CPU-baseline port (reference batch driver restated) is exact."""
    case = next(c for c in QUERY if c["name"] == "sweep_single_4095")
    xs = gd.knots_for(case)
    z = gd.queries_for(case, xs)
    for algo in ("direct", "direct-cache", "direct-gap2", "bitset2"):
        prep = orc.PreparedPort(algo, xs)
        out = np.empty(len(z), dtype=np.int32)
        orc.batch_search_port(prep, z, out, d=4096, threads=4)
        gd.check_answers(case, out)


def test_worked_example_constants():
    """test_direct.py:38-52 / test_acceptance.py:198-217."""
    for dt in (np.float32, np.float64):
        xs = np.array([0.0, 0.5, 0.7, 1.1], dtype=dt)
        h, r, inc, _ = orc.compute_h_r(xs)
        assert h == np.nextafter(dt(5.0), dt(np.inf)) and r == 5 and inc == 0
        assert orc.build_table(xs, h, r).tolist() == [0, 1, 1, 2, 3, 3]
        assert orc.direct_lanes(xs, h, orc.build_table(xs, h, r), np.array([0.6], dtype=dt))[0] == 1
