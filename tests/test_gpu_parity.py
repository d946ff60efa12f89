"""GPU parity: the CUDA build and search paths against the reference's own
outputs (golden fixtures) and the pinned oracle, through the drop-in API
(which calls the C-ABI in include/fsgpu.h).  Bit-exact: h (raw bits), r,
growth increments, K, fused records, every query answer."""

import numpy as np
import pytest

import golden_data as gd
from oracle import fs_oracle as orc

pytestmark = pytest.mark.gpu

BUILD = gd.build_cases()
QUERY = gd.query_cases()


def _bits(v):
    v = np.asarray(v)
    return int(v.view(np.uint32 if v.dtype == np.float32 else np.uint64))


@pytest.mark.parametrize("case", BUILD, ids=[c["name"] for c in BUILD])
def test_gpu_build_matches_reference(cuda, case):
    import paper_1506_08620_b200 as fs

    xs = gd.knots_for(case)
    p = fs.validate_partition(xs)
    if "error" in case:
        exc = fs.NotDistinguishable if case["error"] == "not_distinguishable" else fs.Overflow
        with pytest.raises(exc) as e:
            fs.compute_h_r(p, qbits=case["qbits"], q=case["q"])
        if case["error"] == "not_distinguishable":
            assert e.value.position == case["position"]
        return
    h, r, st = fs.compute_h_r(p, qbits=case["qbits"], q=case["q"])
    assert h.dtype == xs.dtype
    assert _bits(h) == case["h_bits"], (float(h), case["h_repr"])
    assert r == case["r"]
    assert st.increments == case["increments"]
    assert gd.sha(fs.knot_buckets(p, h)) == case["f_sha"]
    if case["k_len"] > 1_200_000_000:
        pytest.skip("table larger than the GPU test budget")
    idx = fs.build_index(p, h, r, q=case["q"], qbits=case["qbits"])
    a = gd.arrays()
    name = case["name"]
    import torch

    kd = idx.k_dev.view(torch.int32)
    pos = a[f"{name}/k_sample_pos"]
    sample = kd[torch.from_numpy(pos).to(kd.device)].cpu().numpy().view(np.uint32)
    assert np.array_equal(sample, a[f"{name}/k_sample"])
    assert gd.sha(idx.k) == case["k_sha"]
    if f"{name}/k" in a:
        assert np.array_equal(idx.k, a[f"{name}/k"])
        assert idx.k.dtype == np.uint32
    if "fused_sha" in case and case["k_len"] <= 1 << 22:
        fidx = fs.with_fused(idx, p)
        assert gd.sha(fidx.fused) == case["fused_sha"]


ALGOS = ("classic", "bitset1", "bitset2", "bitset3", "offset", "eytzinger", "direct", "direct-gap2", "direct-cache")


@pytest.mark.parametrize("case", QUERY, ids=[c["name"] for c in QUERY])
def test_gpu_search_matches_reference(cuda, case):
    import paper_1506_08620_b200 as fs

    xs = gd.knots_for(case)
    z = gd.queries_for(case, xs)
    p = fs.validate_partition(xs)
    algos = ALGOS if len(xs) <= 70_000 else ("bitset2", "direct", "direct-cache")
    ran = 0
    for algo in algos:
        try:
            prep = fs.prepare(algo, p)
        except fs.InfeasibleError:
            continue
        got = fs.run_batch(prep, z, d=65536)
        gd.check_answers(case, got)
        ran += 1
    assert ran >= 1


@pytest.mark.parametrize("algo", ["direct", "bitset2", "direct-cache"])
@pytest.mark.parametrize("prec", ["single", "double"])
def test_gpu_global_placement_parity(cuda, algo, prec):
    """Force the L2-gather code path (no smem staging) on small tables."""
    import paper_1506_08620_b200 as fs

    case = next(c for c in QUERY if c["name"] == f"sweep_{prec}_4095")
    xs = gd.knots_for(case)
    z = gd.queries_for(case, xs)
    prep = fs.prepare(algo, fs.validate_partition(xs))
    prep.plan.smem_policy = 1
    assert prep.placement()["smem_bytes"] == 0
    gd.check_answers(case, fs.run_batch(prep, z))
    prep.plan.smem_policy = 0
    gd.check_answers(case, fs.run_batch(prep, z))


def test_gpu_out_of_domain_positions(cuda):
    import paper_1506_08620_b200 as fs

    a = gd.arrays()
    xs = a["ood/right_endpoint/x"]
    p = fs.validate_partition(xs)
    for algo in ALGOS:
        prep = fs.prepare(algo, p)
        out = np.full(10, -7, dtype=np.int64)
        with pytest.raises(fs.OutOfDomain) as e:
            fs.batch_search(fs.LaneConfig(2, algo, prep), a["ood/right_endpoint/z"], out)
        assert e.value.position == 3
        assert (out == -7).all(), "nothing may be written on OutOfDomain"
        with pytest.raises(fs.OutOfDomain) as e:
            fs.run_batch(prep, a["ood/nan/z"], d=4)
        assert e.value.position == 5


def test_gpu_worked_example(cuda):
    """test_direct.py:38-52,140-145,188-193; test_acceptance.py:198-217."""
    import paper_1506_08620_b200 as fs

    for dt in (np.float32, np.float64):
        p = fs.validate_partition(np.array([0.0, 0.5, 0.7, 1.1], dtype=dt))
        h, r, st = fs.compute_h_r(p)
        assert h == np.nextafter(dt(5.0), dt(np.inf)) and r == 5 and st.increments == 0
        assert st.growth_total == 0.0
        idx, _ = fs.build(p)
        assert idx.k.tolist() == [0, 1, 1, 2, 3, 3]
        assert fs.direct_search(idx, p, dt(0.6)) == 1
    p = fs.validate_partition([0.0, 0.5, 0.7, 1.1])
    idx, _ = fs.build(p, fused=True)
    assert fs.direct_search(idx, p, 0.6) == 1
    assert fs.direct_search(idx, p, 0.0) == 0
    assert fs.direct_search(idx, p, np.nextafter(1.1, -np.inf)) == 2
    assert fs.direct_search_cache(idx, 0.6) == 1
    for fn in (lambda z: fs.direct_search(idx, p, z), lambda z: fs.direct_search_cache(idx, z)):
        with pytest.raises(fs.OutOfDomain):
            fn(1.1)
        with pytest.raises(fs.OutOfDomain):
            fn(-0.5)


def test_gpu_oracle_on_random_configs(cuda):
    """Config query streams at moderate M vs the rank oracle, int32 and int64 out."""
    import paper_1506_08620_b200 as fs
    from paper_1506_08620_b200 import workloads

    for name, kw in (("cfg1", {}), ("cfg3", {}), ("cfg4", {}), ("cfg2", {}), ("cfg5", {"n1": 1025})):
        p = workloads.knots(name, **kw)
        z = workloads.queries_host(name, p, 1_000_003, seed=5)
        want = orc.rank_oracle(p.values, z)
        for algo in ("direct", "bitset2", "direct-cache"):
            prep = fs.prepare(algo, p)
            for odt in (np.int32, np.int64):
                out = np.empty(len(z), dtype=odt)
                fs.batch_search(fs.LaneConfig(65536, algo, prep), z, out)
                assert np.array_equal(out, want), (name, algo, odt)
