"""The count directory of gap-q tables (fs_build_countdir) and the gap-q
fall-back for infeasible gap-1 layouts (prepare_with_fallback,
PAPER.md:754-762).  Directory words are checked bit for bit against a numpy
construction from the oracle's knot buckets; every answer against the
oracle (and the reference's generic lane restated, oracle.generic_lanes)."""

import numpy as np
import pytest

from oracle import fs_oracle as orc

pytestmark = pytest.mark.gpu


def _fs():
    import paper_1506_08620_b200 as fs

    return fs


def _numpy_countdir(xs, h, r, q):
    """{counts, base} words from the oracle's knot buckets (direct.py:194-197)."""
    f = orc.knot_buckets(xs, h).astype(np.int64)
    b = 2 if q <= 3 else 4
    lg = 4 if q <= 3 else 3
    words = (r >> lg) + 1
    counts = np.zeros(words, dtype=np.uint64)
    np.add.at(counts, f >> lg, np.left_shift(np.uint64(1), (b * (f & ((1 << lg) - 1))).astype(np.uint64)))
    base = np.searchsorted(f, np.arange(words, dtype=np.int64) << lg, side="left")
    return counts.astype(np.uint32), base.astype(np.uint32)


def _clustered(q, dtype, seed, n=3000):
    """Knots in clusters of exactly q tiny steps: the largest gap a gap-q
    certificate allows puts q knots into one bucket."""
    rng = np.random.default_rng(seed)
    starts = np.cumsum(rng.uniform(1.0, 2.0, n // q))
    xs = (starts[:, None] + np.arange(q)[None, :] * 1e-3).ravel()
    return xs.astype(dtype)


CASES = [(q, prec, kind) for q in (2, 3, 4, 7, 15) for prec in ("single", "double") for kind in ("uniform", "cluster")]


@pytest.mark.parametrize("q,prec,kind", CASES)
def test_countdir_words_and_answers(cuda, q, prec, kind):
    import torch

    fs = _fs()
    dtype = np.float32 if prec == "single" else np.float64
    xs = orc.gen_uniform_gap(4001, 1, 5, q, dtype) if kind == "uniform" else _clustered(q, dtype, q)
    p = fs.validate_partition(xs)
    prep = fs.prepare_direct_gap(p, q)
    assert prep.algorithm == "direct-generic" and prep.structure.q == q
    h, r, inc, _ = orc.compute_h_r(xs, q=q)
    assert prep.structure.h == h and prep.structure.r == r
    d = prep.buffers[-1].view(torch.int32).cpu().numpy().view(np.uint32).reshape(-1, 2)
    counts, base = _numpy_countdir(xs, h, r, q)
    assert np.array_equal(d[:, 0], counts) and np.array_equal(d[:, 1], base)
    if kind == "cluster":
        b = 2 if q <= 3 else 4
        fields = (counts[:, None] >> (b * np.arange(32 // b)[None, :])) & ((1 << b) - 1)
        assert fields.max() == q  # buckets holding the full q knots are exercised
    z = np.concatenate([orc.random_queries(xs, 200_000, seed=q), orc.boundary_probes(xs),
                        orc.bucket_edge_probes(xs, h, r, 50_000, seed=q + 1)])
    want = orc.rank_oracle(xs, z)
    k = orc.build_table(xs, h, r, q=q)
    assert np.array_equal(orc.generic_lanes(xs, h, k, q, z), want)  # the reference's lane, restated
    assert np.array_equal(fs.run_batch(prep, z), want)
    zt = torch.from_numpy(z).cuda()
    for odt in (torch.int32, torch.int64):
        out = torch.empty(len(z), dtype=odt, device=cuda)
        fs.batch_search(fs.LaneConfig(4, "direct-generic", prep), zt, out)
        assert np.array_equal(out.cpu().numpy(), want)
    plan = prep.plan
    saved = plan.smem_policy
    plan.smem_policy = 1  # directory and X through L2
    try:
        assert not prep.placement()["smem_table"]
        assert np.array_equal(fs.run_batch(prep, z), want)
    finally:
        plan.smem_policy = saved


def test_gap_fallback_for_the_overflow_instance(cuda):
    """configs[4]'s unfiltered 2^20+1 draw overflows at gap 1; the fall-back
    takes the smallest gap whose count directory stays L2-resident (q = 3:
    ~29 MB) and answers exactly; gap_fallback=False keeps bitset2."""
    fs = _fs()
    from paper_1506_08620_b200 import workloads

    p = workloads.knots("cfg5", n1=1_048_577, filtered=False)
    with pytest.raises(fs.Overflow):
        fs.prepare("direct", p)
    prep = fs.prepare_with_fallback(p)
    assert prep.algorithm == "direct-generic" and prep.structure.q == 3
    assert prep.buffers[-1].numel() * 4 <= fs.batch.GAP_FALLBACK_MAX_DIR_BYTES
    z = np.concatenate([workloads.queries_host("cfg5", p, 1_000_003, seed=9), p.values[:-1][::7],
                        np.nextafter(p.values[1:], -np.inf)[::7]])
    want = orc.rank_oracle(p.values, z)
    assert np.array_equal(fs.run_batch(prep, z), want)
    assert fs.prepare_with_fallback(p, gap_fallback=False).algorithm == "bitset2"
