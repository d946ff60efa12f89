"""GPU tests of the API surfaces around the hot path: device tensors,
misaligned views, lane/thread invariance, the speculative write-back mode,
the direct->bitset2 fallback policy, placement variants, and full-size
configs checked by the bracket property (unique answer => equals oracle)."""

import numpy as np
import pytest

import golden_data as gd
from oracle import fs_oracle as orc

pytestmark = pytest.mark.gpu


def _fs():
    import paper_1506_08620_b200 as fs

    return fs


def _bracket_ok(p, z, out):
    import torch

    x = p.device_values()
    o = out.long()
    ok = (o >= 0) & (o < p.n_intervals)
    o = o.clamp(0, p.n_intervals - 1)
    return bool((ok & (x[o] <= z) & (z < x[o + 1])).all().item())


@pytest.fixture(scope="module")
def sweep4095():
    case = next(c for c in gd.query_cases() if c["name"] == "sweep_single_4095")
    xs = gd.knots_for(case)
    return case, xs, gd.queries_for(case, xs)


def test_device_tensor_path(cuda, sweep4095):
    import torch

    fs = _fs()
    case, xs, z = sweep4095
    p = fs.validate_partition(xs)
    zt = torch.from_numpy(z).to(cuda)
    for algo in ("direct", "bitset2", "direct-cache", "eytzinger"):
        prep = fs.prepare(algo, p)
        for odt in (torch.int32, torch.int64):
            out = torch.empty(len(z), dtype=odt, device=cuda)
            assert fs.batch_search(fs.LaneConfig(8, algo, prep), zt, out) == len(z)
            gd.check_answers(case, out.cpu().numpy())
        gd.check_answers(case, fs.run_batch(prep, zt).cpu().numpy())
        gd.check_answers(case, prep.lanes(zt).cpu().numpy())


def test_device_path_rejects_what_the_kernel_cannot_take(cuda, sweep4095):
    """Strided outputs land in the right slots (searched into a contiguous
    temporary); a query dtype other than the partition's is refused by
    batch_search, lanes and launch alike, before any kernel reads it."""
    import torch

    fs = _fs()
    case, xs, z = sweep4095
    p = fs.validate_partition(xs)
    zt = torch.from_numpy(z).to(cuda)
    prep = fs.prepare("direct", p)
    cfg = fs.LaneConfig(8, "direct", prep)
    for odt in (torch.int32, torch.int64):
        buf = torch.full((2 * len(z),), -7, dtype=odt, device=cuda)
        assert fs.batch_search(cfg, zt, buf[::2]) == len(z)
        gd.check_answers(case, buf[::2].cpu().numpy())
        assert bool((buf[1::2] == -7).all())
        col = torch.full((len(z), 3), -7, dtype=odt, device=cuda)
        fs.batch_search(cfg, zt, col[:, 1])
        gd.check_answers(case, col[:, 1].cpu().numpy())
        assert bool((col[:, 0] == -7).all() and (col[:, 2] == -7).all())
    wrong = zt.double() if zt.dtype == torch.float32 else zt.float()
    out = torch.empty(len(z), dtype=torch.int64, device=cuda)
    st = fs.new_status(cuda)
    with pytest.raises(ValueError):
        fs.batch_search(cfg, wrong, out)
    with pytest.raises(ValueError):
        prep.lanes(wrong)
    with pytest.raises(ValueError):
        prep.launch(wrong, out, st)
    with pytest.raises(ValueError):
        prep.launch(zt, out[::2], st)
    with pytest.raises(ValueError):
        prep.launch(zt, out.float(), st)
    with pytest.raises(ValueError):
        prep.launch(zt, out[: len(z) - 1], st)
    prep.launch(zt, out, st)
    assert fs.first_bad_of(st) is None
    gd.check_answers(case, out.cpu().numpy())


def test_misaligned_views_and_odd_sizes(cuda, sweep4095):
    """Every head/tail peel and the non-vector store path."""
    import torch

    fs = _fs()
    case, xs, z = sweep4095
    p = fs.validate_partition(xs)
    want = orc.rank_oracle(xs, z)
    zt = torch.from_numpy(z).to(cuda)
    prep = fs.prepare("direct", p)
    # f32 + int32 runs 8-query groups (32-B aligned: heads of 0..7 queries;
    # outputs 32-B, 16-B or 4-B aligned relative to the group), with one
    # (direct) or two (bitset2) groups in flight per thread
    for algo, pr in (("direct", prep), ("bitset2", fs.prepare("bitset2", p))):
        for a in range(0, 9):
            for b in (len(z), len(z) - 1, len(z) - 3, len(z) - 7, a + 1, a + 9, a + 17):
                for oshift in range(0, 8):
                    out = torch.full((b - a + oshift,), -9, dtype=torch.int32, device=cuda)
                    fs.batch_search(fs.LaneConfig(1, algo, pr), zt[a:b], out[oshift:])
                    got = out[oshift:].cpu().numpy()
                    assert np.array_equal(got, want[a:b]), (algo, a, b, oshift)
                    assert (out[:oshift].cpu().numpy() == -9).all()
    # f64 queries (32-B groups of 4) and int64 outputs (32-B stores)
    z64 = zt.double()
    p64 = fs.validate_partition(xs.astype(np.float64))
    prep64 = fs.prepare("direct", p64)
    for a in range(0, 5):
        for oshift in range(0, 5):
            for odt in (torch.int32, torch.int64):
                b = len(z) - 1
                out = torch.full((b - a + oshift,), -9, dtype=odt, device=cuda)
                fs.batch_search(fs.LaneConfig(1, "direct", prep64), z64[a:b], out[oshift:])
                assert np.array_equal(out[oshift:].cpu().numpy(), orc.rank_oracle(p64.values, z64[a:b].cpu().numpy()))
                assert (out[:oshift].cpu().numpy() == -9).all()
    # host arrays: odd lengths, non-contiguous out, other integer dtypes
    for m in (1, 2, 3, 5, 4001):
        out = np.empty(m, dtype=np.int16) if m < 3000 else np.empty(m, dtype=np.uint32)
        fs.batch_search(fs.LaneConfig(3, "direct", prep), z[:m], out)
        assert np.array_equal(out.astype(np.int64), want[:m])
    out = np.zeros(2 * 101, dtype=np.int64)[::2]
    fs.batch_search(fs.LaneConfig(3, "direct", prep), z[:101], out)
    assert np.array_equal(out, want[:101])


def test_python_sequences(cuda, sweep4095):
    """Queries as a Python list / QueryBatch, out as a Python list
    (the reference's slice assignment, batch.py:423)."""
    fs = _fs()
    _, xs, z = sweep4095
    p = fs.validate_partition(xs)
    want = orc.rank_oracle(xs, z[:1000])
    prep = fs.prepare("direct", p)
    out = [None] * 1002
    assert fs.batch_search(fs.LaneConfig(4, "direct", prep), z[:1000].tolist(), out) == 1000
    assert out[:1000] == want.tolist() and out[1000:] == [None, None]
    qb = fs.QueryBatch(values=z[:1000], precision="single")
    assert np.array_equal(fs.run_batch(prep, qb), want)
    assert prep.scalar(float(z[5])) == want[5]
    assert np.array_equal(prep.lanes(z[:1000]), want)


def test_empty_batch_and_capacity(cuda, sweep4095):
    fs = _fs()
    _, xs, z = sweep4095
    prep = fs.prepare("direct", fs.validate_partition(xs))
    assert fs.batch_search(fs.LaneConfig(4, "direct", prep), z[:0], np.empty(0, np.int64)) == 0
    with pytest.raises(ValueError):
        fs.batch_search(fs.LaneConfig(4, "direct", prep), z[:10], np.empty(9, np.int64))


def test_lane_and_thread_invariance(cuda, sweep4095):
    """test_batch.py:32-52, 115-123: d and threads never change results."""
    fs = _fs()
    case, xs, z = sweep4095
    p = fs.validate_partition(xs)
    for algo in fs.ALGORITHMS:
        prep = fs.prepare(algo, p)
        base = fs.run_batch(prep, z, d=1)
        for d in (2, 3, 64, 4001, 100_000):
            assert np.array_equal(fs.run_batch(prep, z, d=d, threads=3), base)
        gd.check_answers(case, base)


def test_speculative_write_back(cuda, sweep4095):
    fs = _fs()
    case, xs, z = sweep4095
    p = fs.validate_partition(xs)
    prep = fs.prepare("direct", p)
    out = np.empty(len(z), dtype=np.int32)
    from paper_1506_08620_b200 import batch as fb

    fb._search_host_array(prep.plan, z, out, chunk_bytes=4096, overlap=True)  # many chunks
    gd.check_answers(case, out)
    bad = z.copy()
    bad[77_777] = np.nan
    bad[90_000] = xs[-1]
    with pytest.raises(fs.OutOfDomain) as e:
        fb._search_host_array(prep.plan, bad, out, chunk_bytes=4096, overlap=True)
    assert e.value.position == 77_777
    with pytest.raises(fs.OutOfDomain) as e:
        fs.batch_search(fs.LaneConfig(4, "direct", prep), bad, out, atomic=False)
    assert e.value.position == 77_777


def test_atomic_contract_with_chunks(cuda, sweep4095):
    """Default mode: many chunks, a bad query in the last one, out untouched."""
    fs = _fs()
    _, xs, z = sweep4095
    prep = fs.prepare("bitset2", fs.validate_partition(xs))
    bad = z.copy()
    bad[-1] = -1.0
    out = np.full(len(z), 123, dtype=np.int64)
    from paper_1506_08620_b200 import batch as fb

    with pytest.raises(fs.OutOfDomain) as e:
        fb._search_host_array(prep.plan, bad, out, chunk_bytes=4096)
    assert e.value.position == len(z) - 1
    assert (out == 123).all()


@pytest.mark.parametrize("precheck", [True, False])
@pytest.mark.parametrize("where", ["first", "middle", "last", "nan", "none"])
def test_host_precheck_atomic_contract(cuda, sweep4095, precheck, where):
    """Atomic mode over many chunks, with and without the host-side domain
    pre-check that lets write-back overlap the uploads: exact answers when
    clean; the device's first-bad position and an untouched `out` when not."""
    fs = _fs()
    from paper_1506_08620_b200 import batch as fb

    _, xs, z = sweep4095
    p = fs.validate_partition(xs)
    prep = fs.prepare("direct", p)
    bad = z.copy()
    pos = {"first": 0, "middle": len(z) // 2, "last": len(z) - 1, "nan": len(z) // 3, "none": None}[where]
    if pos is not None:
        bad[pos] = np.nan if where == "nan" else xs[-1]
        bad[pos + 1:] = np.where(np.arange(len(z) - pos - 1) % 7 == 0, -1.0, bad[pos + 1:]).astype(z.dtype)
    out = np.full(len(z), 123, dtype=np.int32)
    if pos is None:
        fb._search_host_array(prep.plan, bad, out, chunk_bytes=4096, precheck=precheck)
        assert np.array_equal(out, orc.rank_oracle(p.values, z))
    else:
        with pytest.raises(fs.OutOfDomain) as e:
            fb._search_host_array(prep.plan, bad, out, chunk_bytes=4096, precheck=precheck)
        assert e.value.position == pos
        assert (out == 123).all()


@pytest.mark.parametrize("prec", ["single", "double"])
def test_host_precheck_pinned_threads(cuda, prec):
    """Page-locked buffers of several million queries: the host check runs
    on many threads; a bad query deep in a later thread's span is reported
    at its position with `out` untouched, and a clean batch is exact."""
    import torch

    fs = _fs()
    from paper_1506_08620_b200 import batch as fb
    from paper_1506_08620_b200 import workloads

    name = "cfg3" if prec == "single" else "cfg5"
    p = workloads.knots(name) if prec == "single" else workloads.knots("cfg5", n1=1025)
    m = 3_000_017
    zh = workloads.queries_host(name, p, m, seed=12)
    z = torch.from_numpy(zh).pin_memory().numpy()
    out = torch.full((m,), 5, dtype=torch.int32).pin_memory().numpy()
    prep = fs.prepare("direct", p)
    fb._search_host_array(prep.plan, z, out, chunk_bytes=1 << 20)
    assert np.array_equal(out, orc.rank_oracle(p.values, zh))
    out[:] = 5
    z[2_345_678] = -np.inf
    z[2_999_999] = np.nan
    with pytest.raises(fs.OutOfDomain) as e:
        fb._search_host_array(prep.plan, z, out, chunk_bytes=1 << 20)
    assert e.value.position == 2_345_678
    assert (out == 5).all()


@pytest.mark.parametrize("name,kw", [("cfg3", {}), ("cfg5", {"n1": 1025}), ("cfg2", {})])
def test_bitset2_bank_replicated_layout(cuda, name, kw):
    """Large batches of fully smem-resident bitset2 tables use the bank-
    private replicated middle levels (Bitset2Probe); answers equal the
    oracle exactly, and a small batch (plain layout) agrees."""
    fs = _fs()
    from paper_1506_08620_b200 import workloads

    p = workloads.knots(name, **kw)
    prep = fs.prepare("bitset2", p)
    plain = ((1 << p.n_intervals.bit_length()) - 1) * p.values.dtype.itemsize
    assert prep.placement()["smem_bytes"] > plain  # replication planned
    z = workloads.queries_host(name, p, 6_000_001, seed=31)
    want = orc.rank_oracle(p.values, z)
    assert np.array_equal(fs.run_batch(prep, z), want)
    assert np.array_equal(fs.run_batch(prep, z[:5000]), want[:5000])


@pytest.mark.parametrize("dtype,n1", [(np.float32, (1 << 18) + 1), (np.float32, (1 << 19) + 1),
                                       (np.float32, (1 << 20) + 1), (np.float64, (1 << 16) + 1),
                                       (np.float64, (1 << 17) + 1)])
def test_bitset2_subtree_records(cuda, dtype, n1):
    """bitset2 on tables too large for shared memory reads its global levels
    through 32-B subtree records (fs_build_b2_deep): 3 levels per f32 record,
    2 per f64, a leftover level from the padded array.  These sizes cover
    every chunk split (f32: 3+1, 3+2, 3+3; f64: 2+1, 2+2); answers equal the
    oracle on random queries, every knot and its neighbours."""
    fs = _fs()
    rng = np.random.default_rng(n1)
    xs = np.unique(rng.uniform(0.0, 1.0, n1 + n1 // 4).astype(dtype))[:n1]
    p = fs.validate_partition(xs)
    prep = fs.prepare("bitset2", p)
    assert prep.plan.b2_deep  # records built and used
    z = np.concatenate([orc.random_queries(xs, 1_000_000, seed=3), orc.boundary_probes(xs)])
    assert np.array_equal(fs.run_batch(prep, z), orc.rank_oracle(xs, z))


@pytest.mark.parametrize("algo", ["direct", "bitset2", "classic"])
def test_first_bad_across_tail_and_vector_body(cuda, algo):
    """The scalar head/tail queries of a batch are checked before the vector
    body by the same threads: a bad tail query must not hide a smaller bad
    position in the body (thread tid owns tail query tail0 + tid and vector
    group tid).  Every tail length 1..3 and head offset 0..3."""
    import torch

    fs = _fs()
    from paper_1506_08620_b200 import workloads

    p = workloads.knots("cfg3")
    prep = fs.prepare(algo, p)
    base = workloads.queries_device("cfg3", p, 100_000 + 8, seed=4)
    out = torch.empty(base.numel(), dtype=torch.int32, device=cuda)
    for off in range(4):  # head = (4 - off) % 4 queries before the first 16-B group
        for tail in (1, 2, 3):
            m = 4 * 20_000 + tail + (4 - off) % 4
            zz = base.clone()[off:off + m]
            head = (4 - (zz.data_ptr() // 4) % 4) % 4
            tail0 = head + 4 * ((m - head) // 4)
            tid = (m - 1) - tail0
            body = head + 4 * tid + 2  # vector group tid of thread tid, element 2
            zz[m - 1] = float("nan")
            zz[body] = -1.0
            with pytest.raises(fs.OutOfDomain) as e:
                fs.batch_search(fs.LaneConfig(4, algo, prep), zz, out[off:off + m])
            assert e.value.position == body, (off, tail, head)


def test_direct_cache_with_records_too_large_for_smem(cuda):
    """prepare("direct-cache") keeps the reference structure (fused records,
    host view, scalar cache lane) but, when the records cannot be staged,
    searches through direct's device layouts: same answers (direct.py:303-312
    equals 570-574 by construction), no 16-B L2 record gathers."""
    fs = _fs()
    from paper_1506_08620_b200 import workloads

    p = workloads.knots("cfg5", n1=1025)
    prep = fs.prepare("direct-cache", p)
    assert prep.algorithm == "direct-cache"
    assert prep.structure.fused is not None and prep.structure.fused.dtype.itemsize == 16
    assert prep.placement()["smem_sparse"]
    z = workloads.queries_host("cfg5", p, 1_000_003, seed=17)
    want = orc.rank_oracle(p.values, z)
    assert np.array_equal(fs.run_batch(prep, z), want)
    assert [fs.direct_search_cache(prep.structure, v) for v in z[:50]] == want[:50].tolist()


@pytest.mark.parametrize("pinned", [True, False])
def test_host_uploads_ordered_after_pending_work(cuda, pinned):
    """Found by the large-table property test: the caller's allocator may hand
    z_dev a block whose previous owner still has work queued on the current
    stream (an index build's scratch).  The library uploads on its copy
    stream, which must therefore wait for that work -- here a delayed fill
    of the freed block with an out-of-domain value."""
    import torch

    fs = _fs()
    from paper_1506_08620_b200 import workloads

    p = workloads.knots("cfg3")
    prep = fs.prepare("direct", p)
    cfg = fs.LaneConfig(64, "direct", prep)
    m = 3_000_000 if pinned else 6_000_000  # pageable >= 4 MB takes the staged path
    zh = workloads.queries_host("cfg3", p, m, seed=23)
    z = torch.from_numpy(zh).pin_memory().numpy() if pinned else zh
    want = orc.rank_oracle(p.values, zh)
    fs.batch_search(cfg, z, np.empty(m, np.int32))  # warm: library streams and slots exist
    for _ in range(3):
        victim = torch.empty(m, dtype=torch.float32, device=cuda)
        torch.cuda._sleep(200_000_000)  # ~0.1 s of queued work on the current stream ...
        victim.fill_(-5.0)              # ... then a write into the block
        del victim                      # freed while the write is still queued
        out = np.empty(m, np.int32)
        fs.batch_search(cfg, z, out)    # z_dev may reuse the block
        assert np.array_equal(out, want)


@pytest.mark.parametrize("name,kw", [("cfg5", {"n1": 32_769}), ("cfg4", {})])
def test_gap2_rank_directory(cuda, name, kw):
    """direct-gap2 with K and X too large to stage reads a gap-2 directory:
    the count directory (fs_build_countdir, the default) or the rank2 one
    (fs_build_rank2: 16-B words, up to two knots per bucket).
    The layout holds buckets with two knots; answers equal the oracle on
    random queries, every knot and its neighbours."""
    fs = _fs()
    from paper_1506_08620_b200 import workloads

    from paper_1506_08620_b200 import batch as fsb

    p = workloads.knots(name, **kw)
    xs = p.values
    z = np.concatenate([workloads.queries_host(name, p, 2_000_000, seed=29), orc.boundary_probes(xs)])
    want = orc.rank_oracle(xs, z)
    keep = fsb.GAP2_DIRECTORY
    try:
        for layout in ("countdir", "rank2"):  # the default, and the 16-B rank2 words
            fsb.GAP2_DIRECTORY = layout
            prep = fs.prepare("direct-gap2", p)
            assert prep.plan.rank and prep.structure.q == 2 and prep.algorithm == "direct-gap2"
            f = fs.knot_buckets(p, prep.structure.h)
            assert np.any(f[1:] == f[:-1]), "no two-knot bucket: the case is not exercised"
            assert np.array_equal(fs.run_batch(prep, z), want), layout
    finally:
        fsb.GAP2_DIRECTORY = keep


def test_concurrent_big_tables_prepare_then_search(cuda):
    """Soak: five threads on one stream each repeatedly build a large index
    (sparse table, rank directory, subtree records, gap-2 directory) and
    search immediately through the device, pageable and pinned paths, while
    the others' builds are still queued -- the pattern behind the upload
    ordering fix.  Every answer equals the oracle."""
    import threading

    import torch

    fs = _fs()
    from paper_1506_08620_b200 import workloads

    specs = [("cfg5", {"n1": 32_769}, "direct"), ("cfg5", {"n1": 1025}, "direct"),
             ("cfg4", {}, "direct-gap2"), ("cfg5", {"n1": 1_048_577, "filtered": False}, "bitset2"),
             ("cfg4", {}, "direct")]  # zoned records
    errors = []

    def work(k):
        try:
            name, kw, algo = specs[k]
            p = workloads.knots(name, **kw)
            zh = workloads.queries_host(name, p, 5_000_011, seed=40 + k)
            want = orc.rank_oracle(p.values, zh)
            zp = torch.from_numpy(zh).pin_memory().numpy()
            for it in range(3):
                prep = fs.prepare(algo, p)
                cfg = fs.LaneConfig(64, algo, prep)
                out = np.empty(len(zh), np.int64)
                fs.batch_search(cfg, zh, out)  # pageable, staged
                assert np.array_equal(out, want), ("pageable", k, it)
                out32 = np.empty(len(zh), np.int32)
                fs.batch_search(cfg, zp, out32)  # pinned, two-sided check
                assert np.array_equal(out32, want), ("pinned", k, it)
                ot = torch.empty(len(zh), dtype=torch.int32, device=cuda)
                fs.batch_search(cfg, torch.from_numpy(zh).to(cuda), ot)
                assert np.array_equal(ot.cpu().numpy(), want), ("device", k, it)
        except BaseException as ex:  # noqa: BLE001 -- reported by the main thread
            errors.append((k, repr(ex)[:300]))

    threads = [threading.Thread(target=work, args=(k,)) for k in range(len(specs))]
    for t in threads:
        t.start()
    for t in threads:
        t.join()
    assert not errors, errors


def test_batch_beyond_2_pow_32(cuda):
    """Positions and offsets are 64-bit: one batch of 2^32 + 9 queries (16 GiB
    in, 16 GiB out).  Every answer satisfies the bracket property, the tail
    (positions > 2^32) equals the oracle, and a bad query at 2^32 + 3 is
    reported there by both the direct and the bitset2 kernels."""
    import torch

    fs = _fs()
    from paper_1506_08620_b200 import workloads

    p = workloads.knots("cfg3")
    m = (1 << 32) + 9
    z = workloads.queries_device("cfg3", p, m, seed=21)
    out = torch.empty(m, dtype=torch.int32, device=cuda)
    direct = fs.LaneConfig(64, "direct", fs.prepare("direct", p))
    fs.batch_search(direct, z, out)
    x = p.device_values()
    step = 1 << 28
    for a in range(0, m, step):
        zz, o = z[a:a + step], out[a:a + step].long()
        assert bool(((o >= 0) & (o < p.n_intervals)).all())
        assert bool(((x[o] <= zz) & (zz < x[o + 1])).all())
    tail = z[-100_000:].cpu().numpy()
    assert np.array_equal(out[-100_000:].cpu().numpy(), orc.rank_oracle(p.values, tail))
    pos = (1 << 32) + 3
    z[pos] = float("nan")
    for cfg in (direct, fs.LaneConfig(64, "bitset2", fs.prepare("bitset2", p))):
        with pytest.raises(fs.OutOfDomain) as e:
            fs.batch_search(cfg, z, out)
        assert e.value.position == pos
    del z, out
    torch.cuda.empty_cache()


def test_concurrent_callers_share_a_stream(cuda):
    """fsgpu.h "calls are thread-safe" / partition.py:9-10: six threads on the
    SAME (default) stream each build their own index and run device,
    pageable-staged and chunked host searches with out-of-domain queries at
    thread-specific positions; each sees exactly its own answers and
    positions (no shared status word between callers)."""
    import threading

    import torch

    fs = _fs()
    from paper_1506_08620_b200 import batch as fb
    from paper_1506_08620_b200 import workloads

    errors = []

    def work(k):
        try:
            p = workloads.knots("cfg3", seed=k)
            prep = fs.prepare("direct", p)
            cfg = fs.LaneConfig(64, "direct", prep)
            for it in range(4):
                z = workloads.queries_host("cfg3", p, 1_200_000 + 1000 * k, seed=100 * k + it)
                want = orc.rank_oracle(p.values, z)
                out = np.empty(len(z), np.int32)
                fs.batch_search(cfg, z, out)
                assert np.array_equal(out, want), "pageable"
                ot = torch.empty(len(z), dtype=torch.int32, device=cuda)
                fs.batch_search(cfg, torch.from_numpy(z).to(cuda), ot)
                assert np.array_equal(ot.cpu().numpy(), want), "device"
                pos = 1000 * k + 17 * it + 1
                bad = z.copy()
                bad[pos] = np.nan
                with pytest.raises(fs.OutOfDomain) as e:
                    fs.batch_search(cfg, torch.from_numpy(bad).to(cuda), ot)
                assert e.value.position == pos, "device position"
                out2 = np.full(len(z), 9, np.int32)
                with pytest.raises(fs.OutOfDomain) as e:
                    fs.batch_search(cfg, bad, out2)
                assert e.value.position == pos and (out2 == 9).all(), "staged"
                with pytest.raises(fs.OutOfDomain) as e:
                    fb._search_host_array(prep.plan, bad, out2, chunk_bytes=1 << 20)
                assert e.value.position == pos and (out2 == 9).all(), "chunked"
        except BaseException as ex:  # noqa: BLE001 -- reported by the main thread
            errors.append((k, repr(ex)))

    threads = [threading.Thread(target=work, args=(k,)) for k in range(6)]
    for t in threads:
        t.start()
    for t in threads:
        t.join()
    assert not errors, errors


@pytest.mark.parametrize("prec,odt", [("single", np.int32), ("double", np.int64)])
def test_pageable_staged_host_path(cuda, prec, odt):
    """Pageable numpy buffers >= 4 MB go through the library's pinned staging
    ring (several 16 MB slots): answers exact, OutOfDomain in the last chunk
    leaves `out` untouched, atomic=False still reports the position."""
    fs = _fs()
    from paper_1506_08620_b200 import workloads

    p = workloads.knots("cfg3") if prec == "single" else workloads.knots("cfg5", n1=1025)
    name = "cfg3" if prec == "single" else "cfg5"
    z = workloads.queries_host(name, p, 10_000_003, seed=8)
    want = orc.rank_oracle(p.values, z)
    prep = fs.prepare("direct", p)
    out = np.empty(len(z), dtype=odt)
    fs.batch_search(fs.LaneConfig(64, "direct", prep), z, out)
    assert np.array_equal(out, want)
    bad = z.copy()
    bad[-2] = np.nan
    out2 = np.full(len(z), 7, dtype=odt)
    with pytest.raises(fs.OutOfDomain) as e:
        fs.batch_search(fs.LaneConfig(64, "direct", prep), bad, out2)
    assert e.value.position == len(z) - 2 and (out2 == 7).all()
    with pytest.raises(fs.OutOfDomain) as e:
        fs.batch_search(fs.LaneConfig(64, "direct", prep), bad, out2, atomic=False)
    assert e.value.position == len(z) - 2


def test_fallback_policy(cuda):
    """PAPER.md:877 / 754-762: infeasible direct layouts fall back to a larger
    gap (its count directory) or to bitset2."""
    fs = _fs()
    from paper_1506_08620_b200 import workloads

    p = workloads.knots("cfg5", n1=1_048_577, filtered=False)
    with pytest.raises(fs.Overflow):
        fs.prepare("direct", p)
    z = workloads.queries_host("cfg5", p, 300_001, seed=9)
    for prep, algo in ((fs.prepare_with_fallback(p), "direct-generic"),
                       (fs.prepare_with_fallback(p, gap_fallback=False), "bitset2")):
        assert prep.algorithm == algo
        assert np.array_equal(fs.run_batch(prep, z), orc.rank_oracle(p.values, z))
    collide = fs.validate_partition(np.array([-1e9, 0.0, 1.0], dtype=np.float32))
    assert fs.prepare_with_fallback(collide).algorithm == "bitset2"
    assert fs.prepare_with_fallback(collide, algorithm="direct-gap2").algorithm == "direct-gap2"


@pytest.mark.parametrize("variant", ["records", "rank", "k", "global"])
def test_direct_table_variants_agree(cuda, variant):
    """The direct kernel's table encodings (fused records in smem, rank
    directory, plain K, forced L2) give identical answers."""
    fs = _fs()
    from paper_1506_08620_b200 import workloads

    for name, kw in (("cfg3", {}), ("cfg1", {}), ("cfg5", {"n1": 33}), ("cfg4", {})):
        p = workloads.knots(name, **kw)
        z = workloads.queries_host(name, p, 500_003, seed=4)
        prep = fs.prepare("direct", p)
        if variant in ("rank", "k", "global"):
            prep.plan.records = None
        if variant in ("k", "global"):
            prep.plan.rank = None
        if variant == "global":
            prep.plan.smem_policy = 1
        assert np.array_equal(fs.run_batch(prep, z), orc.rank_oracle(p.values, z)), (name, variant)


def test_sparse_table_with_dense_super_buckets(cuda):
    """A mostly-sparse layout with one tight cluster: the two-level sparse
    table with dense (bitmask) super-buckets is chosen and is exact."""
    fs = _fs()
    rng = np.random.default_rng(17)
    base = np.sort(rng.uniform(0.0, 1.0, 1000))
    base = base[np.concatenate([[True], np.diff(base) > 1e-5])]
    cluster = 0.5 + 1e-7 * np.arange(1, 201)
    xs = np.unique(np.concatenate([base[(base < 0.5) | (base > 0.5 + 1e-4)], cluster, [0.0, 1.0]]))
    p = fs.validate_partition(xs)
    from paper_1506_08620_b200 import batch

    old = batch.SPARSE_FORMATS
    try:
        batch.SPARSE_FORMATS = ("two-level",)  # group records are tested in test_gpu_sparse_records.py
        prep = fs.prepare("direct", p)
    finally:
        batch.SPARSE_FORMATS = old
    assert prep.placement()["sparse_format"] == "two-level" and prep.plan.sparse_ndense > 0
    z = np.concatenate([orc.random_queries(xs, 300_000, seed=2), orc.boundary_probes(xs),
                        np.random.default_rng(3).uniform(0.5, 0.5 + 2.1e-5, 100_000)])
    z = z[(z >= xs[0]) & (z < xs[-1])]
    assert np.array_equal(fs.run_batch(prep, z), orc.rank_oracle(xs, z))
    # and the same answers with the dense path's competitors
    prep.plan.sparse = None
    assert np.array_equal(fs.run_batch(prep, z), orc.rank_oracle(xs, z))


def test_scalar_entry_points(cuda):
    """binsearch.py / eytzinger.py scalar wrappers (test_binsearch.py:43-79)."""
    fs = _fs()
    p = fs.validate_partition([0, 1, 2, 3])
    assert fs.classic_search(p, 2.9) == 2 and fs.classic_search(p, 0.0) == 0
    assert fs.bitset_search_v1(p, fs.probe_constant(3), 1.5) == 1
    assert fs.bitset_search_v2(fs.pad_right_pow2(p), 2.5) == 2
    assert fs.bitset_search_v3(p, fs.probe_constant(3), 1.0) == 1
    assert fs.offset_search(p, fs.offset_constants(3), 2.2) == 2
    assert fs.eytzinger_search(fs.build_layout(p), 2.5) == 2
    p9 = fs.gen_uniform_gap_partition(9, 1, 5, seed=9)
    zt = np.nextafter(p9.values[-1], -np.inf)
    assert fs.bitset_search_v1(p9, fs.probe_constant(8), zt) == 7
    assert fs.bitset_search_v2(fs.pad_right_pow2(p9), zt) == 7
    pp = fs.pad_right_pow2(fs.gen_uniform_gap_partition(17, 1, 5, seed=1))
    assert len(pp.padded) == 32 and pp.p == 5 and pp.probe == 16
    for search in (lambda z: fs.classic_search(p, z), lambda z: fs.bitset_search_v2(fs.pad_right_pow2(p), z)):
        with pytest.raises(fs.OutOfDomain):
            search(3.0)
    # gap-2 / generic (test_direct.py:73-79, 110-116, 266-289)
    pc = fs.validate_partition(np.array([-1e9, 0.0, 1.0], dtype=np.float32))
    idx2, _ = fs.build(pc, q=2)
    for z in orc.boundary_probes(pc.values):
        assert fs.direct_search_gap2(idx2, pc, z) == orc.linear_scan(pc.values, z)
    p3 = fs.gen_uniform_gap_partition(63, 1, 5, seed=8)
    idx3, _ = fs.build(p3, q=3)
    for z in orc.boundary_probes(p3.values)[::7]:
        assert fs.direct_search_generic(idx3, p3, z) == orc.linear_scan(p3.values, z)
    pw = fs.validate_partition([0.0, 2.5])
    idxw, _ = fs.build(pw, q=2)
    assert fs.direct_search_gap2(idxw, pw, 1.0) == 0


def test_float64_queries_on_float32_partition(cuda):
    fs = _fs()
    xs = orc.gen_uniform_gap(300, 1, 5, 3, np.float32)
    p = fs.validate_partition(xs)
    rng = np.random.default_rng(0)
    z64 = np.concatenate([rng.uniform(float(xs[0]), float(xs[-1]), 100_000),
                          np.nextafter(xs[1:].astype(np.float64), -np.inf)])
    exact = np.searchsorted(xs.astype(np.float64), z64, side="right") - 1
    for algo in ("direct", "bitset2"):
        assert np.array_equal(fs.run_batch(fs.prepare(algo, p), z64), exact)


@pytest.mark.slow
@pytest.mark.parametrize("name,kw,m", [
    ("cfg3", {}, 1 << 30),
    ("cfg4", {}, 1 << 28),
    ("cfg2", {"seed": 0}, 100_000_000),
    ("cfg5", {"n1": 1_048_577}, 1 << 28),
    ("cfg5", {"n1": 33}, 1 << 28),
])
def test_full_size_configs(cuda, name, kw, m):
    """BASELINE sizes: every answer satisfies X[i] <= z < X[i+1] (bracket
    property, exact float compares), direct == bitset2 elementwise, and a 1e6
    sample equals the CPU oracle."""
    import torch

    fs = _fs()
    from paper_1506_08620_b200 import workloads

    p = workloads.knots(name, **kw)
    z = workloads.queries_device(name, p, m, seed=3)
    outs = []
    for algo in ("direct", "bitset2"):
        prep = fs.prepare(algo, p)
        out = torch.empty(m, dtype=torch.int32, device=cuda)
        fs.batch_search(fs.LaneConfig(65536, algo, prep), z, out)
        assert _bracket_ok(p, z, out), algo
        outs.append(out)
    assert torch.equal(outs[0], outs[1])
    idx = torch.randint(0, m, (1_000_000,), device=cuda)
    zs = z[idx].cpu().numpy()
    assert np.array_equal(outs[0][idx].cpu().numpy(), orc.rank_oracle(p.values, zs))


def test_launch_counts_match_the_kernels_launched(cuda):
    """launches_per_batch / host_launches (fs_search_launches /
    fs_search_host_launches) equal the search kernels CUPTI sees for the
    device path, the chunked pinned path and the staged pageable path."""
    import torch
    from torch.profiler import ProfilerActivity, profile

    fs = _fs()
    p = fs.gen_uniform_gap_partition(4097, 0.5, 1.5, seed=0, precision="single")
    prep = fs.prepare("direct", p)
    cfg = fs.LaneConfig(8, "direct", prep)

    def count(fn):
        torch.cuda.synchronize()
        with profile(activities=[ProfilerActivity.CUDA]) as prof:
            fn()
            torch.cuda.synchronize()
        return sum(1 for e in prof.events() if "search_kernel" in e.name and e.device_type.name == "CUDA")

    m = 3 * (16 << 20) // 4 + 12345  # 50 MB of f32 queries
    z = orc.random_queries(p.values, m, seed=3)
    zt = torch.from_numpy(z).cuda()
    out_t = torch.empty(m, dtype=torch.int32, device=cuda)
    assert count(lambda: fs.batch_search(cfg, zt, out_t)) == prep.launches_per_batch(m) == 1
    out = np.empty(m, dtype=np.int32)
    n_pageable = prep.host_launches(z, out)
    chunk = (min(4 << 20, max((2 << 20) // 4, m // 8)) + 7) & ~7  # staged chunks: m/8 within 2..16 MB
    assert n_pageable == -(-m // chunk) == 8
    assert count(lambda: fs.batch_search(cfg, z, out)) == n_pageable
    zp = torch.from_numpy(z).pin_memory()
    op = torch.empty(m, dtype=torch.int32).pin_memory()
    n_pinned = prep.host_launches(zp.numpy(), op.numpy())
    assert n_pinned == 1  # 50 MB of queries < one 64-MB chunk
    assert count(lambda: fs.batch_search(cfg, zp.numpy(), op.numpy())) == n_pinned
    assert prep.launches_per_batch(0) == 0 and prep.host_launches(z[:0], out[:0]) == 0


@pytest.mark.parametrize("pinned", [False, True])
@pytest.mark.parametrize("nspan", [2, 3])
def test_multi_device_spans_on_one_device(cuda, pinned, nspan):
    """batch_search(..., devices=[0]*k): the batch split into k contiguous
    spans, each a gated native call of its own (the multi-GPU host path,
    exercised with every span on cuda:0).  Answers bit-identical to the
    single call; an out-of-domain query in any span leaves ALL of out
    untouched and reports the batch's first bad position; atomic=False
    reports the same position."""
    import torch

    fs = _fs()
    for prec, odt in (("single", np.int32), ("double", np.int64)):
        p = fs.gen_uniform_gap_partition(4097, 0.5, 1.5, seed=2, precision=prec)
        m = 3_000_011  # odd size: ragged last span, chunked per span
        z = orc.random_queries(p.values, m, seed=5)
        want = orc.rank_oracle(p.values, z)
        prep = fs.prepare("direct", p)
        cfg = fs.LaneConfig(8, "direct", prep)
        if pinned:
            zt = torch.from_numpy(z).pin_memory()
            ot = torch.empty(m, dtype=torch.int32 if odt == np.int32 else torch.int64).pin_memory()
            zz, out = zt.numpy(), ot.numpy()
        else:
            zz, out = z.copy(), np.empty(m, dtype=odt)
        assert fs.batch_search(cfg, zz, out, devices=[0] * nspan) == m
        assert np.array_equal(out, want)
        for bad_at in (m - 1, m // 2 + 3, 5):
            zb = zz.copy()
            zb[bad_at] = np.nan
            zb[min(m - 1, bad_at + 1000)] = p.values[-1]  # a later bad one in the same or next span
            out[:] = -9
            with pytest.raises(fs.OutOfDomain) as ei:
                fs.batch_search(cfg, zb, out, devices=[0] * nspan)
            assert ei.value.position == bad_at
            assert bool((out == -9).all()), "atomic: nothing written when any span is bad"
            with pytest.raises(fs.OutOfDomain) as ei:
                fs.batch_search(cfg, zb, out, devices=[0] * nspan, atomic=False)
            assert ei.value.position == bad_at
        # a tiny batch uses fewer spans; one device entry = the plain path
        assert np.array_equal(fs.run_batch(prep, z[:13]), want[:13])
        small = np.empty(13, dtype=np.int64)
        fs.batch_search(cfg, z[:13], small, devices=[0] * nspan)
        assert np.array_equal(small, want[:13])
        one = np.empty(1000, dtype=np.int64)
        fs.batch_search(cfg, z[:1000], one, devices=[0])
        assert np.array_equal(one, want[:1000])
    with pytest.raises(ValueError):
        fs.batch_search(cfg, z, np.empty(m, dtype=np.int64), devices=[99])


def test_sharded_batch_search_spans_on_one_device(cuda):
    """dist.sharded_batch_search, the call bench.py times per rank, driven
    over k spans of one stream on cuda:0 (no process group: the all-reduce
    is the identity): answers equal the oracle, out-of-domain positions are
    global (span offset added on the device)."""
    import torch

    from paper_1506_08620_b200 import dist as fsdist

    fs = _fs()
    p = fs.gen_uniform_gap_partition(4097, 0.5, 1.5, seed=0, precision="single")
    prep = fs.prepare("direct", p)
    m = 1_000_003
    z = orc.random_queries(p.values, m, seed=9)
    want = orc.rank_oracle(p.values, z)
    zt = torch.from_numpy(z).to(cuda)
    out = torch.empty(m, dtype=torch.int32, device=cuda)
    st = fs.new_status(cuda)
    for k in (1, 2, 5):
        for r in range(k):
            a, b = fsdist.shard_span(m, r, k, granularity=8)
            assert fsdist.sharded_batch_search(prep, zt[a:b], out[a:b], a, status=st) == b - a
        assert np.array_equal(out.cpu().numpy(), want)
    zt[777_777] = float("nan")
    a, b = fsdist.shard_span(m, 1, 2, granularity=8)
    with pytest.raises(fs.OutOfDomain) as ei:
        fsdist.sharded_batch_search(prep, zt[a:b], out[a:b], a)
    assert ei.value.position == 777_777


@pytest.mark.parametrize("precision", ["single", "double"])
def test_staged_rank_directory_beats_unstaged_sparse(cuda, precision, monkeypatch):
    """Uniform gaps U[1, 5] at N+1 = 65535 (R / N = 3): X cannot be staged
    beside any sparse layout, so the rank directory (49 KB) is staged alone
    and X read through L2 for the buckets holding a knot (place();
    profiles/r02/unif_layouts.txt).  Answers equal the oracle at every knot,
    its neighbours and random queries."""
    fs = _fs()
    from paper_1506_08620_b200 import batch

    # (round 2: a byte per knot is staged beside this directory by default, tests/test_gpu_knot_bytes.py;
    # the placement rule under test is the one without it)
    monkeypatch.setattr(batch, "KNOT_BYTES", False)
    p = fs.gen_uniform_gap_partition(65535, 1.0, 5.0, 42, precision)
    prep = fs.prepare("direct", p)
    pl = prep.placement()
    assert pl["smem_table"] and not pl["smem_x"] and not pl["smem_sparse"], pl
    xs = p.values
    z = np.concatenate([orc.random_queries(xs, 300_000, seed=6), orc.boundary_probes(xs),
                        xs[:-1], np.nextafter(xs[1:], -np.inf)]).astype(xs.dtype)
    z = z[(z >= xs[0]) & (z < xs[-1])]
    assert np.array_equal(fs.run_batch(prep, z), orc.rank_oracle(xs, z))
