"""Multi-process query sharding on CPU (gloo, world_size 2): the span split,
the per-batch MIN all-reduce of the first out-of-domain position, and the
invariance of results under sharding (the reference's thread-invariance
pattern, pkg/tests/test_batch.py:115-123, with ranks for threads).  The
per-rank searcher here is the CPU oracle; on GPUs it is the CUDA kernel.
The product call itself, dist.sharded_batch_search (device-side global
first-bad, MIN all-reduce, one host read), runs on gloo with a CPU stand-in
for the kernel launch (its status word written the way the kernel's last
CTA writes it)."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import fs_oracle as orc
from paper_1506_08620_b200 import dist as fsdist
from paper_1506_08620_b200.errors import OutOfDomain


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, xs, z, bad_positions, outq):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        a, b = fsdist.shard_span(len(z), rank, world)
        zl = z[a:b].copy()
        for pos in bad_positions:
            if a <= pos < b:
                zl[pos - a] = np.nan
        local_bad = orc.first_bad(xs, zl)
        first = fsdist.global_first_bad(local_bad, a)
        out = None
        if first is None:
            out = orc.rank_oracle(xs, zl)
        outq.put((rank, a, b, first, out))
    finally:
        dist.destroy_process_group()


class _CpuLaunch:
    """PreparedKernel.launch stand-in on CPU tensors: answers from the oracle,
    status word 0 = first bad position or UINT64_MAX (the kernel's contract)."""

    def __init__(self, xs):
        self.xs = xs

    def launch(self, z, out, status, base=0):
        zn = z.numpy()
        bad = orc.first_bad(self.xs, zn)
        w = status.view(torch.int64)
        w[0] = -1 if bad is None else base + bad  # UINT64_MAX = clean
        w[3] = (1 << 63) - 1 if bad is None else base + bad - (1 << 63)  # word 0 XOR 2^63, as int64
        if bad is None:
            out.copy_(torch.from_numpy(orc.rank_oracle(self.xs, zn).astype(np.int32)))


def _product_worker(rank, world, port, xs, z, bad_positions, outq):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        a, b = fsdist.shard_span(len(z), rank, world, granularity=8)
        zl = z[a:b].copy()
        for pos in bad_positions:
            if a <= pos < b:
                zl[pos - a] = np.nan
        out = torch.empty(b - a, dtype=torch.int32)
        status = torch.zeros(4, dtype=torch.uint64)
        try:
            n = fsdist.sharded_batch_search(_CpuLaunch(xs), torch.from_numpy(zl), out, a, status=status)
            outq.put((rank, a, b, None, out.numpy().astype(np.int64), n))
        except OutOfDomain as e:
            outq.put((rank, a, b, e.position, None, 0))
    finally:
        dist.destroy_process_group()


def _run(world, xs, z, bad_positions, worker=None):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=worker or _worker, args=(r, world, port, xs, z, bad_positions, q))
             for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    return sorted(res, key=lambda t: t[0])


@pytest.fixture(scope="module")
def data():
    xs = orc.gen_uniform_gap(4097, 0.5, 1.5, 0, np.float32)
    z = orc.random_queries(xs, 100_003, 1)
    return xs, z


def test_sharded_results_equal_unsharded(data):
    xs, z = data
    res = _run(2, xs, z, [])
    assert all(r[3] is None for r in res)
    got = np.concatenate([r[4] for r in res])
    assert np.array_equal(got, orc.rank_oracle(xs, z))
    assert res[0][1] == 0 and res[-1][2] == len(z)


def test_first_bad_is_global_min_over_ranks(data):
    xs, z = data
    # bad queries on both ranks: every rank must report the global first one
    res = _run(2, xs, z, [90_000, 70_001, 20_000 + 3])
    assert all(r[3] == 20_003 for r in res)
    res = _run(2, xs, z, [99_999])
    assert all(r[3] == 99_999 for r in res)


@pytest.mark.parametrize("world", [2, 3])
def test_sharded_batch_search_product_call(data, world):
    """The product call on gloo: spans tile the batch, results equal the
    unsharded oracle, and an out-of-domain query on any rank raises
    OutOfDomain(global first position) on every rank."""
    xs, z = data
    res = _run(world, xs, z, [], worker=_product_worker)
    assert all(r[3] is None for r in res)
    assert [r[1] for r in res][0] == 0 and res[-1][2] == len(z)
    assert all(r[5] == r[2] - r[1] for r in res)
    assert np.array_equal(np.concatenate([r[4] for r in res]), orc.rank_oracle(xs, z))
    res = _run(world, xs, z, [99_000, 60_001, 40_000 + 5], worker=_product_worker)
    assert all(r[3] == 40_005 for r in res)
