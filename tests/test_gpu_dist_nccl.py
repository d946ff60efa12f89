"""The sharded product call over a real NCCL process group on the GPU.

Only one GPU is visible to this build, so the group has one rank; what it
covers is what gloo on CPU cannot: dist.sharded_batch_search's MIN all-reduce
issued by NCCL on the int64 view of the kernel's status word (in place, on
the search stream), with global out-of-domain positions, and bench.py's
torchrun code path (init_process_group("nccl"), barriers, max-over-ranks
reductions, the weak-scaling leg).  Each case runs in its own process so the
test session's CUDA context and default process group stay untouched
(reference: batch.py:385-396 spans, batch.py:411-413 domain check).
"""

import json
import os
import socket
import subprocess
import sys
import textwrap
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parent.parent


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


_WORKER = textwrap.dedent(
    """
    import json, sys
    import numpy as np
    import torch
    import torch.distributed as dist
    sys.path.insert(0, {root!r})
    import paper_1506_08620_b200 as fs
    from paper_1506_08620_b200 import dist as fsdist
    from oracle import fs_oracle as orc

    torch.cuda.set_device(0)
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    res = {{}}
    try:
        for precision, algo in (("single", "direct"), ("double", "direct"), ("single", "bitset2")):
            p = fs.gen_uniform_gap_partition(4097, 0.5, 1.5, seed=3, precision=precision)
            prep = fs.prepare(algo, p)
            m = 300_007
            z = orc.random_queries(p.values, m, seed=11)
            want = orc.rank_oracle(p.values, z)
            zt = torch.from_numpy(z).cuda()
            out = torch.full((m,), -7, dtype=torch.int32, device="cuda")
            st = fs.new_status(zt.device)
            # three spans of one global stream, each through the NCCL all-reduce
            for r in range(3):
                a, b = fsdist.shard_span(m, r, 3, granularity=8)
                assert fsdist.sharded_batch_search(prep, zt[a:b], out[a:b], a, status=st) == b - a
            torch.cuda.synchronize()
            ok = bool(np.array_equal(out.cpu().numpy(), want))
            zt[123_457] = float("inf")
            a, b = fsdist.shard_span(m, 1, 3, granularity=8)
            pos = None
            try:
                fsdist.sharded_batch_search(prep, zt[a:b], out[a:b], a, status=st)
            except fs.OutOfDomain as e:
                pos = e.position
            # the status workspace is reusable after an error
            a0, b0 = fsdist.shard_span(m, 0, 3, granularity=8)
            fsdist.sharded_batch_search(prep, zt[a0:b0], out[a0:b0], a0, status=st)
            res[precision + "/" + algo] = {{"equal": ok, "bad_position": pos,
                                            "global_first_bad": fsdist.global_first_bad(5, 100, device="cuda")}}
    finally:
        dist.destroy_process_group()
    print("RESULT " + json.dumps(res))
    """
)


def _env(port):
    env = dict(os.environ)
    env.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK="0", LOCAL_RANK="0", WORLD_SIZE="1",
               LOCAL_WORLD_SIZE="1")
    return env


def test_sharded_batch_search_over_nccl(cuda):
    done = subprocess.run([sys.executable, "-c", _WORKER.format(root=str(ROOT))], env=_env(_free_port()),
                          capture_output=True, text=True, timeout=600, cwd=str(ROOT))
    assert done.returncode == 0, done.stderr[-3000:]
    line = [ln for ln in done.stdout.splitlines() if ln.startswith("RESULT ")][-1]
    res = json.loads(line[len("RESULT "):])
    assert set(res) == {"single/direct", "double/direct", "single/bitset2"}
    for name, r in res.items():
        assert r["equal"], name
        assert r["bad_position"] == 123_457, (name, r)
        assert r["global_first_bad"] == 105, (name, r)


def test_bench_under_torchrun_one_rank(cuda):
    """bench.py launched the way the driver launches N > 1 (torch.distributed.run),
    with one rank on the one visible GPU and a reduced stream: the JSON line
    carries the contract's keys and the verified flag."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "1", "--master-addr",
           "127.0.0.1", "--master-port", str(_free_port()), "bench.py", "--gpus", "1", "--steps", "3", "--warmup",
           "3", "--queries", str(1 << 24), "--no-cpu-baseline", "--dist-single"]
    done = subprocess.run(cmd, capture_output=True, text=True, timeout=900, cwd=str(ROOT))
    assert done.returncode == 0, done.stderr[-3000:]
    lines = [ln for ln in done.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, done.stdout[-2000:]
    d = json.loads(lines[0])
    assert d["n_gpus"] == 1 and d["config"]["verified"] is True
    assert d["config"]["global_queries"] == 1 << 24 and d["config"]["shards"] == [[0, 1 << 24]]
    assert d["weak"]["queries_per_gpu"] == 1 << 24  # the N>1-only leg ran
    assert all(row["direct"]["verified"] and row["bitset2"]["verified"] for row in d["per_config"].values())
    for key in ("value", "roofline", "e2e", "gpu_launches", "clocks", "kernel_only"):
        assert key in d, key
    assert d["e2e"]["h2d_bytes_per_step"] == 4 << 24 and d["gpu_launches"] >= 3
