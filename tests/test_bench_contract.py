"""The root bench.py contract on CPU: the reference arm (`--impl reference`,
the CPU lane path timed on host cores) prints exactly one well-formed JSON
line, also when launched by torchrun with two ranks (rank 0 runs and prints,
rank 1 exits 0 without work).  The GPU arm is exercised by the driver on
the B200."""

import json
import socket
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
FAST = ["--impl", "reference", "--steps", "2", "--warmup", "3", "--ref-sample", "65536", "--ref-min-time", "0"]


def _json_lines(stdout: str):
    return [json.loads(line) for line in stdout.splitlines() if line.startswith("{")]


def _check_line(d, n_gpus):
    assert d["impl"] == "reference" and d["n_gpus"] == n_gpus
    assert d["unit"] == "queries/s" and d["higher_is_better"] is True and d["value"] > 0
    assert d["steps"] == 2 and d["warmup"] == 3 and d["scaling"] == "strong" and d["vs_baseline"] is None
    cb = d["cpu_baseline"]
    assert cb["kind"] in ("port", "reference") and cb["cores"] >= 1 and cb["value"] == d["value"] and cb["sample"]
    if (ROOT / "baseline" / "_ref" / "fastsearch" / "__init__.py").exists():
        assert cb["kind"] == "reference" and "baseline/_ref" in cb["sample"], cb  # the unmodified reference ran
    assert cb["cpu_model"]
    assert d["e2e"] == {"value": d["value"], "unit": d["unit"], "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}
    assert d["config"]["workload"].startswith("cfg3")


def test_reference_arm_json_line():
    r = subprocess.run([sys.executable, "bench.py", *FAST], cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = _json_lines(r.stdout)
    assert len(lines) == 1
    _check_line(lines[0], 1)


def test_reference_arm_under_torchrun_two_ranks():
    r = _torchrun(2, FAST)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = _json_lines(r.stdout)
    assert len(lines) == 1
    _check_line(lines[0], 2)


def _torchrun(n, args):
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", str(n), "--master-addr",
           "127.0.0.1", "--master-port", str(port), "bench.py", "--gpus", str(n), *args]
    return subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=600)


def test_sharding_plan_is_configs2_as_written():
    """At every N the GPU arm times ONE global stream of 2^30 queries
    (configs[2]), rank r owning dist.shard_span(2^30, r, N): the spans tile
    [0, 2^30) contiguously and config.global_queries == 2^30 (the plan is
    computed by the same code the GPU arm uses, under torchrun + gloo)."""
    for n in (1, 2, 4, 8):
        if n == 1:
            r = subprocess.run([sys.executable, "bench.py", "--plan-only"], cwd=ROOT, capture_output=True, text=True,
                               timeout=600)
        else:
            r = _torchrun(n, ["--plan-only"])
        assert r.returncode == 0, r.stderr[-2000:]
        lines = _json_lines(r.stdout)
        assert len(lines) == 1, r.stdout
        d = lines[0]
        assert d["n_gpus"] == n and d["scaling"] == "strong"
        cfg = d["config"]
        assert cfg["global_queries"] == 1 << 30
        spans = cfg["shards"]
        assert len(spans) == n and spans[0][0] == 0 and spans[-1][1] == 1 << 30
        for (a, b), (c, _) in zip(spans, spans[1:]):
            assert b == c and a < b and a % 8 == 0
        assert sum(cfg["queries_per_gpu"]) == 1 << 30
        assert max(cfg["queries_per_gpu"]) - min(cfg["queries_per_gpu"]) <= 8
