"""The GPU throughput sweep (paper_1506_08620_b200.throughput, the
counterpart of the reference's ``bench throughput``, bench/cli.py:76-135):
argument handling and exit codes on CPU; on the GPU, every registered
algorithm measured and checked, infeasible direct indices skipped with
exit code 2 when nothing else ran."""

import subprocess
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent


def _run(*args):
    return subprocess.run([sys.executable, "-m", "paper_1506_08620_b200.throughput", *args], cwd=ROOT,
                          capture_output=True, text=True, timeout=600)


def test_usage_errors_exit_1():
    for bad in (["--sizes", "a,b"], ["--precision", "half"], ["--format", "xml"], ["--out-bytes", "2"],
                ["--reps", "0"], ["--queries", "0"], ["--algos", "direct,nope"]):
        r = _run(*bad)
        assert r.returncode == 1, (bad, r.stderr)
        assert "usage" in r.stderr


def test_help_lists_algorithms_default():
    from paper_1506_08620_b200 import throughput
    from paper_1506_08620_b200.batch import ALGORITHMS

    args = throughput.parser().parse_args([])
    assert args.algos == list(ALGORITHMS) and args.sizes == [15, 255, 4095, 65535, 1048575]


def test_emit_formats():
    from paper_1506_08620_b200 import throughput

    rows = [{"algorithm": "direct", "precision": "single", "size": 15, "queries": 8, "gqps": 1.5, "gbps": 12.0,
             "placement": "smem_x"}]
    csv = throughput.emit(rows, "csv").splitlines()
    assert csv[0].startswith("algorithm,precision,size") and csv[1] == "direct,single,15,8,1.50,12.00,smem_x"
    md = throughput.emit(rows, "md").splitlines()
    assert md[0].startswith("| algorithm |") and md[2].startswith("| direct | single | 15 |")


@pytest.mark.gpu
def test_every_algorithm_measured(cuda):
    from paper_1506_08620_b200 import throughput
    from paper_1506_08620_b200.batch import ALGORITHMS

    for precision in ("single", "double"):
        rows, skipped = throughput.run_throughput([255, 4095], precision, list(ALGORITHMS), 1 << 20, 42, 2,
                                                  min_time=0.002)
        assert not skipped
        assert {(r["algorithm"], r["size"]) for r in rows} == {(a, s) for a in ALGORITHMS for s in (255, 4095)}
        assert all(r["gqps"] > 0 for r in rows)


@pytest.mark.gpu
def test_infeasible_only_exit_2(cuda):
    # 10^6 gaps uniform in [1e-9, 1]: the smallest is ~1e-6 against a span of
    # ~5e5, so h * D_N exceeds 2^32 -- Overflow for both direct indices
    r = _run("--sizes", "1000000", "--precision", "double", "--algos", "direct,direct-cache", "--gap-lo", "1e-9",
             "--gap-hi", "1", "--queries", "1024", "--reps", "1")
    assert r.returncode == 2, r.stderr
    assert r.stderr.count("skipped direct") == 2 and "Overflow" in r.stderr


@pytest.mark.gpu
def test_infeasible_recorded_not_fatal(cuda):
    """A sweep where the direct index is infeasible for one size keeps the
    other sizes and algorithms (the reference's harness behaviour)."""
    from paper_1506_08620_b200 import throughput

    rows, skipped = throughput.run_throughput([255, 1_000_000], "double", ["direct", "bitset2"], 1 << 16, 42, 1,
                                              min_time=0.0, gap_lo=1e-9, gap_hi=1.0)
    assert ("direct", 1_000_000) in {(a, s) for a, s, _ in skipped}
    got = {(r["algorithm"], r["size"]) for r in rows}
    assert ("bitset2", 1_000_000) in got and ("direct", 255) in got and ("bitset2", 255) in got
