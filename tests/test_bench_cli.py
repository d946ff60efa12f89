"""The bench/index CLI, harness and report on the GPU path (reference
pkg/tests/test_bench.py:41-362 mirrored).  Report formatting, argument
errors and file errors are CPU tests; sweeps and index round trips are GPU."""

import numpy as np
import pytest

from paper_1506_08620_b200.bench import (
    SetupStatsRow,
    ThroughputRow,
    aligned_empty,
    bench_main,
    emit_report,
    index_main,
    run_setup_stats,
    run_throughput,
)


class TestReport:
    def rows(self):
        return [
            ThroughputRow("direct", "single", 4, 255, 120.5, 1000, 5),
            ThroughputRow("classic", "single", 1, 15, 48.25, 1000, 5),
            ThroughputRow("classic", "single", 1, 255, 20.0, 1000, 5),
        ]

    def test_csv_header_and_order(self):
        lines = emit_report(self.rows(), "csv").strip().split("\n")
        assert lines[0] == "algorithm,precision,lane_width,size,throughput_msps,queries,repetitions"
        assert lines[1].startswith("classic,single,1,15")
        assert lines[2].startswith("classic,single,1,255")
        assert lines[3].startswith("direct,single,4,255,120.50")

    def test_extended_columns(self):
        row = ThroughputRow("direct", "single", 1, 4097, 700000.0, 1 << 20, 5, gbs=5600.0, roofline_frac=0.8667,
                            placement="smem_table:65280", table_bytes=81920)
        lines = emit_report([row], "csv", extended=True).strip().split("\n")
        assert lines[0].endswith(",gbs,roofline_frac,placement,table_bytes,gpus")
        assert lines[1].endswith(",5600.0,0.8667,smem_table:65280,81920,1")

    def test_markdown_escapes_pipes(self):
        text = emit_report([ThroughputRow("weird|name", "single", 1, 15, 1.0, 10, 1)], "md")
        assert r"weird\|name" in text and text.startswith("| algorithm |")

    def test_empty_rows_emit_header_only(self):
        assert emit_report([], "csv").strip().count("\n") == 0
        assert emit_report([], "md", kind="setup").strip().split("\n")[0].startswith("| size |")

    def test_setup_rows(self):
        row = SetupStatsRow(255, 100, 0.01, 0.0, 1.0, 0.0995, 150.0, 120.0, 900.0, 40.0)
        assert "0.0100,0.0000,1.0000,0.0995,150.00" in emit_report([row], "csv", kind="setup")

    def test_unknown_format(self):
        with pytest.raises(ValueError):
            emit_report([], "html")


def test_aligned_allocation():
    for dtype in (np.float32, np.float64):
        arr = aligned_empty(1000, dtype)
        assert arr.ctypes.data % 32 == 0 and len(arr) == 1000 and arr.dtype == dtype


def test_usage_error_exit_code():
    with pytest.raises(SystemExit) as exc:
        bench_main(["throughput", "--format", "yaml"])
    assert exc.value.code == 1


def _write_partition(tmp_path, values, name="knots.csv"):
    path = tmp_path / name
    path.write_text("\n".join(str(v) for v in values) + "\n")
    return path


def test_index_file_errors_are_io_errors(tmp_path, capsys):
    bad = tmp_path / "bad.idx"
    bad.write_bytes(b"NOTANIDX" + b"\0" * 64)
    assert index_main(["load", "--path", str(bad)]) == 3
    assert index_main(["load", "--path", str(tmp_path / "absent.idx")]) == 3


def test_invalid_partition_is_usage_error(tmp_path, capsys):
    knots = _write_partition(tmp_path, [0.0, 1.0, 1.0])
    assert index_main(["save", "--path", str(tmp_path / "o.idx"), "--partition", str(knots)]) == 1
    assert "invalid partition" in capsys.readouterr().err
    path = tmp_path / "nan.csv"
    path.write_text("0.0\nabc\n")
    assert index_main(["save", "--path", str(tmp_path / "o.idx"), "--partition", str(path)]) == 1


# ---------------------------------------------------------------- GPU ----


def _tiny(**overrides):
    kw = dict(sizes=[15], precisions=["double"], algorithms=["classic", "direct"], d_widths=[1, 4], queries=500,
              seed=42, repetitions=2, min_time=0.001)
    kw.update(overrides)
    return run_throughput(**kw)


@pytest.mark.gpu
def test_throughput_rows_well_formed(cuda):
    rep = _tiny()
    assert {(r.algorithm, r.lane_width) for r in rep.rows} == {("classic", 1), ("classic", 4), ("direct", 1),
                                                                 ("direct", 4)}
    for r in rep.rows:
        assert r.throughput_msps > 0 and r.queries == 500 and r.repetitions == 2 and r.size == 15
    assert rep.skipped == []
    rep = _tiny(resident=True, algorithms=["direct", "bitset2"], d_widths=[1])
    assert all(r.gbs > 0 and 0 < r.roofline_frac for r in rep.rows)


@pytest.mark.gpu
def test_infeasible_configs_recorded_not_fatal(cuda):
    rep = _tiny(sizes=[262144], algorithms=["classic", "direct", "direct-cache"], d_widths=[1], gap_hi=1e9,
                queries=200)
    assert {r.algorithm for r in rep.rows} == {"classic"}
    assert {s.algorithm for s in rep.skipped} == {"direct", "direct-cache"}
    assert all("Overflow" in s.cause for s in rep.skipped)


@pytest.mark.gpu
def test_setup_stats_shape(cuda):
    rep = run_setup_stats(sizes=[15, 255], precision="single", samples=40, seed=3)
    assert rep.infeasible == {} and [r.size for r in rep.rows] == [15, 255]
    for r in rep.rows:
        assert r.samples == 40 and r.h_updates_min <= r.h_updates_mean <= r.h_updates_max
        assert 0 < r.setup_ns_per_elem_min <= r.setup_ns_per_elem_mean <= r.setup_ns_per_elem_max


@pytest.mark.gpu
def test_cli_throughput_and_setup(cuda, capsys):
    code = bench_main(["throughput", "--sizes", "15,255", "--precision", "single", "--algos", "direct",
                       "--lanes", "1", "--queries", "1000", "--reps", "1", "--min-time", "0.001"])
    out = capsys.readouterr().out.strip().split("\n")
    assert code == 0 and out[0].startswith("algorithm,precision") and len(out) == 3
    code = bench_main(["setup-stats", "--sizes", "15", "--samples", "5", "--format", "md"])
    assert code == 0 and capsys.readouterr().out.startswith("| size |")
    code = bench_main(["throughput", "--sizes", "262144", "--precision", "double", "--algos", "direct", "--lanes",
                       "1", "--queries", "100", "--reps", "1", "--min-time", "0.001", "--gap-hi", "1e9"])
    captured = capsys.readouterr()
    assert code == 2 and "skipped direct" in captured.err and captured.out.startswith("algorithm,")


@pytest.mark.gpu
def test_index_cli_save_then_load_with_verification(cuda, tmp_path, capsys):
    knots = _write_partition(tmp_path, [0.0, 0.5, 0.7, 1.1])
    out = tmp_path / "w.idx"
    assert index_main(["save", "--path", str(out), "--partition", str(knots)]) == 0
    assert "wrote" in capsys.readouterr().out
    code = index_main(["load", "--path", str(out), "--partition", str(knots), "--verify-queries", "500"])
    printed = capsys.readouterr().out
    assert code == 0 and "verified 500 queries" in printed and "n=3 r=5" in printed
