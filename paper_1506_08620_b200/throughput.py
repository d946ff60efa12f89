"""GPU counterpart of the reference's ``bench throughput`` sweep
(bench/cli.py:76-135, bench/harness.py): every registered algorithm of
``batch.ALGORITHMS`` over generated partitions, timed on device-resident
queries, so the direct search and the comparison searches are compared
under the same names the reference uses.

    python -m paper_1506_08620_b200.throughput --sizes 15,255,4095,65535 \\
        --precision single --algos direct,bitset2 --queries 16777216 --format md

Per (size, algorithm): the partition is ``gen_uniform_gap_partition(size,
gap_lo, gap_hi, seed, precision)``, the queries ``gen_queries`` of it; the
structure is prepared before timing; the first launch's answers are checked
against ``linear_scan_oracle_batch`` (the GPU classic search, an algorithm
independent of the one timed) and must match exactly; each measurement
spans at least ``--min-time`` seconds of back-to-back launches timed with
CUDA events; the figure is the median over ``--reps``.  Algorithms whose
index is infeasible for a partition (Overflow / NotDistinguishable) are
reported on stderr and skipped, as the reference does.

Exit codes (the reference's): 0 success, 1 usage error, 2 every
configuration infeasible.
"""

from __future__ import annotations

import argparse
import statistics
import sys

import numpy as np

EXIT_OK, EXIT_USAGE, EXIT_INFEASIBLE = 0, 1, 2


class _Parser(argparse.ArgumentParser):
    def error(self, message):
        self.print_usage(sys.stderr)
        self.exit(EXIT_USAGE, f"{self.prog}: error: {message}\n")


def _ints(text: str) -> list[int]:
    try:
        return [int(v) for v in text.split(",") if v]
    except ValueError:
        raise argparse.ArgumentTypeError(f"not a comma-separated int list: {text!r}")


def parser() -> argparse.ArgumentParser:
    from .batch import ALGORITHMS

    ap = _Parser(prog="throughput", description="GPU search throughput per algorithm (device-resident queries).")
    ap.add_argument("--sizes", type=_ints, default=[15, 255, 4095, 65535, 1048575])
    ap.add_argument("--precision", choices=("single", "double"), default="single")
    ap.add_argument("--algos", type=lambda t: [a.strip() for a in t.split(",") if a.strip()], default=list(ALGORITHMS))
    ap.add_argument("--queries", type=int, default=1 << 24)
    ap.add_argument("--seed", type=int, default=42)
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--min-time", type=float, default=0.05, help="minimum seconds per measurement")
    ap.add_argument("--gap-lo", type=float, default=1.0)
    ap.add_argument("--gap-hi", type=float, default=5.0)
    ap.add_argument("--qbits", type=int, choices=(32, 64), default=32)
    ap.add_argument("--out-bytes", type=int, choices=(4, 8), default=4, help="int32 or int64 indices")
    ap.add_argument("--format", choices=("csv", "md"), default="csv")
    return ap


def _time_launches(launch, min_time: float, reps: int) -> float:
    """Median seconds per launch over `reps` measurements of >= min_time."""
    import torch

    launch()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    n = 1
    while True:  # launches per measurement
        a.record()
        for _ in range(n):
            launch()
        b.record()
        b.synchronize()
        if a.elapsed_time(b) / 1e3 >= min_time or n >= 1 << 16:
            break
        n *= 2
    samples = []
    for _ in range(reps):
        a.record()
        for _ in range(n):
            launch()
        b.record()
        b.synchronize()
        samples.append(a.elapsed_time(b) / 1e3 / n)
    return statistics.median(samples)


def run_throughput(sizes, precision, algorithms, queries, seed, reps, *, min_time=0.05, gap_lo=1.0, gap_hi=5.0,
                   qbits=32, out_bytes=4):
    """Rows (dicts) of measured configurations and (algorithm, size, cause)
    of the infeasible ones."""
    import torch

    from . import batch
    from .errors import InfeasibleError
    from .partition import gen_queries, gen_uniform_gap_partition, linear_scan_oracle_batch

    unknown = [a for a in algorithms if a not in batch.ALGORITHMS]
    if unknown:
        raise ValueError(f"unknown algorithm(s) {unknown}; pick from {batch.ALGORITHMS}")
    if reps < 1 or queries < 1 or min_time < 0:
        raise ValueError("repetitions and queries must be >= 1, min_time >= 0")
    rows, skipped = [], []
    for size in sizes:
        p = gen_uniform_gap_partition(size, gap_lo, gap_hi, seed, precision)
        zh = np.array(gen_queries(p, queries, seed + 1).values)  # writable copy for torch
        z = torch.from_numpy(zh).cuda()
        want = torch.from_numpy(linear_scan_oracle_batch(p, zh)).cuda()
        out = torch.empty(queries, dtype=torch.int32 if out_bytes == 4 else torch.int64, device=z.device)
        status = batch.new_status()
        for algo in algorithms:
            try:
                prep = batch.prepare(algo, p, qbits)
            except InfeasibleError as e:
                skipped.append((algo, size, f"{type(e).__name__}: {e}"))
                continue
            prep.launch(z, out, status)
            if batch.first_bad_of(status) is not None or not torch.equal(out.long(), want):
                raise RuntimeError(f"{algo} size={size}: answers differ from the oracle")
            t = _time_launches(lambda: prep.launch(z, out, status), min_time, reps)
            rows.append({
                "algorithm": algo, "precision": precision, "size": size, "queries": queries,
                "gqps": queries / t / 1e9, "gbps": queries * (z.element_size() + out_bytes) / t / 1e9,
                "placement": "+".join(k for k, v in prep.placement().items() if v is True) or "global",
            })
            del prep
    return rows, skipped


def emit(rows, fmt: str) -> str:
    cols = ("algorithm", "precision", "size", "queries", "gqps", "gbps", "placement")
    cell = lambda r, c: f"{r[c]:.2f}" if isinstance(r[c], float) else str(r[c])  # noqa: E731
    if fmt == "csv":
        return "".join(",".join(line) + "\n" for line in [cols] + [[cell(r, c) for c in cols] for r in rows])
    head = "| " + " | ".join(cols) + " |\n|" + "---|" * len(cols) + "\n"
    return head + "".join("| " + " | ".join(cell(r, c) for c in cols) + " |\n" for r in rows)


def main(argv=None) -> int:
    ap = parser()
    args = ap.parse_args(argv)
    try:
        rows, skipped = run_throughput(args.sizes, args.precision, args.algos, args.queries, args.seed, args.reps,
                                       min_time=args.min_time, gap_lo=args.gap_lo, gap_hi=args.gap_hi,
                                       qbits=args.qbits, out_bytes=args.out_bytes)
    except ValueError as e:  # unknown algorithm, size < 2, bad gap range
        ap.error(str(e))
    for algo, size, cause in skipped:
        print(f"skipped {algo} size={size} ({args.precision}): {cause}", file=sys.stderr)
    sys.stdout.write(emit(rows, args.format))
    return EXIT_INFEASIBLE if not rows and skipped else EXIT_OK


if __name__ == "__main__":
    sys.exit(main())
