"""Index files written by the REFERENCE's own save_index (bench/persist.py),
for byte-exact round-trip tests of the device loader/saver.

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden_persist.py
"""

from pathlib import Path

import numpy as np

from fastsearch.bench.persist import save_index
from fastsearch.direct import build
from fastsearch.partition import gen_uniform_gap_partition, validate_partition

OUT = Path(__file__).resolve().parent / "idx"


def main():
    OUT.mkdir(exist_ok=True)
    cases = {
        "worked_double": (validate_partition([0.0, 0.5, 0.7, 1.1]), 1),
        "worked_single": (validate_partition(np.array([0.0, 0.5, 0.7, 1.1], dtype=np.float32)), 1),
        "s100_double": (gen_uniform_gap_partition(100, 1, 5, seed=31, precision="double"), 1),
        "s100_single": (gen_uniform_gap_partition(100, 1, 5, seed=31, precision="single"), 1),
        "s100_double_q2": (gen_uniform_gap_partition(100, 1, 5, seed=31, precision="double"), 2),
        "s4097_single": (gen_uniform_gap_partition(4097, 0.5, 1.5, seed=0, precision="single"), 1),
    }
    for name, (p, q) in cases.items():
        idx, _ = build(p, q=q)
        n = save_index(idx, OUT / f"{name}.idx")
        print(name, n, "bytes")


if __name__ == "__main__":
    main()
