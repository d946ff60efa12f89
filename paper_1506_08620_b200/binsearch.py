"""Comparison-based lower-bound searches (drop-in for ``fastsearch/binsearch.py``).

The constant builders are the reference's (binsearch.py:34-45); every
search runs on the device through the batch kernels of csrc/search.cuh:

  classic_search     binsearch.py:48-57  (Alg 1)
  bitset_search_v1   binsearch.py:60-69  (Alg 2, range-guarded)
  bitset_search_v2   binsearch.py:72-86  (Alg 3, padded -- the comparison path)
  bitset_search_v3   binsearch.py:89-99  (Alg 4, clamped)
  offset_search      binsearch.py:102-114 (Alg 5)

The pure-Python ``*_seq`` kernels of the reference (used there to count
probes on instrumented sequences) are CPU code and are not part of this
package; the oracle restatement in ``oracle/`` carries them for the tests.
"""

from __future__ import annotations

from dataclasses import dataclass

from .partition import PaddedPartition, SortedPartition, check_domain


@dataclass(frozen=True)
class OffsetConstants:
    """F = (N+1)//2, S = N+1-F, J = floor(log2(N+1)) (binsearch.py:21-31)."""

    F: int
    S: int
    J: int


def offset_constants(n: int) -> OffsetConstants:
    """binsearch.py:34-38."""
    if n < 1:
        raise ValueError("need at least one interval")
    f = (n + 1) >> 1
    return OffsetConstants(F=f, S=n + 1 - f, J=(n + 1).bit_length() - 1)


def probe_constant(n: int) -> int:
    """Leading probe 2**floor(log2 N) (binsearch.py:41-45)."""
    if n < 1:
        raise ValueError("need at least one interval")
    return 1 << (n.bit_length() - 1)


def _one(algorithm: str, structure, p: SortedPartition, z) -> int:
    from .direct import _run_single

    return _run_single(algorithm, structure, p, z)


def classic_search(p: SortedPartition, z) -> int:
    """binsearch.py:117-120."""
    check_domain(p, z)
    return _one("classic", p, p, z)


def bitset_search_v1(p: SortedPartition, probe: int, z) -> int:
    """binsearch.py:123-126."""
    check_domain(p, z)
    return _one("bitset1", probe, p, z)


def bitset_search_v2(pp: PaddedPartition, z) -> int:
    """binsearch.py:129-132."""
    check_domain(pp.base, z)
    return _one("bitset2", pp, pp.base, z)


def bitset_search_v3(p: SortedPartition, probe: int, z) -> int:
    """binsearch.py:135-138."""
    check_domain(p, z)
    return _one("bitset3", probe, p, z)


def offset_search(p: SortedPartition, c: OffsetConstants, z) -> int:
    """binsearch.py:141-144."""
    check_domain(p, z)
    return _one("offset", c, p, z)
