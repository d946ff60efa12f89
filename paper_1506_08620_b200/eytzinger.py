"""Heap-order (Eytzinger) layout built on the device (drop-in for
``fastsearch/eytzinger.py``).

``build_layout`` fills the 2**L - 1 slot tree with one kernel
(``fs_build_eytzinger``: slot q at level l holds the padded knot of in-order
rank (q - 2^l) 2^(L-l) + 2^(L-l-1) - 1, eytzinger.py:45-63); the descent runs
in the batch search kernel (eytzinger.py:84-89).
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from . import _device, _lib
from .partition import SortedPartition, check_domain, fs_dtype


@dataclass(frozen=True)
class EytzingerLayout:
    """Knots in heap order (eytzinger.py:22-32); ``tree_dev`` on the device,
    ``tree`` a host view."""

    tree_dev: object
    L: int
    source: SortedPartition
    _host: dict = field(default_factory=dict, compare=False, repr=False)

    @property
    def tree(self) -> np.ndarray:
        v = self._host.get("tree")
        if v is None:
            v = _device.download(self.tree_dev)
            v.setflags(write=False)
            self._host["tree"] = v
        return v


def tree_depth(n: int) -> int:
    """Smallest L with 2**L - 1 >= n + 1 knots (eytzinger.py:35-37)."""
    return (n + 1).bit_length()


def build_layout(p: SortedPartition) -> EytzingerLayout:
    """O(2**L) device construction (eytzinger.py:40-58)."""
    depth = tree_depth(p.n_intervals)
    x = p.device_values()
    tree = _device.empty((1 << depth) - 1, p.values.dtype)
    rc = _lib.load().fs_build_eytzinger(fs_dtype(p.precision), x.data_ptr(), len(p.values), depth,
                                        tree.data_ptr(), _device.stream_ptr())
    _lib.check(rc, what="fs_build_eytzinger")
    return EytzingerLayout(tree_dev=tree, L=depth, source=p)


def in_order(lay: EytzingerLayout) -> np.ndarray:
    """Flatten the tree back to sorted order, padding included
    (eytzinger.py:61-76); index arithmetic instead of recursion."""
    size = (1 << lay.L) - 1
    slots = np.arange(1, size + 1, dtype=np.int64)
    levels = np.frexp(slots.astype(np.float64))[1] - 1
    stride = np.int64(1) << (lay.L - levels)
    rank = (slots - (np.int64(1) << levels)) * stride + (stride >> 1) - 1
    out = np.empty(size, dtype=lay.tree.dtype)
    out[rank] = lay.tree
    return out


def eytzinger_search(lay: EytzingerLayout, z) -> int:
    """One query on the device (eytzinger.py:82-85)."""
    check_domain(lay.source, z)
    from .direct import _run_single

    return _run_single("eytzinger", lay, lay.source, z)
