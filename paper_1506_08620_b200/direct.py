"""O(1) bucket-indexed search: certified construction and lookups on the GPU.

Drop-in for ``fastsearch/direct.py`` (direct.py:1-329).  Construction runs on
the device through the C-ABI:

  compute_h_r   -> fs_certify      (direct.py:135-191; K1/K2 kernels)
  knot_buckets  -> fs_knot_buckets (direct.py:194-197)
  build_index   -> fs_build_table  (direct.py:200-243; K3 bucket-parallel fill)
  with_fused    -> fs_build_fused  (direct.py:255-263; K4)

and every arithmetic step is the reference's in the partition's own
precision (see csrc/build.cuh), so h, r, the growth statistics and K are
bit-identical to the reference.  The tables stay resident on the device;
``DirectIndex.k`` / ``.fused`` are read-only host views materialised on
first access for callers (and tests) that inspect them.

The advisory helpers (feasibility_*, closed_form_h_r, memory_cost_estimate,
minimal_index_bytes) are O(N) float64 planning arithmetic identical to the
reference's and run on the host; they never sit on the search path.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass, field, replace
from math import ceil

import numpy as np

from . import _device, _lib
from .errors import NotDistinguishable, OutOfDomain, Overflow
from .partition import ROUNDOFF, SortedPartition, check_domain, fs_dtype

#: Table-entry width is fixed at 32-bit unsigned (direct.py:35).
K_DTYPE = np.uint32

_FUSED_DTYPES = {
    # (knot index, knot value): 8 bytes single, 16 double with 4 zero pad
    # bytes keeping the value aligned (direct.py:39-44).
    "single": np.dtype([("idx", "<u4"), ("val", "<f4")]),
    "double": np.dtype([("idx", "<u4"), ("pad", "<u4"), ("val", "<f8")]),
}


@dataclass(frozen=True)
class HGrowthStats:
    """How often and how far the scale factor grew (direct.py:47-53)."""

    increments: int
    final_h: float
    growth_total: float


@dataclass(frozen=True)
class FeasibilityReport:
    """direct.py:56-61."""

    feasible: bool
    margin: float
    ratio: float
    threshold: float


@dataclass(frozen=True)
class DirectIndex:
    """Immutable bucket index (direct.py:64-83), device resident.

    ``k_dev`` (uint32, r+1) and ``fused_dev`` (records) are the device
    tables the kernels read; ``k`` / ``fused`` are host views.
    """

    x0: np.floating
    h: np.floating
    r: int
    q: int
    k_dev: object
    qbits: int
    n: int
    precision: str
    left_pad: np.ndarray
    fused_dev: object = None
    _host: dict = field(default_factory=dict, compare=False, repr=False)

    @property
    def k(self) -> np.ndarray:
        v = self._host.get("k")
        if v is None:
            v = _device.download(self.k_dev).view(np.uint32)
            v.setflags(write=False)
            self._host["k"] = v
        return v

    @property
    def fused(self) -> np.ndarray | None:
        if self.fused_dev is None:
            return None
        v = self._host.get("fused")
        if v is None:
            raw = _device.download(self.fused_dev)
            v = raw.view(_FUSED_DTYPES[self.precision]).reshape(-1)
            v.setflags(write=False)
            self._host["fused"] = v
        return v


def feasibility_threshold(precision: str, qbits: int) -> float:
    """direct.py:86-101."""
    table = {
        ("single", 32): 2.0 ** -23,
        ("double", 32): 2.0 ** -32,
        ("double", 64): 2.0 ** -51,
    }
    try:
        return table[(precision, qbits)]
    except KeyError:
        return max(2.0 ** -qbits, 2.0 * ROUNDOFF[precision])


def feasibility_estimate(p: SortedPartition, qbits: int = 32, q: int = 1) -> FeasibilityReport:
    """Advisory: smallest gap-q spacing against the span (direct.py:104-120)."""
    xs = p.values.astype(np.float64)
    ratio = float((xs[q:] - xs[:-q]).min() / (xs[-1] - xs[0]))
    threshold = feasibility_threshold(p.precision, qbits)
    return FeasibilityReport(feasible=ratio > threshold, margin=ratio / threshold, ratio=ratio,
                             threshold=threshold)


def closed_form_h_r(p: SortedPartition, q: int = 1) -> tuple[float, int]:
    """Rounding-naive sizing R = 1 + ceil(span / min gap), H = R / span
    (direct.py:123-132)."""
    xs = p.values.astype(np.float64)
    span = float(xs[-1] - xs[0])
    r = 1 + ceil(span / float((xs[q:] - xs[:-q]).min()))
    return r / span, r


def compute_h_r(p: SortedPartition, qbits: int = 32, q: int = 1):
    """Certified scale factor and bucket count, on the GPU (direct.py:135-191).

    Returns ``(h, r, HGrowthStats)`` with ``h`` a numpy scalar of the
    partition's dtype.  Raises NotDistinguishable(position) / Overflow
    exactly where the reference does.
    """
    if qbits not in (32, 64):
        raise ValueError("qbits must be 32 or 64")
    if q < 1:
        raise ValueError("gap must be >= 1")
    scalar = p.values.dtype.type
    x = p.device_values()
    ws = _device.Workspace.get()
    ct = ctypes.c_float if p.precision == "single" else ctypes.c_double
    h = ct(0)
    h0 = ct(0)
    r = ctypes.c_uint64(0)
    inc = ctypes.c_uint32(0)
    pos = ctypes.c_int64(-1)
    rc = _lib.load().fs_certify(
        fs_dtype(p.precision), x.data_ptr(), len(p.values), qbits, q, ws.data_ptr(),
        ctypes.byref(h), ctypes.byref(h0), ctypes.byref(r), ctypes.byref(inc), ctypes.byref(pos),
        _device.stream_ptr(),
    )
    if rc == _lib.FS_OVERFLOW:
        grown = inc.value > 0
        raise Overflow(f"floor(H * D_N) >= 2**{qbits} " + ("while growing H" if grown else "at the initial guess"))
    _lib.check(rc, pos=pos.value, what="fs_certify")
    h_np = scalar(h.value)
    stats = HGrowthStats(
        increments=int(inc.value),
        final_h=float(h_np),
        growth_total=float(h_np - scalar(h0.value)),
    )
    return h_np, int(r.value), stats


def knot_buckets(p: SortedPartition, h) -> np.ndarray:
    """f evaluated at every knot, as int64, in the partition's precision
    (direct.py:194-197), computed on the device."""
    x = p.device_values()
    f = _device.empty(len(p.values), np.uint64)
    rc = _lib.load().fs_knot_buckets(fs_dtype(p.precision), x.data_ptr(), len(p.values), float(h), f.data_ptr(),
                                     _device.stream_ptr())
    _lib.check(rc, what="fs_knot_buckets")
    return _device.download(f).view(np.uint64).astype(np.int64)


def build_index(p: SortedPartition, h, r: int, q: int = 1, qbits: int = 32, fused: bool = False) -> DirectIndex:
    """Materialise the bucket table K on the device (direct.py:200-243).

    gap 1: K_j = i exactly when f(X_{i-1}) < j <= f(X_i), K_0 = 0;
    gap > 1: K_j = max{i : f(X_i) <= j}.  O(N + R) work, R+1 coalesced writes.
    """
    n = p.n_intervals
    if n >= 2 ** 32:
        raise ValueError("table entries are 32-bit; partition is too large")
    if q < 1:
        raise ValueError("gap must be >= 1")
    r = int(r)
    if r < 0:
        raise ValueError("(h, r) pair is inconsistent with this partition")
    x = p.device_values()
    h_s = p.values.dtype.type(h)
    k = _device.empty(r + 1, np.uint32)
    f = _device.empty(len(p.values), np.uint64)
    ws = _device.Workspace.get()
    rc = _lib.load().fs_build_table(fs_dtype(p.precision), x.data_ptr(), len(p.values), float(h_s), r, q,
                                    k.data_ptr(), f.data_ptr(), ws.data_ptr(), _device.stream_ptr())
    _lib.check(rc, what="fs_build_table")
    left_pad = np.full(q - 1, p.values[0], dtype=p.values.dtype)
    left_pad.setflags(write=False)
    idx = DirectIndex(x0=p.values[0], h=h_s, r=r, q=q, k_dev=k, qbits=qbits, n=n, precision=p.precision,
                      left_pad=left_pad)
    return with_fused(idx, p) if fused else idx


def build(p: SortedPartition, qbits: int = 32, q: int = 1, fused: bool = False):
    """compute_h_r then build_index; returns (DirectIndex, HGrowthStats)
    (direct.py:246-252)."""
    h, r, stats = compute_h_r(p, qbits=qbits, q=q)
    return build_index(p, h, r, q=q, qbits=qbits, fused=fused), stats


def with_fused(idx: DirectIndex, p: SortedPartition) -> DirectIndex:
    """Attach cache-fused (index, value) records; gap-1 only (direct.py:255-263)."""
    if idx.q != 1:
        raise ValueError("fused records pair with the gap-1 kernel")
    rec_bytes = _FUSED_DTYPES[idx.precision].itemsize
    rec = _device.empty((idx.r + 1) * rec_bytes, np.uint8)
    x = p.device_values()
    rc = _lib.load().fs_build_fused(fs_dtype(idx.precision), x.data_ptr(), len(p.values), idx.k_dev.data_ptr(),
                                    idx.r, rec.data_ptr(), _device.stream_ptr())
    _lib.check(rc, what="fs_build_fused")
    return replace(idx, fused_dev=rec, _host={})


def _scalar_query(p: SortedPartition, z):
    """One query in the partition's dtype, rounded toward -inf when wider
    (answer-preserving, see partition.coerce_queries)."""
    from .partition import coerce_queries

    return coerce_queries(np.asarray([z]), p.values.dtype)


def _run_single(algorithm: str, structure, p: SortedPartition, z) -> int:
    from .batch import _plan_for, _search_host_array

    plan, keep = _plan_for(algorithm, structure, p)
    out = np.empty(1, dtype=np.int64)
    _search_host_array(plan, _scalar_query(p, z), out)
    del keep
    return int(out[0])


def bucket_of(idx: DirectIndex, z) -> int:
    """f(z) = floor(H * (z - X_0)) in the index's precision (direct.py:266-269).
    A scalar helper; the batch kernels fuse it."""
    t = idx.h.dtype.type
    return int(idx.h * (t(z) - idx.x0))


def direct_search(idx: DirectIndex, p: SortedPartition, z) -> int:
    """Gap-1 kernel, one query on the device (direct.py:272-276)."""
    check_domain(p, z)
    return _run_single("direct", idx, p, z)


def direct_search_gap2(idx: DirectIndex, p: SortedPartition, z) -> int:
    """Gap-2 kernel, one query on the device (direct.py:279-291)."""
    if idx.q != 2:
        raise ValueError("index was not built with gap 2")
    check_domain(p, z)
    return _run_single("direct-gap2", idx, p, z)


def direct_search_generic(idx: DirectIndex, p: SortedPartition, z) -> int:
    """Gap-q kernel, one query on the device (direct.py:294-300)."""
    check_domain(p, z)
    return _run_single("direct-generic", idx, p, z)


def direct_search_cache(idx: DirectIndex, z, p: SortedPartition | None = None) -> int:
    """Gap-1 kernel over fused records (direct.py:303-312).

    The reference signature has no partition; the records carry X_N as
    the value of bucket R, which is the domain's upper end.
    """
    if idx.fused_dev is None:
        raise ValueError("index has no fused records; build with fused=True")
    sentinel = _fused_sentinel(idx)  # equals X_N, since K_R = N
    if not (idx.x0 <= z < sentinel):
        raise OutOfDomain(f"z={z!r} outside [{idx.x0!r}, {sentinel!r})")
    if p is None:
        p = _partition_of_index(idx)
    return _run_single("direct-cache", idx, p, z)


def _fused_sentinel(idx: DirectIndex):
    """Value field of record R (one record read back, not the whole table)."""
    v = idx._host.get("sentinel")
    if v is None:
        dt = _FUSED_DTYPES[idx.precision]
        raw = _device.download(idx.fused_dev[idx.r * dt.itemsize:(idx.r + 1) * dt.itemsize])
        v = raw.view(dt)["val"][0]
        idx._host["sentinel"] = v
    return v


def _partition_of_index(idx: DirectIndex) -> SortedPartition:
    """A minimal partition carrying the domain of a fused index: the cache
    kernel reads only H, X0 and the records, plus X0/XN for the domain."""
    p = idx._host.get("partition")
    if p is None:
        xs = np.array([idx.x0, _fused_sentinel(idx)], dtype=np.dtype(type(idx.x0)))
        p = SortedPartition(values=xs, precision=idx.precision)
        p.values.setflags(write=False)
        idx._host["partition"] = p
    return p


def minimal_index_bytes(n: int) -> int:
    """Smallest power-of-two byte width covering index n (direct.py:315-320)."""
    for b in (1, 2, 4, 8):
        if 2 ** (8 * b) >= n:
            return b
    raise ValueError("n exceeds the largest supported entry width")


def memory_cost_estimate(p: SortedPartition, b: int | None = None) -> int:
    """Estimated gap-1 table footprint (direct.py:323-329)."""
    if b is None:
        b = minimal_index_bytes(p.n_intervals)
    xs = p.values.astype(np.float64)
    entries = ceil(float(xs[-1] - xs[0]) / float(np.diff(xs).min()))
    return entries * b


__all__ = [
    "K_DTYPE",
    "HGrowthStats",
    "FeasibilityReport",
    "DirectIndex",
    "feasibility_threshold",
    "feasibility_estimate",
    "closed_form_h_r",
    "compute_h_r",
    "knot_buckets",
    "build_index",
    "build",
    "with_fused",
    "bucket_of",
    "direct_search",
    "direct_search_gap2",
    "direct_search_generic",
    "direct_search_cache",
    "minimal_index_bytes",
    "memory_cost_estimate",
    "NotDistinguishable",
]
