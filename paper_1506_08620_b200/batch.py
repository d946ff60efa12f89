"""The operator boundary: prepare / PreparedKernel / batch_search on the GPU.

Drop-in for ``fastsearch/batch.py`` (batch.py:1-451).  ``prepare`` builds the
search structure of any of the nine ``ALGORITHMS`` on the device and returns
a ``PreparedKernel`` whose ``lanes``/``scalar`` callables and whose use in
``batch_search``/``run_batch`` dispatch one CUDA kernel over the whole batch
(csrc/search.cuh).  What the reference guarantees, this keeps:

  * ``out[j]`` is query j's answer, independent of the lane width ``d`` and
    the thread count (batch.py:402-403) -- the GPU has no lane/tail split,
    so invariance holds by construction;
  * OutOfDomain(position = first bad j) for any !(X0 <= z < XN), NaN
    included, with nothing written to a host ``out`` (batch.py:404, 411-413):
    the check is fused into the search kernel and results are copied back
    only when the batch is clean;
  * infeasible direct layouts raise from ``prepare`` (batch.py:159-160).
    ``prepare_with_fallback`` is the explicit policy the paper implies
    (PAPER.md:877): direct when feasible, else the padded bit-set search.

Inputs: numpy arrays / QueryBatch (host; copied in chunks overlapped with
the kernel) or CUDA torch tensors (device-resident; no copies).
"""

from __future__ import annotations

import ctypes
import os
import threading
from dataclasses import dataclass, field
from typing import Callable

import numpy as np

from . import _device, _lib
from .binsearch import offset_constants, probe_constant
from .direct import DirectIndex, build
from .errors import InfeasibleError, OutOfDomain
from .eytzinger import EytzingerLayout, build_layout
from .partition import PaddedPartition, QueryBatch, SortedPartition, coerce_queries, fs_dtype, pad_right_pow2

ALGORITHMS = (
    "classic",
    "bitset1",
    "bitset2",
    "bitset3",
    "offset",
    "eytzinger",
    "direct",
    "direct-gap2",
    "direct-cache",
)

THREADS_ENV = "FASTSEARCH_THREADS"

#: host->device chunk for the end-to-end path (elements); ~64 MB of queries
HOST_CHUNK_BYTES = 64 << 20

#: fused (K[j], X[K[j]]) records are built for the direct kernel when they can
#: be staged in shared memory (227 KB per CTA on sm_100a, less static use)
SMEM_RECORDS_MAX = 226 * 1024

_copy_streams: dict = {}


def _copy_stream():
    import torch

    dev = torch.cuda.current_device()
    s = _copy_streams.get(dev)
    if s is None:
        s = torch.cuda.Stream(device=dev)
        _copy_streams[dev] = s
    return s


def _plan_for(algorithm: str, structure, p: SortedPartition):
    """fs_plan for ``algorithm`` over ``structure``; returns (plan, keepalive)."""
    plan = _lib.FsPlan()
    plan.algorithm = _lib.ALGO_CODES[algorithm]
    plan.dtype = fs_dtype(p.precision)
    plan.n1 = len(p.values)
    x = p.device_values()
    plan.x = x.data_ptr()
    plan.device_index = x.get_device()  # (Python-side only: the device the tables live on)
    plan.x0 = float(p.values[0])
    plan.xn = float(p.values[-1])
    plan.q = 1
    plan.pbits = max(1, p.n_intervals.bit_length())
    keep = [x]
    if algorithm.startswith("direct"):
        idx: DirectIndex = structure
        plan.r = idx.r
        plan.h = float(idx.h)
        plan.q = idx.q
        if algorithm == "direct-cache":
            plan.table = idx.fused_dev.data_ptr()
            keep.append(idx.fused_dev)
        else:
            plan.table = idx.k_dev.data_ptr()
            keep.append(idx.k_dev)
    elif algorithm == "bitset2":
        pp: PaddedPartition = structure
        plan.table = pp.padded_dev.data_ptr()
        plan.pbits = pp.p
        keep.append(pp.padded_dev)
        _set_b2_deep(plan, pp, keep)
    elif algorithm == "eytzinger":
        lay: EytzingerLayout = structure
        plan.table = lay.tree_dev.data_ptr()
        plan.pbits = lay.L
        keep.append(lay.tree_dev)
    return plan, keep


def _search_host_array(plan, z: np.ndarray, out: np.ndarray, chunk_bytes: int = HOST_CHUNK_BYTES,
                       overlap: bool = False, precheck: bool = True, gate=None) -> None:
    """End-to-end search of host queries into host ``out[:m]`` (fs_search_host).
    ``overlap`` = speculative per-chunk write-back (FS_HOST_OVERLAP);
    ``precheck=False`` = wait for the device's domain check before any
    write-back (FS_HOST_NO_PRECHECK); ``gate`` = this call is one span of a
    batch split over devices (fs_search_host_gated)."""
    m = len(z)
    if m == 0:
        return
    try:
        _device.require_cuda()
        z = np.ascontiguousarray(z)
        direct_out = out.dtype in (np.int32, np.int64) and out.flags.c_contiguous and out.flags.writeable
        target = out[:m] if direct_out else np.empty(m, dtype=np.int64)
        ob = target.dtype.itemsize
        z_dev = _device.empty(m, z.dtype)
        o_dev = _device.empty(m, target.dtype)
        fb = _cached_status(z_dev.device, _device.stream_ptr())
    except BaseException:
        if gate is not None:  # this span cannot make its call: release the others
            _lib.load().fs_gate_abort(gate)
        raise
    pos = ctypes.c_int64(-1)
    rc = _lib.load().fs_search_host_gated(
        ctypes.byref(plan), z.ctypes.data, m, target.ctypes.data, ob, z_dev.data_ptr(), o_dev.data_ptr(),
        fb.data_ptr(), max(4, chunk_bytes // z.dtype.itemsize), ctypes.byref(pos), _device.stream_ptr(),
        _device.stream_ptr(_copy_stream()),
        (_lib.FS_HOST_OVERLAP if overlap else 0) | (0 if precheck else _lib.FS_HOST_NO_PRECHECK), gate,
    )
    _lib.check(rc, pos=pos.value, what="fs_search_host")
    if not direct_out:
        out[:m] = target


def new_status(device=None):
    """A zeroed search status workspace (FS_SEARCH_WS_WORDS uint64) for
    PreparedKernel.launch: word 0 receives the first out-of-domain position
    (UINT64_MAX when clean).  Reusable by stream-ordered searches, not by
    concurrent ones."""
    import torch

    dev = device if device is not None else _device.require_cuda()
    return torch.zeros(int(_lib.load().fs_search_ws_words()), dtype=torch.uint64, device=dev)


_tls = threading.local()


def _cached_status(device, stream_ptr: int):
    """One status workspace per (thread, device, stream).  One thread's calls
    on a stream are ordered, so they can share it; two threads on the same
    stream must not, or one's launch could land between the other's kernel
    and its read-back of the first-bad word."""
    cache = getattr(_tls, "status", None)
    if cache is None:
        cache = _tls.status = {}
    key = (device.index, stream_ptr)
    s = cache.get(key)
    if s is None:
        s = new_status(device)
        cache[key] = s
    return s


def _launch_device(plan, z, out, status, base: int = 0) -> None:
    """Asynchronous device search (fs_search_device_at): exactly one kernel;
    status[0] receives base + the first out-of-domain position, status[3]
    the same XOR 2^63 (signed order, clean = INT64_MAX)."""
    lib = _lib._lib or _lib.load()
    rc = lib.fs_search_device_at(ctypes.byref(plan), z.data_ptr(), z.numel(), out.data_ptr(), out.element_size(),
                                 status.data_ptr(), int(base), _device.stream_ptr(device_index=z.get_device()))
    if rc:
        _lib.check(rc, what="fs_search_device")


def first_bad_of(status):
    """Read the first out-of-domain position from a status workspace (syncs);
    None when every query was in domain."""
    import torch

    bad = int(status[:1].view(torch.int64).item())
    return None if bad == -1 else bad


def _check_device_batch(plan, z, out) -> None:
    """Device batches the C-ABI can take as they are: query dtype = the
    partition's (a narrower or wider buffer would be read with the wrong
    element size), int32/int64 ``out``, both contiguous and on the
    partition's device (the kernel writes ``out.numel()`` consecutive
    elements from its base address)."""
    import torch

    want = torch.float32 if plan.dtype == _lib.FS_F32 else torch.float64
    if z.dtype != want:
        raise ValueError(f"query dtype {z.dtype} does not match the partition's {want}")
    if out.dtype not in (torch.int32, torch.int64):
        raise ValueError("out must be int32 or int64")
    if not (z.is_cuda and out.is_cuda):
        raise ValueError("device-resident batches need CUDA tensors for both queries and out")
    if z.device != out.device or z.get_device() != plan.device_index:
        raise ValueError(f"queries ({z.device}), out ({out.device}) and the prepared structure "
                         f"(cuda:{plan.device_index}) must be on one device")
    if not out.is_contiguous():
        raise ValueError("out must be contiguous (search into a contiguous tensor and copy_ it)")
    if out.numel() < z.numel():
        raise ValueError("output array is smaller than the query batch")


def _search_device_tensor(plan, z, out) -> None:
    _check_device_batch(plan, z, out)
    st = _cached_status(z.device, _device.stream_ptr())
    _launch_device(plan, z, out, st)
    bad = first_bad_of(st)
    if bad is not None:
        raise OutOfDomain(position=bad)


def _is_torch(a) -> bool:
    mod = type(a).__module__
    return mod.startswith("torch")


@dataclass(frozen=True)
class PreparedKernel:
    """A device search structure plus its scalar and batch entry points
    (batch.py:132-140).  ``plan`` is the C-ABI descriptor; ``buffers`` keeps
    its device tables alive."""

    algorithm: str
    partition: SortedPartition
    structure: object
    scalar: Callable
    lanes: Callable | None
    plan: object = field(default=None, repr=False, compare=False)
    buffers: tuple = field(default=(), repr=False, compare=False)
    replicas: dict = field(default_factory=dict, repr=False, compare=False)

    @property
    def device_index(self) -> int:
        return self.plan.device_index

    def on_device(self, device: int) -> "PreparedKernel":
        """This kernel's structure built on another CUDA device (once, then
        cached): the build is deterministic, so every replica is
        bit-identical."""
        import torch

        device = int(device)
        if device == self.plan.device_index:
            return self
        rep = self.replicas.get(device)
        if rep is None:
            with torch.cuda.device(device):
                qbits = getattr(self.structure, "qbits", 32)
                if self.algorithm == "direct-generic":  # gap q >= 3 (prepare_direct_gap / prepare_loaded)
                    from .persist import prepare_loaded

                    idx, _ = build(self.partition, qbits=qbits, q=self.structure.q)
                    rep = prepare_loaded(idx, self.partition)
                else:
                    rep = prepare(self.algorithm, self.partition, qbits)
            self.replicas[device] = rep
        return rep

    # -- device-level API (no host copies, no synchronisation) -------------
    def launch(self, z, out, status, base: int = 0) -> None:
        """Enqueue exactly one search kernel on the current stream.  ``z``:
        CUDA tensor of the partition's dtype; ``out``: int32/int64 CUDA
        tensor; ``status``: a workspace from ``new_status()`` whose word 0
        receives the first out-of-domain position (UINT64_MAX when clean;
        read it with ``first_bad_of``).  ``out`` is unspecified for
        out-of-domain queries.  No host synchronisation; capturable in a
        CUDA graph.  Raises ValueError for a dtype, device or layout the
        kernel cannot take as is (``_check_device_batch``).  ``base``: the
        global position of z[0] when z is a shard of a larger batch (status
        positions are then global; word 3 = word 0 XOR 2^63 orders them as
        signed int64 for a MIN all-reduce)."""
        _check_device_batch(self.plan, z, out)
        _launch_device(self.plan, z, out, status, base)

    def placement(self) -> dict:
        """Where the kernel keeps its tables: {'smem_x', 'smem_table',
        'smem_top', 'smem_bytes'}."""
        flags = ctypes.c_int32(0)
        smem = ctypes.c_uint64(0)
        _lib.check(_lib.load().fs_plan_placement(ctypes.byref(self.plan), ctypes.byref(flags), ctypes.byref(smem)))
        f = flags.value
        return {
            "smem_x": bool(f & _lib.PLACE_SMEM_X),
            "smem_table": bool(f & _lib.PLACE_SMEM_K),
            "smem_top": bool(f & _lib.PLACE_SMEM_TOP),
            "smem_hot": bool(f & _lib.PLACE_SMEM_HOT),
            "smem_sparse": bool(f & _lib.PLACE_SMEM_SPARSE),
            "sparse_format": {_lib.SPARSE_RECORDS: "records", _lib.SPARSE_RECORDS8: "records8",
                              _lib.SPARSE_RECORDS12: "records12", _lib.SPARSE_RECORDS8X3: "records8x3",
                              _lib.SPARSE_ZONED: "zoned", _lib.SPARSE_ZONED_RANK: "zoned-rank",
                              _lib.SPARSE_COUNT: "count-words", _lib.SPARSE_KNOT_BYTES: "knot-bytes", _lib.SPARSE_RANK_ROWS: "rank-rows"}.get(
                self.plan.sparse_format, "two-level") if f & _lib.PLACE_SMEM_SPARSE else None,
            "smem_bytes": int(smem.value),
            # what a search that stages nothing gathers through L2 besides X
            "l2_directory": (None if smem.value else
                             "rank-rows" if self.plan.sparse and self.plan.sparse_format == _lib.SPARSE_RANK_ROWS else
                             "rank" if self.plan.rank else None),
        }

    def launches_per_batch(self, m: int) -> int:
        """Kernels one device-resident search of m queries launches (1)."""
        return int(_lib.load().fs_search_launches(ctypes.byref(self.plan), m))

    def host_launches(self, z: np.ndarray, out: np.ndarray) -> int:
        """Kernels ``batch_search`` launches for these host arrays: one per
        chunk (fs_search_host_launches, the same chunking fs_search_host
        applies; pageable buffers go through 16 MB staging slots)."""
        z = np.ascontiguousarray(z)
        return int(_lib.load().fs_search_host_launches(
            ctypes.byref(self.plan), z.ctypes.data, len(z), out.ctypes.data, out.dtype.itemsize,
            max(4, HOST_CHUNK_BYTES // z.dtype.itemsize), 0))


@dataclass(frozen=True)
class LaneConfig:
    """Lane width, kernel name, prepared structure (batch.py:143-153).  ``d``
    is validated and otherwise has no effect on the GPU."""

    d: int
    kernel: str
    structure: PreparedKernel

    def __post_init__(self):
        if self.d < 1:
            raise ValueError("lane width must be >= 1")


def _make_callables(plan, p: SortedPartition):
    dtype = p.values.dtype

    def lanes(z):
        if _is_torch(z):
            import torch

            out = torch.empty(z.numel(), dtype=torch.int64, device=z.device)
            _search_device_tensor(plan, z.contiguous(), out)
            return out
        zz = coerce_queries(z, dtype)
        out = np.empty(len(zz), dtype=np.int64)
        _search_host_array(plan, zz, out)
        return out

    def scalar(z):
        out = np.empty(1, dtype=np.int64)
        _search_host_array(plan, coerce_queries(np.asarray([z]), dtype), out)
        return int(out[0])

    return scalar, lanes


def prepare(algorithm: str, p: SortedPartition, qbits: int = 32, *, hot_window: bool = True) -> PreparedKernel:
    """Build the device search structure for ``algorithm`` (batch.py:156-255).

    Direct-family preparation propagates NotDistinguishable/Overflow from
    index construction, as the reference does.  ``hot_window`` (direct
    only) stages the knot-densest slice of a directory too large for shared
    memory (fs_build_hot_window) when the table is skewed enough
    (HOT_WINDOW_MIN_DENSITY_RATIO); cfg4 373 -> 390 G queries/s with
    8-query groups (profiles/r01/tune_hot_window_vw8.txt).  False keeps the
    whole directory in L2.
    """
    n = p.n_intervals
    if algorithm == "classic":
        structure = p
    elif algorithm in ("bitset1", "bitset3"):
        structure = probe_constant(n)
    elif algorithm == "bitset2":
        structure = pad_right_pow2(p)
    elif algorithm == "offset":
        structure = offset_constants(n)
    elif algorithm == "eytzinger":
        structure = build_layout(p)
    elif algorithm in ("direct", "direct-gap2", "direct-cache"):
        q = 2 if algorithm == "direct-gap2" else 1
        structure, _ = build(p, qbits=qbits, q=q, fused=(algorithm == "direct-cache"))
    else:
        raise ValueError(f"unknown algorithm {algorithm!r}; pick one of {ALGORITHMS}")
    plan, keep = _plan_for(algorithm, structure, p)
    rec_bytes = 8 if p.precision == "single" else 16
    if algorithm == "direct-cache" and (structure.r + 1) * rec_bytes > SMEM_RECORDS_MAX:
        # Records that cannot be staged would be gathered 16 B at a time
        # through L2 (cfg5 N+1 = 1025: 89 G queries/s).  The cache lane's
        # answers are the gap-1 direct answers by definition (direct.py:
        # 601-610 vs 570-574), so the device plan uses direct's layouts over
        # the same index (K, rank directory, sparse table); the structure
        # and its fused host view are unchanged.
        plan.algorithm = _lib.ALGO_CODES["direct"]
        plan.table = structure.k_dev.data_ptr()
        keep.append(structure.k_dev)
    x_bytes = (len(p.values) * p.values.dtype.itemsize + 127) // 128 * 128
    if (algorithm == "direct-gap2" and structure.q == 2
            and x_bytes + (structure.r + 1) * 4 > SMEM_RECORDS_MAX and structure.r < (1 << 32)):
        # K and X cannot both be staged: a directory 8x smaller than K, X read
        # only for the knots of the query's own bucket, beats K via L2 -- the
        # count directory (8-B words of 16 buckets, 2-bit counts) over the
        # rank2 one (16-B words of 32): cfg5 N+1 = 32769 132 (K) -> 220
        # (rank2) -> 232 G queries/s, N+1 = 2^20+1 147 -> 181 (8-B gathers
        # cost fewer L1 cycles than 16-B ones; profiles/r02/tune_countdir.txt).
        # When K and X fit, plain K in smem stays faster (cfg3: 686 vs 305).
        if GAP2_DIRECTORY == "countdir":
            d = build_count_directory(p, structure)
            plan.algorithm = _lib.ALGO_CODES["direct-generic"]  # same answers (direct.py:279-300)
        else:
            d = build_rank2_directory(p, structure)
        plan.rank = d.data_ptr()
        keep.append(d)
    if plan.algorithm == _lib.ALGO_CODES["direct"] and structure.q == 1:
        set_direct_layouts(plan, p, structure, keep, hot_window)
    scalar, lanes = _make_callables(plan, p)
    return PreparedKernel(algorithm, p, structure, scalar, lanes, plan=plan, buffers=tuple(keep))


def set_direct_layouts(plan, p: SortedPartition, structure: DirectIndex, keep: list, hot_window: bool = True) -> None:
    """The device layouts of a gap-1 table K that the direct kernel can search
    instead of K itself, all with identical answers: fused records when they
    fit in shared memory, the rank directory, and -- when the directory (plus
    X) cannot be staged -- count words / group records / the two-level table
    for R >> N, zoned tables for skewed ones, else a hot window of the
    directory.  Shared by prepare() and persist.prepare_loaded()."""
    rec_bytes = 8 if p.precision == "single" else 16
    if (structure.r + 1) * rec_bytes <= SMEM_RECORDS_MAX:
        rec = _device.empty((structure.r + 1) * rec_bytes, np.uint8)
        rc = _lib.load().fs_build_fused(fs_dtype(p.precision), p.device_values().data_ptr(), len(p.values),
                                        structure.k_dev.data_ptr(), structure.r, rec.data_ptr(),
                                        _device.stream_ptr())
        _lib.check(rc, what="fs_build_fused")
        plan.records = rec.data_ptr()
        keep.append(rec)
    rank = build_rank_directory(p, structure)
    plan.rank = rank.data_ptr()
    keep.append(rank)
    if not plan.records and _set_knot_bytes(plan, p, structure, keep):
        return
    if not plan.records:
        _set_sparse_table(plan, p, structure, keep)
    if ZONED and not plan.records and not plan.sparse:
        _set_zoned(plan, p, structure, keep)
    if hot_window and not plan.sparse:
        _set_hot_window(plan, p, structure, rank)
    if not plan.records and not plan.sparse and not plan.hot_words:
        _set_rank_rows(plan, p, structure, keep)


#: the sparse two-level table is used when its dense (bitmask) super-buckets
#: hold at most this fraction of the knots
SPARSE_MAX_DENSE_KNOT_FRACTION = 0.25
#: group records are used when at most this share of uniform queries (parts
#: per million) falls past a sixth knot of its super-bucket (the slow path)
SPARSE_RECORDS_MAX_PAST_SIXTH_PPM = 20_000
#: group records replace the two-level table when its super-buckets would
#: hold at least this many knots on average (measured: cfg2 at 0.41 knots
#: per super-bucket 342 -> 413 G queries/s with records, cfg5 N+1 = 32769 at
#: 0.84: 336 -> 368; cfg5 N+1 = 1025 at 0.03 stays two-level, 484 vs 446)
SPARSE_RECORDS_MIN_LOAD = 0.2
#: 8-B group records (two offsets) are used when at most this share of
#: uniform queries (ppm) falls past a record's second knot
SPARSE_RECORDS8_MAX_PAST_PPM = 5_000
#: sparse layouts allowed; a tuning run or test may narrow it to one
#: (a leading records format also skips the load rule)
SPARSE_FORMATS = ("count-words", "two-level", "records8", "records8x3", "records", "records12")
#: Count words (fs_build_count_words), by what is staged beside them:
#: * all of X (tried before the group records): used when at most
#:   COUNT_WORDS_MAX_XREAD_PPM of the buckets lie in knot-holding stripes
#:   (cfg2 at 5%: 516 vs 496 / 436 G queries/s on group records; cfg5 N+1 =
#:   8193 at 5%: 545 vs 465; N+1 = 16385 at 21%: 455 vs 506, records stay);
#: * a byte per knot, X being too large to stage (tried after the 8-B group
#:   records, before the 16-B ones): used when at most
#:   COUNT_WORDS_MAX_RARE_PPM lie in stripes of two or more knots -- the
#:   queries that take the probe's scan path (cfg5 N+1 = 32769 at 0.4%: 452
#:   vs 430); or nothing, when at most COUNT_WORDS_MAX_L2_XREAD_PPM lie in
#:   knot-holding stripes (every knot is then read through L2);
#: * when no group record layout fits either, they replace the two-level
#:   table up to COUNT_WORDS_LATE_MAX_RARE_PPM (cfg5 N+1 = 49153 / 65537: 413
#:   / 378 vs 308 / 300), with all of shared memory.
#: profiles/r02/count_words.txt.  COUNT_WORDS_MAX_RARE_PPM = 0 skips them.
COUNT_WORDS_MAX_XREAD_PPM = 80_000
COUNT_WORDS_MAX_RARE_PPM = 10_000
COUNT_WORDS_MAX_L2_XREAD_PPM = 20_000
COUNT_WORDS_LATE_MAX_RARE_PPM = 50_000
#: shared memory the count words and what is staged beside them may take
#: before the late stage: past the 196 KB carve-out step the streaming loads
#: are left 28 KB of L1 to be in flight through, and this probe is bound by
#: their latency (cfg5 N+1 = 8193: 545 G queries/s at 142 KB with stripes
#: twice as wide, 454 at 218 KB)
COUNT_WORDS_BUDGET_BYTES = 195 * 1024
#: count words with a byte per knot (its bucket inside its stripe) staged
#: instead of an X that does not fit; False keeps the group records there
COUNT_WORDS_OFFSETS = True

#: hot-window staging budget: small enough that the L2-gather kernel keeps
#: full occupancy (3-4 CTAs per SM) for the queries outside the window
HOT_WINDOW_BYTES = 48 * 1024
#: used only for skewed tables: knots per byte inside the window at least
#: this multiple of the table-wide average (uniform layouts gain nothing)
HOT_WINDOW_MIN_DENSITY_RATIO = 4.0


#: zoned records (fs_build_zoned) are tried when neither the rank directory
#: nor a sparse layout can be staged, before the hot window; False skips
#: them (tuning, tests).  cfg4: 451 G queries/s against the hot window's 405
#: -- 449 vs 242 on its uniform half, 438 vs 510 on its clustered half
#: (profiles/r02/zoned_cfg4.txt)
ZONED = True
#: striped rank words (fs_build_zoned_rank: every zone in {mask, base} words
#: whose bits stand for 2^k-bucket stripes) are tried before the mixed
#: slot/rank records, and used when at most this share (ppm) of the buckets
#: lies in knot-holding stripes -- the uniform queries that read X.  False /
#: 0 skips them.
ZONED_RANK_MAX_XREAD_PPM = 150_000


#: planner override of the shared-memory budget in bytes (tuning: tools/tune.py --smem-kb); None = the device's
SMEM_BUDGET_OVERRIDE = None


def _smem_budget() -> int:
    import torch

    props = torch.cuda.get_device_properties(torch.cuda.current_device())
    full = int(getattr(props, "shared_memory_per_block_optin", 227 * 1024)) - 1024
    return min(full, SMEM_BUDGET_OVERRIDE) if SMEM_BUDGET_OVERRIDE else full


def _set_hot_window(plan, p: SortedPartition, idx: DirectIndex, rank) -> None:
    """When neither records nor the whole directory fit in shared memory,
    stage the directory window (and the knots it references) holding the
    most knots: queries distributed like the knots then resolve from smem
    (fs_build_hot_window)."""
    dir_bytes = ((idx.r >> 5) + 1) * 8
    if plan.records or dir_bytes <= _smem_budget() or idx.r >= (1 << 32):
        return
    out = [ctypes.c_uint64(0) for _ in range(5)]
    ws = _device.Workspace.get()
    rc = _lib.load().fs_build_hot_window(fs_dtype(p.precision), rank.data_ptr(), idx.r, HOT_WINDOW_BYTES,
                                         ws.data_ptr(), *[ctypes.byref(o) for o in out], _device.stream_ptr())
    _lib.check(rc, what="fs_build_hot_window")
    w0, nw, t0, nt, inside = (o.value for o in out)
    table_bytes = dir_bytes + p.values.dtype.itemsize * len(p.values)
    density_ratio = (inside / HOT_WINDOW_BYTES) / (p.n_intervals / table_bytes)
    if nw and density_ratio >= HOT_WINDOW_MIN_DENSITY_RATIO:
        plan.hot_word0, plan.hot_words, plan.hot_knot0, plan.hot_knots = w0, nw, t0, nt


def _set_zoned(plan, p: SortedPartition, idx: DirectIndex, keep: list) -> None:
    """Zoned records of K (fs_build_zoned): the buckets cut into at most 64
    zones, each zone in the 8-B record form its knot density needs (slot
    records of 2^6..2^11 buckets holding at most three 13-bit knot offsets,
    or 32-bucket rank words), plus a window of the densest knots.  For tables whose
    density varies by orders of magnitude (cfg4's geometric knots: one
    record shift for the whole table overflows at its dense end and exceeds
    shared memory at its sparse end) the whole directory then fits in shared
    memory.  Used when the rank directory cannot be staged, not even
    without X."""
    dir_bytes = ((idx.r >> 5) + 1) * 8
    budget = _smem_budget() - 512
    if idx.r >= (1 << 32) or len(p.values) >= (1 << 31) or dir_bytes <= budget:
        return  # the staged rank directory (X through L2 for knot buckets only) wins
    lib = _lib.load()
    dt = fs_dtype(p.precision)
    n1 = len(p.values)
    x = p.device_values()
    f = _device.empty(n1, np.uint64)
    zs, nrec, nbytes, t0, nt = ctypes.c_int32(-1), *(ctypes.c_uint64(0) for _ in range(4))
    if ZONED_RANK_MAX_XREAD_PPM:
        ppm = ctypes.c_uint64(0)
        rc = lib.fs_plan_zoned_rank(dt, x.data_ptr(), n1, float(idx.h), idx.r, budget, f.data_ptr(), ctypes.byref(zs),
                                    ctypes.byref(nrec), ctypes.byref(nbytes), ctypes.byref(t0), ctypes.byref(nt),
                                    ctypes.byref(ppm), _device.stream_ptr())
        if rc != _lib.FS_TOO_LARGE:
            _lib.check(rc, what="fs_plan_zoned_rank")
        if rc == _lib.FS_OK and ppm.value <= ZONED_RANK_MAX_XREAD_PPM:
            buf = _device.empty(int(nbytes.value), np.uint8)
            rc = lib.fs_build_zoned_rank(dt, x.data_ptr(), n1, float(idx.h), idx.r, zs.value, nrec.value,
                                         f.data_ptr(), buf.data_ptr(), _device.stream_ptr())
            _lib.check(rc, what="fs_build_zoned_rank")
            plan.sparse = buf.data_ptr()
            plan.sparse_format = _lib.SPARSE_ZONED_RANK
            plan.sparse_shift = zs.value
            plan.sparse_ndense = nrec.value
            plan.hot_word0, plan.hot_words = 0, 0
            plan.hot_knot0, plan.hot_knots = t0.value, nt.value
            keep.append(buf)
            return
    rc = lib.fs_plan_zoned(dt, x.data_ptr(), n1, float(idx.h), idx.r, budget, f.data_ptr(), ctypes.byref(zs),
                           ctypes.byref(nrec), ctypes.byref(nbytes), ctypes.byref(t0), ctypes.byref(nt),
                           _device.stream_ptr())
    if rc == _lib.FS_TOO_LARGE:
        return
    _lib.check(rc, what="fs_plan_zoned")
    buf = _device.empty(int(nbytes.value), np.uint8)
    rc = lib.fs_build_zoned(dt, x.data_ptr(), n1, float(idx.h), idx.r, zs.value, f.data_ptr(), buf.data_ptr(),
                            _device.stream_ptr())
    _lib.check(rc, what="fs_build_zoned")
    plan.sparse = buf.data_ptr()
    plan.sparse_format = _lib.SPARSE_ZONED
    plan.sparse_shift = zs.value
    plan.sparse_ndense = nrec.value
    plan.hot_word0, plan.hot_words = 0, 0
    plan.hot_knot0, plan.hot_knots = t0.value, nt.value
    keep.append(buf)


def _set_b2_deep(plan, pp: PaddedPartition, keep: list) -> None:
    """bitset2 levels below the shared-memory top as 32-B subtree records
    (fs_build_b2_deep): one gather per 2 (f64) / 3 (f32) levels instead of
    one per level.  Same comparisons as binsearch.py:72-86."""
    lib = _lib.load()
    dt = fs_dtype(pp.base.precision)
    top, k = ctypes.c_int32(0), ctypes.c_int32(0)
    nbytes = int(lib.fs_b2_deep_bytes(dt, pp.p, ctypes.byref(top), ctypes.byref(k)))
    if nbytes == 0:
        return
    buf = _device.empty(nbytes, np.uint8)
    rc = lib.fs_build_b2_deep(dt, pp.padded_dev.data_ptr(), pp.p, top.value, k.value, buf.data_ptr(),
                              _device.stream_ptr())
    _lib.check(rc, what="fs_build_b2_deep")
    plan.b2_deep = buf.data_ptr()
    plan.b2_deep_top = top.value
    plan.b2_deep_k = k.value
    keep.append(buf)


def _set_sparse_records(plan, p: SortedPartition, idx: DirectIndex, keep: list, f, budget: int, name: str,
                        with_x: tuple = (1, 0)) -> bool:
    """Group records of K (fs_build_sparse_rec): one record per super-bucket
    resolves K[j] with a single shared-memory load ("records8": 8 B, two knot
    offsets; "records8x3": 8 B, three 13-bit offsets, super-buckets of at
    most 2^11 buckets; "records": 16 B, six; "records12": 16 B, eight 12-bit
    offsets, super-buckets of at most 2^10 buckets).  Used when they fit and few uniform queries
    fall past a record's last offset; X is staged beside them (with_x 1) or
    read through L2 for the buckets holding a knot (with_x 0)."""
    lib = _lib.load()
    dt = fs_dtype(p.precision)
    n1 = len(p.values)
    x = p.device_values()
    fmt, max_ppm = {"records8": (_lib.SPARSE_RECORDS8, SPARSE_RECORDS8_MAX_PAST_PPM),
                    "records": (_lib.SPARSE_RECORDS, SPARSE_RECORDS_MAX_PAST_SIXTH_PPM),
                    "records12": (_lib.SPARSE_RECORDS12, SPARSE_RECORDS_MAX_PAST_SIXTH_PPM),
                    "records8x3": (_lib.SPARSE_RECORDS8X3, SPARSE_RECORDS8_MAX_PAST_PPM)}[name]
    for wx in with_x:
        shift, novf, nbytes, ppm = ctypes.c_int32(-1), ctypes.c_uint64(0), ctypes.c_uint64(0), ctypes.c_uint32(0)
        rc = lib.fs_plan_sparse_rec(fmt, dt, x.data_ptr(), n1, float(idx.h), idx.r, budget, wx, f.data_ptr(),
                                    ctypes.byref(shift), ctypes.byref(novf), ctypes.byref(nbytes), ctypes.byref(ppm),
                                    _device.stream_ptr())
        if rc == _lib.FS_TOO_LARGE:
            continue
        _lib.check(rc, what="fs_plan_sparse_rec")
        if ppm.value > max_ppm:
            continue
        buf = _device.empty(int(nbytes.value), np.uint8)
        rc = lib.fs_build_sparse_rec(fmt, dt, x.data_ptr(), n1, float(idx.h), idx.r, shift.value, novf.value,
                                     f.data_ptr(), buf.data_ptr(), _device.stream_ptr())
        _lib.check(rc, what="fs_build_sparse_rec")
        plan.sparse = buf.data_ptr()
        plan.sparse_shift = shift.value
        plan.sparse_ndense = novf.value
        plan.sparse_format = fmt
        keep.append(buf)
        return True
    return False


def _records_ppm(p: SortedPartition, idx: DirectIndex, f, budget: int, fmt: int, with_x: int):
    """Queries (ppm, uniform) past the last recorded offset for the record
    layout fs_plan_sparse_rec would pick, or None if none fits."""
    lib = _lib.load()
    shift, novf, nbytes, ppm = ctypes.c_int32(-1), ctypes.c_uint64(0), ctypes.c_uint64(0), ctypes.c_uint32(0)
    rc = lib.fs_plan_sparse_rec(fmt, fs_dtype(p.precision), p.device_values().data_ptr(), len(p.values),
                                float(idx.h), idx.r, budget, with_x, f.data_ptr(), ctypes.byref(shift),
                                ctypes.byref(novf), ctypes.byref(nbytes), ctypes.byref(ppm), _device.stream_ptr())
    if rc == _lib.FS_TOO_LARGE:
        return None
    _lib.check(rc, what="fs_plan_sparse_rec")
    return ppm.value


def _plan_two_level(p: SortedPartition, idx: DirectIndex, f, budget: int):
    """fs_plan_sparse with X staged if possible: (shift, ndense, bytes) or None."""
    lib = _lib.load()
    x = p.device_values()
    shift, ndense, nbytes = ctypes.c_int32(-1), ctypes.c_uint64(0), ctypes.c_uint64(0)
    for with_x in (1, 0):  # X staged beside the table if possible, else X via L2
        rc = lib.fs_plan_sparse(fs_dtype(p.precision), x.data_ptr(), len(p.values), float(idx.h), idx.r, budget,
                                with_x, f.data_ptr(), ctypes.byref(shift), ctypes.byref(ndense), ctypes.byref(nbytes),
                                _device.stream_ptr())
        if rc == _lib.FS_OK:
            return shift.value, ndense.value, nbytes.value
        if rc != _lib.FS_TOO_LARGE:
            _lib.check(rc, what="fs_plan_sparse")
    return None


#: 16-B rank rows (fs_build_rank_rows: the directory word and the knot bytes of
#: its first eight knots in one gather) for tables searched through L2, when at
#: least this share of the buckets holds a knot (the queries that would gather
#: X as well); 0 keeps the 8-B directory
RANK_ROWS_MIN_KNOT_SHARE = 0.03


def _set_rank_rows(plan, p: SortedPartition, idx: DirectIndex, keep: list) -> None:
    """Tables whose directory and X both stay in L2 (neither fits in shared
    memory): widen the directory word to a 16-B row carrying its knots' bytes."""
    n1 = len(p.values)
    budget = _smem_budget() - 512
    dir_bytes = ((idx.r >> 5) + 1) * 8
    x_bytes = n1 * p.values.dtype.itemsize
    if (not RANK_ROWS_MIN_KNOT_SHARE or idx.r >= (1 << 32) or n1 >= (1 << 31) or dir_bytes <= budget
            or x_bytes <= budget or n1 < RANK_ROWS_MIN_KNOT_SHARE * (idx.r + 1)):
        return
    f = _device.empty(n1, np.uint64)
    scratch = _device.empty((n1 + 15) // 16 * 16, np.uint8)
    rows = _device.empty(2 * dir_bytes, np.uint8)
    rc = _lib.load().fs_build_rank_rows(fs_dtype(p.precision), p.device_values().data_ptr(), n1, float(idx.h), idx.r,
                                        f.data_ptr(), scratch.data_ptr(), rows.data_ptr(), _device.stream_ptr())
    _lib.check(rc, what="fs_build_rank_rows")
    plan.sparse = rows.data_ptr()
    plan.sparse_format = _lib.SPARSE_RANK_ROWS
    plan.sparse_shift = 0
    plan.sparse_ndense = 0
    keep.append(rows)


#: a byte per knot staged beside the rank directory when X does not fit there
#: (fs_build_knot_bytes); False keeps the directory alone, X through L2
KNOT_BYTES = True


def _set_knot_bytes(plan, p: SortedPartition, idx: DirectIndex, keep: list) -> bool:
    """Tables whose rank directory fits in shared memory but whose X does not:
    stage a byte per knot -- where inside its bucket the knot falls, to 1/256,
    from the same rounded product the bucket index comes from -- and read X
    through L2 only when the query's byte ties with the knot's."""
    n1 = len(p.values)
    budget = _smem_budget() - 512
    dir_bytes = ((idx.r >> 5) + 1) * 8
    x_bytes = (n1 * p.values.dtype.itemsize + 127) // 128 * 128
    nbytes = (n1 + 15) // 16 * 16
    if (not KNOT_BYTES or idx.r >= (1 << 32) or n1 >= (1 << 31) or x_bytes + dir_bytes <= budget
            or (nbytes + 127) // 128 * 128 + dir_bytes > budget):
        return False
    buf = _device.empty(nbytes, np.uint8)
    rc = _lib.load().fs_build_knot_bytes(fs_dtype(p.precision), p.device_values().data_ptr(), n1, float(idx.h),
                                         buf.data_ptr(), _device.stream_ptr())
    _lib.check(rc, what="fs_build_knot_bytes")
    plan.sparse = buf.data_ptr()
    plan.sparse_format = _lib.SPARSE_KNOT_BYTES
    plan.sparse_shift = 0
    plan.sparse_ndense = n1
    keep.append(buf)
    return True


def _set_count_words(plan, p: SortedPartition, idx: DirectIndex, keep: list, f, budget: int, modes=(1,),
                     late: bool = False) -> bool:
    """Count words of K (fs_build_count_words): 8-B words of sixteen 2^k-bucket
    stripes with a 2-bit knot count each, one k for the table; a popcount
    decode, one compare when the query's stripe holds a knot, a short scan
    when it holds several.  Staged beside all of X (mode 1), beside a byte
    per knot -- its bucket inside its stripe, so that X is read through L2
    only for a knot in the query's own bucket (mode 2) -- or alone (mode 0).
    Used when the rank directory and X cannot be staged together and the
    table's statistics pass the COUNT_WORDS_* bounds; ``late`` = nothing but
    the two-level table is left to try.  ``f``: n1 uint64 scratch."""
    n1 = len(p.values)
    x_bytes = (n1 * p.values.dtype.itemsize + 127) // 128 * 128
    if x_bytes + ((idx.r >> 5) + 1) * 8 <= budget:
        return False  # the staged rank directory + X: one knot per mask bit, no scan path
    lib = _lib.load()
    dt = fs_dtype(p.precision)
    x = p.device_values()
    k = ctypes.c_int32(-1)
    nbytes, xread, rare = (ctypes.c_uint64(0) for _ in range(3))
    if not late:
        budget = min(budget, COUNT_WORDS_BUDGET_BYTES)
    for mode in modes:
        if mode == 2 and not COUNT_WORDS_OFFSETS:
            continue
        rc = lib.fs_plan_count_words(dt, x.data_ptr(), n1, float(idx.h), idx.r, budget, mode, f.data_ptr(),
                                     ctypes.byref(k), ctypes.byref(nbytes), ctypes.byref(xread), ctypes.byref(rare),
                                     _device.stream_ptr())
        if rc == _lib.FS_TOO_LARGE:
            continue
        _lib.check(rc, what="fs_plan_count_words")
        if late:
            ok = rare.value <= COUNT_WORDS_LATE_MAX_RARE_PPM
        else:
            ok = rare.value <= COUNT_WORDS_MAX_RARE_PPM and xread.value <= {
                1: COUNT_WORDS_MAX_XREAD_PPM, 2: 10**6, 0: COUNT_WORDS_MAX_L2_XREAD_PPM}[mode]
        if ok:
            break
    else:
        return False
    buf = _device.empty(int(nbytes.value), np.uint8)
    rc = lib.fs_build_count_words(dt, x.data_ptr(), n1, float(idx.h), idx.r, k.value, int(mode == 2),
                                  f.data_ptr(), buf.data_ptr(), _device.stream_ptr())
    _lib.check(rc, what="fs_build_count_words")
    plan.sparse = buf.data_ptr()
    plan.sparse_format = _lib.SPARSE_COUNT
    plan.sparse_shift = k.value
    plan.sparse_ndense = n1 if mode == 2 else 0
    keep.append(buf)
    return True


def _set_sparse_table(plan, p: SortedPartition, idx: DirectIndex, keep: list) -> None:
    """For R >> N, a sparse encoding of K fits in shared memory where the
    rank directory does not; the kernel picks it over L2 gathers when the
    directory (plus X) cannot be staged.  Two layouts: the two-level table
    (fs_build_sparse; a short search per query, cheapest when super-buckets
    are nearly empty) and group records (fs_build_sparse_rec; one 8-B or 16-B
    record load plus fixed arithmetic per query).  Measured per config:
    profiles/r01/tune_sparse_records.txt."""
    if idx.r >= (1 << 32) or len(p.values) >= (1 << 31):
        return
    lib = _lib.load()
    budget = _smem_budget() - 512
    n1 = len(p.values)
    f = _device.empty(n1, np.uint64)
    # In order: 8-B records (two, then three offsets) with X staged; the two-level table when its
    # super-buckets are nearly empty; 16-B records with X (eight 12-bit
    # offsets when that sends fewer queries past the last offset, else six
    # 16-bit ones); then 8-B and 16-B records with X read through L2 (fine
    # for uniform queries, but streams with many exact-knot queries, like
    # cfg2's 1%, lose: 433 -> 423).
    count_words = "count-words" in SPARSE_FORMATS and COUNT_WORDS_MAX_RARE_PPM
    if count_words and _set_count_words(plan, p, idx, keep, f, budget, (1,)):
        return

    def records(name, wx):
        return name in SPARSE_FORMATS and _set_sparse_records(plan, p, idx, keep, f, budget, name, wx)

    def wide_records(wx):
        """16-B records: the 8- or 6-offset layout with fewer slow-path queries."""
        names = [n for n in ("records12", "records") if n in SPARSE_FORMATS]
        if len(names) == 2:
            a = _records_ppm(p, idx, f, budget, _lib.SPARSE_RECORDS12, wx)
            b = _records_ppm(p, idx, f, budget, _lib.SPARSE_RECORDS, wx)
            if a is not None and (b is None or a < b):
                names = ["records12", "records"]
            else:
                names = ["records", "records12"]
        return any(records(n, (wx,)) for n in names)

    if records("records8", (1,)) or records("records8x3", (1,)):
        return
    two = _plan_two_level(p, idx, f, budget) if "two-level" in SPARSE_FORMATS else None
    load = n1 / ((idx.r >> two[0]) + 1) if two else None
    if load is None or load >= SPARSE_RECORDS_MIN_LOAD:
        if wide_records(1) or records("records8", (0,)) or records("records8x3", (0,)):
            return
        if count_words and _set_count_words(plan, p, idx, keep, f, budget, (2, 0)):
            return
        if wide_records(0):
            return
    if count_words and _set_count_words(plan, p, idx, keep, f, budget, (1, 2), late=True):
        return
    if two is None:
        return
    shift, ndense, nbytes = two
    x = p.device_values()
    buf = _device.empty(int(nbytes), np.uint8)
    rc = lib.fs_build_sparse(fs_dtype(p.precision), x.data_ptr(), n1, float(idx.h), idx.r, shift, f.data_ptr(),
                             buf.data_ptr(), _device.stream_ptr())
    _lib.check(rc, what="fs_build_sparse")
    if ndense:
        # queries in dense super-buckets still read X through L2 for almost
        # every bucket; when those regions hold many knots (cfg4's start:
        # 31%) the L2-gather kernel at full occupancy is faster (measured
        # 354 vs 214 Gq/s), so the sparse table is kept for mostly-sparse
        # layouts only
        import torch

        c = buf[: 4 * ((idx.r >> shift) + 2)].view(torch.int32).long() & 0x7FFFFFFF
        occ = c[1:] - c[:-1]
        if int(occ[occ > 64].sum().item()) > SPARSE_MAX_DENSE_KNOT_FRACTION * n1:
            return
    plan.sparse = buf.data_ptr()
    plan.sparse_shift = shift
    plan.sparse_ndense = ndense
    plan.sparse_format = _lib.SPARSE_TWO_LEVEL
    keep.append(buf)


def build_rank_directory(p: SortedPartition, idx: DirectIndex):
    """Device rank directory of the gap-1 table (fs_build_rank): K in 2 bits
    per bucket, 8-B words {mask, K[32w]}.  The search kernel recovers K[j]
    exactly from it and skips the X comparison for buckets without a knot."""
    x = p.device_values()
    f = _device.empty(len(p.values), np.uint64)
    words = (idx.r >> 5) + 1
    d = _device.empty(2 * words, np.uint32)
    rc = _lib.load().fs_build_rank(fs_dtype(p.precision), x.data_ptr(), len(p.values), float(idx.h), idx.r,
                                   f.data_ptr(), d.data_ptr(), _device.stream_ptr())
    _lib.check(rc, what="fs_build_rank")
    return d


def build_rank2_directory(p: SortedPartition, idx: DirectIndex):
    """Device rank directory of the gap-2 table (fs_build_rank2): 16-B words
    {m1, m2, K-count base, 0} per 32 buckets (a gap-2 bucket holds at most
    two knots).  The kernel recovers K2[j] exactly and reads X only for
    buckets holding knots."""
    x = p.device_values()
    f = _device.empty(len(p.values), np.uint64)
    words = (idx.r >> 5) + 1
    d = _device.empty(4 * words, np.uint32)
    rc = _lib.load().fs_build_rank2(fs_dtype(p.precision), x.data_ptr(), len(p.values), float(idx.h), idx.r,
                                    f.data_ptr(), d.data_ptr(), _device.stream_ptr())
    _lib.check(rc, what="fs_build_rank2")
    return d


def build_count_directory(p: SortedPartition, idx: DirectIndex):
    """Device count directory of a gap-q table, q = 2..15 (fs_build_countdir):
    8-B words {2- or 4-bit knot counts of 16 / 8 buckets, knots before the
    word}.  The kernel recovers K_q[j] exactly and compares z only with the
    knots of its own bucket (direct.py:294-300)."""
    lib = _lib.load()
    x = p.device_values()
    f = _device.empty(len(p.values), np.uint64)
    nbytes = int(lib.fs_countdir_bytes(idx.q, idx.r))
    d = _device.empty(nbytes // 4, np.uint32)
    rc = lib.fs_build_countdir(fs_dtype(p.precision), x.data_ptr(), len(p.values), float(idx.h), idx.r, idx.q,
                               f.data_ptr(), d.data_ptr(), _device.stream_ptr())
    _lib.check(rc, what="fs_build_countdir")
    return d


def prepare_direct_gap(p: SortedPartition, q: int, qbits: int = 32, idx: DirectIndex | None = None) -> PreparedKernel:
    """Direct search with gap q >= 2 over its count directory -- the
    reference's direct_search_generic (direct.py:294-300) as a batch kernel
    ("direct-generic"; the reference has no lane kernel for q > 2).  Raises
    the index build's InfeasibleError like ``prepare``."""
    if not 2 <= q <= 15:
        raise ValueError("count directories serve gaps 2..15")
    if idx is None:
        idx, _ = build(p, qbits=qbits, q=q)
    plan, keep = _plan_for("direct-generic", idx, p)
    if idx.r < (1 << 32):
        d = build_count_directory(p, idx)
        plan.rank = d.data_ptr()
        keep.append(d)
    scalar, lanes = _make_callables(plan, p)
    return PreparedKernel("direct-generic", p, idx, scalar, lanes, plan=plan, buffers=tuple(keep))


#: directory of a gap-2 table that cannot be staged: "countdir" or "rank2"
GAP2_DIRECTORY = "countdir"
#: gap-q fall-back: largest count directory accepted (it should stay L2-resident)
GAP_FALLBACK_MAX_DIR_BYTES = 64 << 20
#: gap-q fall-back: largest gap tried (4-bit counts)
GAP_FALLBACK_MAX_Q = 15


def prepare_with_fallback(p: SortedPartition, qbits: int = 32, algorithm: str = "direct",
                          fallback: str = "bitset2", gap_fallback: bool = True) -> PreparedKernel:
    """Direct search when its index is feasible, else a fall-back -- the
    paper's policy (the reference leaves it to its harness,
    bench/harness.py:153-159).

    The fall-back, in order: when the padded array fits in shared memory,
    the padded bit-set binary search (fast there); otherwise the direct
    search with the smallest gap q in 2..15 whose certified layout is
    feasible and whose count directory stays L2-resident
    (GAP_FALLBACK_MAX_DIR_BYTES) -- the paper's generalisation to gap q
    "deriving the minimal number of q which achieves a given memory budget"
     -- and else ``fallback`` (bitset2).  Every path returns
    the same unique answers."""
    try:
        return prepare(algorithm, p, qbits)
    except InfeasibleError:
        pass
    es = p.values.dtype.itemsize
    pad_bytes = (1 << p.n_intervals.bit_length()) * es
    if gap_fallback and pad_bytes > _smem_budget():
        from .direct import compute_h_r

        lib = _lib.load()
        for q in range(2, min(GAP_FALLBACK_MAX_Q, p.n_intervals) + 1):
            try:
                h, r, _ = compute_h_r(p, qbits=qbits, q=q)
            except InfeasibleError:
                continue
            if r >= (1 << 32) or int(lib.fs_countdir_bytes(q, r)) > GAP_FALLBACK_MAX_DIR_BYTES:
                continue
            from .direct import build_index

            return prepare_direct_gap(p, q, qbits, idx=build_index(p, h, r, q=q, qbits=qbits))
    return prepare(fallback, p, qbits)


def resolve_threads(threads: int | None) -> int:
    """batch.py:376-382 (validated; the GPU path does not use host threads)."""
    if threads is not None:
        if threads < 1:
            raise ValueError("thread count must be >= 1")
        return threads
    env = os.environ.get(THREADS_ENV)
    return max(1, int(env)) if env else 1


def batch_search(cfg: LaneConfig, queries, out, threads: int | None = None, *, atomic: bool = True,
                 devices=None) -> int:
    """Resolve every query into ``out``; returns the number resolved
    (batch.py:399-441).

    Raises OutOfDomain(position) for the first query outside [X_0, X_N);
    a host ``out`` is left untouched in that case.  ``atomic=False`` (not in
    the reference) relaxes only that last guarantee for host arrays: results
    are written back chunk by chunk while later chunks are still uploading,
    overlapping the two PCIe directions (~2x end to end); the exception and
    its position are unchanged.

    ``devices`` (not in the reference; host arrays only): CUDA device
    indices to split the batch over -- contiguous spans, one per entry, as
    the reference splits spans over threads (batch.py:385-396, 428-440).
    Each device searches its span with its own replica of the structure and
    its own PCIe link; the spans share a gate, so an OutOfDomain anywhere
    still leaves all of ``out`` untouched (atomic mode) and reports the
    batch's first bad position.  ``"all"`` = every visible device.
    """
    kern = cfg.structure
    resolve_threads(threads)
    if isinstance(queries, QueryBatch):
        z = queries.values
    elif _is_torch(queries):
        z = queries
    else:
        z = np.asarray(queries)
    m = len(z)
    if len(out) < m:
        raise ValueError("output array is smaller than the query batch")
    p = kern.partition
    if _is_torch(z) or _is_torch(out):
        import torch

        if not (_is_torch(z) and _is_torch(out) and z.is_cuda and out.is_cuda):
            raise ValueError("device-resident batches need CUDA tensors for both queries and out")
        if z.dtype != _device.torch_dtype(p.values.dtype):
            raise ValueError(f"query dtype {z.dtype} does not match the partition's {p.values.dtype}")
        if out.dtype not in (torch.int32, torch.int64):
            raise ValueError("out must be int32 or int64")
        o = out[:m]
        if o.is_contiguous():
            _search_device_tensor(kern.plan, z.contiguous(), o)
        else:  # any writable view, as the reference's slice assignment allows (batch.py:423)
            tmp = torch.empty(m, dtype=out.dtype, device=out.device)
            _search_device_tensor(kern.plan, z.contiguous(), tmp)
            o.copy_(tmp)
        return m
    zz = coerce_queries(z, p.values.dtype)
    if devices is not None:
        devs = _resolve_devices(devices)
        if len(devs) > 1 and m > 0:
            if isinstance(out, np.ndarray):
                _search_host_spans(kern, zz, out, devs, overlap=not atomic)
            else:
                tmp = np.empty(m, dtype=np.int64)
                _search_host_spans(kern, zz, tmp, devs, overlap=not atomic)
                out[:m] = tmp.tolist()
            return m
        import torch

        with torch.cuda.device(devs[0]):
            return batch_search(LaneConfig(cfg.d, cfg.kernel, kern.on_device(devs[0])), zz, out, threads,
                                atomic=atomic)
    if isinstance(out, np.ndarray):
        _search_host_array(kern.plan, zz, out, overlap=not atomic)
    else:  # any mutable sequence, as the reference's slice assignment allows (batch.py:423)
        tmp = np.empty(m, dtype=np.int64)
        _search_host_array(kern.plan, zz, tmp)
        out[:m] = tmp.tolist()
    return m


def _resolve_devices(devices) -> list:
    import torch

    if isinstance(devices, str):
        if devices != "all":
            raise ValueError('devices must be a sequence of CUDA device indices or "all"')
        devs = list(range(torch.cuda.device_count()))
    else:
        devs = [int(getattr(d, "index", d) if not isinstance(d, int) else d) for d in devices]
    if not devs:
        raise ValueError("devices is empty")
    n = torch.cuda.device_count()
    for d in devs:
        if not 0 <= d < n:
            raise ValueError(f"no CUDA device {d} (visible: {n})")
    return devs


_span_pool = None
_span_pool_lock = threading.Lock()


def _span_executor(n: int):
    """Persistent threads that drive one span each (the native call of a span
    releases the GIL and blocks until its span is done)."""
    global _span_pool
    from concurrent.futures import ThreadPoolExecutor

    with _span_pool_lock:
        if _span_pool is None or _span_pool._max_workers < n:
            _span_pool = ThreadPoolExecutor(max_workers=max(n, 8), thread_name_prefix="fs-span")
        return _span_pool


def _search_host_spans(kern: PreparedKernel, z: np.ndarray, out: np.ndarray, devices: list, overlap: bool) -> None:
    """One host batch over several devices: contiguous spans (8-query
    granularity, dist.shard_span), one gated fs_search_host call per span on
    its device, concurrently.  Raises OutOfDomain(first bad position of the
    whole batch); in atomic mode nothing is written then (fs_gate)."""
    import torch

    from .dist import shard_span
    from .errors import SpanAborted

    m = len(z)
    lib = _lib.load()
    devices = devices[: max(1, min(len(devices), m // 8))]  # no empty spans: every party makes its call
    n = len(devices)
    spans = [shard_span(m, i, n, granularity=8) for i in range(n)]
    reps = {d: kern.on_device(d) for d in set(devices)}  # built before any span starts (no gate held)
    gate = lib.fs_gate_create(n)
    if not gate:
        raise MemoryError("fs_gate_create failed")

    def run(i):
        a, b = spans[i]
        called = False
        try:
            torch.cuda.set_device(devices[i])
            called = True  # from here on the native call arrives at the gate on every path
            _search_host_array(reps[devices[i]].plan, z[a:b], out[a:b], overlap=overlap, gate=gate)
            return None
        except OutOfDomain as e:
            return ("bad", a + int(e.position))
        except SpanAborted:
            return ("aborted", None)
        except BaseException as e:  # noqa: BLE001 -- reported after every span returned
            if not called:
                lib.fs_gate_abort(gate)
            return ("error", e)

    try:
        results = list(_span_executor(n).map(run, range(n)))
    finally:
        lib.fs_gate_destroy(gate)
    errors = [r[1] for r in results if r and r[0] == "error"]
    if errors:
        raise errors[0]
    bad = [r[1] for r in results if r and r[0] == "bad"]
    if bad:
        raise OutOfDomain(position=min(bad))


def run_batch(prepared: PreparedKernel, queries, d: int = 1, threads: int | None = None):
    """Allocate an int64 output and run batch_search (batch.py:444-451)."""
    if isinstance(queries, QueryBatch):
        z = queries.values
    elif _is_torch(queries):
        import torch

        out = torch.empty(len(queries), dtype=torch.int64, device=queries.device)
        batch_search(LaneConfig(d=d, kernel=prepared.algorithm, structure=prepared), queries, out, threads)
        return out
    else:
        z = np.asarray(queries)
    out = np.empty(len(z), dtype=np.int64)
    batch_search(LaneConfig(d=d, kernel=prepared.algorithm, structure=prepared), z, out, threads)
    return out
