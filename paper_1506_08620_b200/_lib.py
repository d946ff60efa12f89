"""ctypes binding of the C-ABI in ``include/fsgpu.h`` (``libfsgpu.so``).

This is the whole native boundary: plain pointers, sizes and an ``fs_plan``
struct; torch only supplies device memory and the current stream.  The
library is loaded from the package directory (built in-tree by
``__graft_entry__.build()``); if it is missing the import of any compute
entry point raises immediately -- there is no CPU fallback.
"""

from __future__ import annotations

import ctypes
import os
import threading
from pathlib import Path

from .errors import DeviceError, NotDistinguishable, OutOfDomain, Overflow, SpanAborted

LIB_NAME = "libfsgpu.so"
LIB_PATH = Path(__file__).with_name(LIB_NAME)

# status codes (fsgpu.h: fs_status)
FS_OK = 0
FS_NOT_DISTINGUISHABLE = 1
FS_OVERFLOW = 2
FS_OUT_OF_DOMAIN = 3
FS_INVALID_ARG = 4
FS_CUDA_ERROR = 5
FS_INCONSISTENT = 6
FS_TOO_LARGE = 7
FS_ABORTED = 8

FS_F32 = 0
FS_F64 = 1

FS_HOST_OVERLAP = 1
FS_HOST_NO_STAGING = 2
FS_HOST_NO_PRECHECK = 4

ALGO_CODES = {
    "classic": 0,
    "bitset1": 1,
    "bitset2": 2,
    "bitset3": 3,
    "offset": 4,
    "eytzinger": 5,
    "direct": 6,
    "direct-gap2": 7,
    "direct-cache": 8,
    "direct-generic": 9,
}

PLACE_SMEM_X = 1
PLACE_SMEM_K = 2
PLACE_SMEM_TOP = 4
PLACE_SMEM_HOT = 8
PLACE_SMEM_SPARSE = 16
SPARSE_TWO_LEVEL = 0
SPARSE_RECORDS = 1
SPARSE_RECORDS8 = 2
SPARSE_RECORDS12 = 3
SPARSE_RECORDS8X3 = 4
SPARSE_ZONED = 5
SPARSE_ZONED_RANK = 6
SPARSE_COUNT = 7
SPARSE_KNOT_BYTES = 8
SPARSE_RANK_ROWS = 9

# Every symbol include/fsgpu.h declares (checked by the CPU test suite).
EXPORTED = (
    "fs_version",
    "fs_last_error",
    "fs_workspace_bytes",
    "fs_certify",
    "fs_knot_buckets",
    "fs_build_table",
    "fs_build_rank",
    "fs_sparse_bytes",
    "fs_plan_sparse",
    "fs_build_sparse",
    "fs_sparse_rec_bytes",
    "fs_plan_sparse_rec",
    "fs_build_sparse_rec",
    "fs_build_hot_window",
    "fs_zoned_bytes",
    "fs_plan_zoned",
    "fs_build_zoned",
    "fs_plan_zoned_rank",
    "fs_build_zoned_rank",
    "fs_build_knot_bytes",
    "fs_build_rank_rows",
    "fs_count_words_bytes",
    "fs_plan_count_words",
    "fs_build_count_words",
    "fs_build_fused",
    "fs_build_padded",
    "fs_build_rank2",
    "fs_countdir_bytes",
    "fs_build_countdir",
    "fs_b2_deep_bytes",
    "fs_build_b2_deep",
    "fs_build_eytzinger",
    "fs_search_ws_words",
    "fs_search_device",
    "fs_search_device_at",
    "fs_search_host",
    "fs_search_host_gated",
    "fs_gate_create",
    "fs_gate_abort",
    "fs_gate_destroy",
    "fs_crc32_ws_bytes",
    "fs_crc32",
    "fs_plan_placement",
    "fs_search_launches",
    "fs_search_host_launches",
)


class FsPlan(ctypes.Structure):
    """Mirror of ``struct fs_plan`` (fsgpu.h)."""

    _fields_ = [
        ("algorithm", ctypes.c_int32),
        ("dtype", ctypes.c_int32),
        ("n1", ctypes.c_uint64),
        ("x", ctypes.c_void_p),
        ("table", ctypes.c_void_p),
        ("r", ctypes.c_uint64),
        ("h", ctypes.c_double),
        ("x0", ctypes.c_double),
        ("xn", ctypes.c_double),
        ("q", ctypes.c_int32),
        ("pbits", ctypes.c_int32),
        ("smem_policy", ctypes.c_int32),
        ("tune", ctypes.c_int32),
        ("rank", ctypes.c_void_p),
        ("records", ctypes.c_void_p),
        ("hot_word0", ctypes.c_uint64),
        ("hot_words", ctypes.c_uint64),
        ("hot_knot0", ctypes.c_uint64),
        ("hot_knots", ctypes.c_uint64),
        ("sparse", ctypes.c_void_p),
        ("sparse_shift", ctypes.c_int32),
        ("sparse_ndense", ctypes.c_uint32),
        ("b2_deep", ctypes.c_void_p),
        ("b2_deep_top", ctypes.c_int32),
        ("b2_deep_k", ctypes.c_int32),
        ("sparse_format", ctypes.c_int32),
    ]


_lock = threading.Lock()
_lib = None

_u64 = ctypes.c_uint64
_i32 = ctypes.c_int32
_vp = ctypes.c_void_p
_p_u64 = ctypes.POINTER(ctypes.c_uint64)
_p_i64 = ctypes.POINTER(ctypes.c_int64)
_p_u32 = ctypes.POINTER(ctypes.c_uint32)
_p_i32 = ctypes.POINTER(ctypes.c_int32)


def _declare(lib):
    lib.fs_version.restype = ctypes.c_char_p
    lib.fs_version.argtypes = []
    lib.fs_last_error.restype = ctypes.c_char_p
    lib.fs_last_error.argtypes = []
    lib.fs_workspace_bytes.restype = ctypes.c_size_t
    lib.fs_workspace_bytes.argtypes = []
    lib.fs_certify.restype = ctypes.c_int
    lib.fs_certify.argtypes = [_i32, _vp, _u64, _i32, _i32, _vp, _vp, _vp, _p_u64, _p_u32, _p_i64, _vp]
    lib.fs_knot_buckets.restype = ctypes.c_int
    lib.fs_knot_buckets.argtypes = [_i32, _vp, _u64, ctypes.c_double, _vp, _vp]
    lib.fs_build_table.restype = ctypes.c_int
    lib.fs_build_table.argtypes = [_i32, _vp, _u64, ctypes.c_double, _u64, _i32, _vp, _vp, _vp, _vp]
    lib.fs_build_rank.restype = ctypes.c_int
    lib.fs_build_rank.argtypes = [_i32, _vp, _u64, ctypes.c_double, _u64, _vp, _vp, _vp]
    lib.fs_build_rank2.restype = ctypes.c_int
    lib.fs_build_rank2.argtypes = [_i32, _vp, _u64, ctypes.c_double, _u64, _vp, _vp, _vp]
    lib.fs_sparse_bytes.restype = ctypes.c_uint64
    lib.fs_sparse_bytes.argtypes = [_u64, _u64, _i32, _u64]
    lib.fs_plan_sparse.restype = ctypes.c_int
    lib.fs_plan_sparse.argtypes = [_i32, _vp, _u64, ctypes.c_double, _u64, _u64, _i32, _vp, _p_i32, _p_u64, _p_u64,
                                   _vp]
    lib.fs_build_sparse.restype = ctypes.c_int
    lib.fs_build_sparse.argtypes = [_i32, _vp, _u64, ctypes.c_double, _u64, _i32, _vp, _vp, _vp]
    lib.fs_sparse_rec_bytes.restype = ctypes.c_uint64
    lib.fs_sparse_rec_bytes.argtypes = [_i32, _u64, _u64, _i32, _u64]
    lib.fs_plan_sparse_rec.restype = ctypes.c_int
    lib.fs_plan_sparse_rec.argtypes = [_i32, _i32, _vp, _u64, ctypes.c_double, _u64, _u64, _i32, _vp, _p_i32,
                                       _p_u64, _p_u64, _p_u32, _vp]
    lib.fs_build_sparse_rec.restype = ctypes.c_int
    lib.fs_build_sparse_rec.argtypes = [_i32, _i32, _vp, _u64, ctypes.c_double, _u64, _i32, _u64, _vp, _vp, _vp]
    lib.fs_zoned_bytes.restype = ctypes.c_uint64
    lib.fs_zoned_bytes.argtypes = [_u64, _i32, _u64]
    lib.fs_plan_zoned.restype = ctypes.c_int
    lib.fs_plan_zoned.argtypes = [_i32, _vp, _u64, ctypes.c_double, _u64, _u64, _vp, _p_i32, _p_u64, _p_u64,
                                  _p_u64, _p_u64, _vp]
    lib.fs_build_zoned.restype = ctypes.c_int
    lib.fs_build_zoned.argtypes = [_i32, _vp, _u64, ctypes.c_double, _u64, _i32, _vp, _vp, _vp]
    lib.fs_plan_zoned_rank.restype = ctypes.c_int
    lib.fs_plan_zoned_rank.argtypes = [_i32, _vp, _u64, ctypes.c_double, _u64, _u64, _vp, _p_i32, _p_u64, _p_u64,
                                       _p_u64, _p_u64, _p_u64, _vp]
    lib.fs_build_zoned_rank.restype = ctypes.c_int
    lib.fs_build_zoned_rank.argtypes = [_i32, _vp, _u64, ctypes.c_double, _u64, _i32, _u64, _vp, _vp, _vp]
    lib.fs_build_knot_bytes.restype = ctypes.c_int
    lib.fs_build_knot_bytes.argtypes = [_i32, _vp, _u64, ctypes.c_double, _vp, _vp]
    lib.fs_build_rank_rows.restype = ctypes.c_int
    lib.fs_build_rank_rows.argtypes = [_i32, _vp, _u64, ctypes.c_double, _u64, _vp, _vp, _vp, _vp]
    lib.fs_count_words_bytes.restype = ctypes.c_uint64
    lib.fs_count_words_bytes.argtypes = [_u64, _i32, _u64]
    lib.fs_plan_count_words.restype = ctypes.c_int
    lib.fs_plan_count_words.argtypes = [_i32, _vp, _u64, ctypes.c_double, _u64, _u64, _i32, _vp, _p_i32, _p_u64,
                                        _p_u64, _p_u64, _vp]
    lib.fs_build_count_words.restype = ctypes.c_int
    lib.fs_build_count_words.argtypes = [_i32, _vp, _u64, ctypes.c_double, _u64, _i32, _i32, _vp, _vp, _vp]
    lib.fs_build_hot_window.restype = ctypes.c_int
    lib.fs_build_hot_window.argtypes = [_i32, _vp, _u64, _u64, _vp, _p_u64, _p_u64, _p_u64, _p_u64, _p_u64, _vp]
    lib.fs_build_fused.restype = ctypes.c_int
    lib.fs_build_fused.argtypes = [_i32, _vp, _u64, _vp, _u64, _vp, _vp]
    lib.fs_build_padded.restype = ctypes.c_int
    lib.fs_build_padded.argtypes = [_i32, _vp, _u64, _i32, _vp, _vp]
    lib.fs_b2_deep_bytes.restype = ctypes.c_uint64
    lib.fs_b2_deep_bytes.argtypes = [_i32, _i32, _p_i32, _p_i32]
    lib.fs_build_b2_deep.restype = ctypes.c_int
    lib.fs_build_b2_deep.argtypes = [_i32, _vp, _i32, _i32, _i32, _vp, _vp]
    lib.fs_build_eytzinger.restype = ctypes.c_int
    lib.fs_build_eytzinger.argtypes = [_i32, _vp, _u64, _i32, _vp, _vp]
    lib.fs_search_ws_words.restype = ctypes.c_size_t
    lib.fs_search_ws_words.argtypes = []
    lib.fs_search_device.restype = ctypes.c_int
    lib.fs_search_device.argtypes = [ctypes.POINTER(FsPlan), _vp, _u64, _vp, _i32, _vp, _vp]
    lib.fs_search_device_at.restype = ctypes.c_int
    lib.fs_search_device_at.argtypes = [ctypes.POINTER(FsPlan), _vp, _u64, _vp, _i32, _vp, _u64, _vp]
    lib.fs_search_host.restype = ctypes.c_int
    lib.fs_search_host.argtypes = [
        ctypes.POINTER(FsPlan), _vp, _u64, _vp, _i32, _vp, _vp, _vp, _u64, _p_i64, _vp, _vp, _i32,
    ]
    lib.fs_search_host_gated.restype = ctypes.c_int
    lib.fs_search_host_gated.argtypes = [
        ctypes.POINTER(FsPlan), _vp, _u64, _vp, _i32, _vp, _vp, _vp, _u64, _p_i64, _vp, _vp, _i32, _vp,
    ]
    lib.fs_gate_create.restype = _vp
    lib.fs_gate_create.argtypes = [_i32]
    lib.fs_gate_abort.restype = None
    lib.fs_gate_abort.argtypes = [_vp]
    lib.fs_gate_destroy.restype = None
    lib.fs_gate_destroy.argtypes = [_vp]
    lib.fs_countdir_bytes.restype = _u64
    lib.fs_countdir_bytes.argtypes = [_i32, _u64]
    lib.fs_build_countdir.restype = ctypes.c_int
    lib.fs_build_countdir.argtypes = [_i32, _vp, _u64, ctypes.c_double, _u64, _i32, _vp, _vp, _vp]
    lib.fs_crc32_ws_bytes.restype = ctypes.c_size_t
    lib.fs_crc32_ws_bytes.argtypes = [_u64]
    lib.fs_crc32.restype = ctypes.c_int
    lib.fs_crc32.argtypes = [_vp, _u64, _vp, _p_u32, _vp]
    lib.fs_plan_placement.restype = ctypes.c_int
    lib.fs_plan_placement.argtypes = [ctypes.POINTER(FsPlan), _p_i32, _p_u64]
    lib.fs_search_launches.restype = ctypes.c_int
    lib.fs_search_launches.argtypes = [ctypes.POINTER(FsPlan), _u64]
    lib.fs_search_host_launches.restype = ctypes.c_int64
    lib.fs_search_host_launches.argtypes = [ctypes.POINTER(FsPlan), _vp, _u64, _vp, _i32, _u64, _i32]


def load(path: str | os.PathLike | None = None):
    """Load (once) and return the native library; raise if it is absent."""
    global _lib
    with _lock:
        if _lib is None:
            p = Path(path) if path else LIB_PATH
            if not p.exists():
                raise ImportError(
                    f"{p} is missing: the CUDA library is not built. "
                    "Run `python -c 'import __graft_entry__ as g; g.build()'` (there is no CPU fallback)."
                )
            lib = ctypes.CDLL(str(p))
            _declare(lib)
            _lib = lib
        return _lib


def last_error() -> str:
    msg = load().fs_last_error()
    return msg.decode() if msg else ""


def check(rc: int, pos: int | None = None, what: str = ""):
    """Map an fs_status code onto the reference exception classes."""
    if rc == FS_OK:
        return
    msg = last_error()
    if rc == FS_NOT_DISTINGUISHABLE:
        raise NotDistinguishable(int(pos))
    if rc == FS_OVERFLOW:
        raise Overflow(msg or "bucket index would overflow")
    if rc == FS_OUT_OF_DOMAIN:
        raise OutOfDomain(position=None if pos is None else int(pos))
    if rc in (FS_INVALID_ARG, FS_INCONSISTENT, FS_TOO_LARGE):
        raise ValueError(msg or what)
    if rc == FS_ABORTED:
        raise SpanAborted(msg or what)
    raise DeviceError(f"{what}: {msg}" if what else msg)
