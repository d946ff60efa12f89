"""Bit-exact FBSIDX1 index files, loaded straight into device memory.

Same file format, return values and exceptions as the reference
(``fastsearch/bench/persist.py:1-112``; the index-file half of the
reference's bench package, the only part on the hot path's data format): 48-byte little-endian header
(magic ``FBSIDX1\\0``, version 1, precision, qbits, gap, N, R, raw binary64
bits of H and X0), the u32 K payload, and the zlib CRC-32 of the payload.
Files written here are byte-identical to the reference's and vice versa.

B200 path: ``load_index`` copies the K payload host->device once and checks
its CRC-32 on the GPU (``fs_crc32``), so the table never takes a second
host pass; ``save_index`` checksums the resident table on the device and
copies it out once.
"""

from __future__ import annotations

import ctypes
import struct
from pathlib import Path

import numpy as np

from . import _device, _lib
from .direct import DirectIndex
from .errors import BadMagic, ChecksumMismatch, TruncatedFile, VersionMismatch

MAGIC = b"FBSIDX1\0"
VERSION = 1

_HEADER = struct.Struct("<8sHBBB3sQQQQ")
_PRECISION_CODE = {"single": 0, "double": 1}
_PRECISION_NAME = {0: "single", 1: "double"}


def device_crc32(t) -> int:
    """zlib CRC-32 of a device tensor's bytes, computed on the GPU."""
    nbytes = t.numel() * t.element_size()
    ws = _device.empty(max(1, _lib.load().fs_crc32_ws_bytes(nbytes) // 4), np.uint32)
    out = ctypes.c_uint32(0)
    rc = _lib.load().fs_crc32(t.data_ptr(), nbytes, ws.data_ptr(), ctypes.byref(out), _device.stream_ptr())
    _lib.check(rc, what="fs_crc32")
    return int(out.value)


def pack_header(idx: DirectIndex) -> bytes:
    """persist.py:48-61."""
    h_bits = struct.unpack("<Q", struct.pack("<d", float(idx.h)))[0]
    x0_bits = struct.unpack("<Q", struct.pack("<d", float(idx.x0)))[0]
    return _HEADER.pack(MAGIC, VERSION, _PRECISION_CODE[idx.precision], idx.qbits, idx.q, b"\0\0\0", idx.n, idx.r,
                        h_bits, x0_bits)


def parse_header(data: bytes, path="<bytes>") -> dict:
    """Header checks in the reference's order (persist.py:71-88): truncation,
    magic, header size, version, field ranges, payload + checksum present."""
    if len(data) < 8:
        raise TruncatedFile(f"{path}: shorter than the magic header")
    if data[:8] != MAGIC:
        raise BadMagic(f"{path}: not an index file")
    if len(data) < _HEADER.size:
        raise TruncatedFile(f"{path}: incomplete header")
    (_, version, prec_code, qbits, gap, _, n, r, h_bits, x0_bits) = _HEADER.unpack(data[: _HEADER.size])
    if version != VERSION:
        raise VersionMismatch(f"{path}: format version {version}, expected {VERSION}")
    if prec_code not in _PRECISION_NAME or qbits not in (32, 64) or gap < 1:
        raise VersionMismatch(f"{path}: unrecognized header fields")
    end = _HEADER.size + (r + 1) * 4
    if len(data) < end + 4:
        raise TruncatedFile(f"{path}: payload or checksum missing")
    return {"precision": _PRECISION_NAME[prec_code], "qbits": int(qbits), "q": int(gap), "n": int(n), "r": int(r),
            "h_bits": h_bits, "x0_bits": x0_bits, "end": end}


def save_index(idx: DirectIndex, path) -> int:
    """Write the index to ``path``; returns the byte count (persist.py:46-66)."""
    crc = device_crc32(idx.k_dev)
    payload = idx.k.astype("<u4", copy=False).tobytes()
    data = pack_header(idx) + payload + struct.pack("<I", crc)
    Path(path).write_bytes(data)
    return len(data)


def load_index(path) -> DirectIndex:
    """Read an index back with K resident on the device (persist.py:69-112);
    fused records are not stored and come back empty."""
    data = Path(path).read_bytes()
    hd = parse_header(data, path)
    end = hd["end"]
    payload = np.frombuffer(data, dtype="<u4", count=hd["r"] + 1, offset=_HEADER.size)
    (crc_stored,) = struct.unpack("<I", data[end:end + 4])
    k_dev = _device.upload(payload.astype(np.uint32, copy=False))
    if device_crc32(k_dev) != crc_stored:
        raise ChecksumMismatch(f"{path}: K payload corrupted")
    dtype = np.float32 if hd["precision"] == "single" else np.float64
    (h64,) = struct.unpack("<d", struct.pack("<Q", hd["h_bits"]))
    (x064,) = struct.unpack("<d", struct.pack("<Q", hd["x0_bits"]))
    left_pad = np.full(hd["q"] - 1, dtype(x064), dtype=dtype)
    left_pad.setflags(write=False)
    return DirectIndex(x0=dtype(x064), h=dtype(h64), r=hd["r"], q=hd["q"], k_dev=k_dev, qbits=hd["qbits"],
                       n=hd["n"], precision=hd["precision"], left_pad=left_pad)


#: the search kernel that serves a loaded index of each gap (direct.py:272-300)
LOADED_ALGORITHM = {1: "direct", 2: "direct-gap2"}


def prepare_loaded(idx: DirectIndex, p, algorithm: str | None = None):
    """A PreparedKernel over a loaded index and its partition (the search
    kernels and shared-memory layouts of batch.prepare, without rebuilding
    the table).  The kernel
    follows the index's gap q: "direct" for q = 1, "direct-gap2" for q = 2,
    "direct-generic" otherwise (the reference's direct_search_generic,
    direct.py:294-300); an explicit ``algorithm`` that does not match q
    raises ValueError, since a gap-1 probe over a gap-q table (or the
    reverse) returns wrong answers."""
    from .batch import PreparedKernel, _make_callables, _plan_for, set_direct_layouts

    want = LOADED_ALGORITHM.get(idx.q, "direct-generic")
    if algorithm is None:
        algorithm = want
    if algorithm not in ("direct", "direct-gap2", "direct-generic"):
        raise ValueError("loaded indices serve the direct, direct-gap2 and direct-generic kernels")
    if algorithm != want:
        raise ValueError(f"an index of gap q={idx.q} is searched by {want!r}, not {algorithm!r}")
    if algorithm == "direct-generic" and idx.q <= 15:
        from .batch import prepare_direct_gap

        return prepare_direct_gap(p, idx.q, idx.qbits, idx=idx)  # over its count directory
    plan, keep = _plan_for(algorithm, idx, p)
    if algorithm == "direct":
        set_direct_layouts(plan, p, idx, keep)  # the same layouts prepare() builds over a fresh table
    scalar, lanes = _make_callables(plan, p)
    return PreparedKernel(algorithm, p, idx, scalar, lanes, plan=plan, buffers=tuple(keep))
