"""Device plumbing: torch supplies device memory and the current stream.

Nothing here computes anything on the search path; it allocates, uploads
and hands raw pointers to the C-ABI (``_lib``).
"""

from __future__ import annotations

import threading

import numpy as np
import torch

from . import _lib

_TORCH = {
    np.dtype(np.float32): torch.float32,
    np.dtype(np.float64): torch.float64,
    np.dtype(np.int32): torch.int32,
    np.dtype(np.int64): torch.int64,
    np.dtype(np.uint32): torch.uint32,
    np.dtype(np.uint64): torch.uint64,
    np.dtype(np.uint8): torch.uint8,
}


def require_cuda() -> torch.device:
    """Current CUDA device; raises when there is none (no CPU fallback)."""
    if not torch.cuda.is_available():
        raise RuntimeError(
            "paper_1506_08620_b200 runs on a CUDA device (sm_100a); none is available "
            "and there is deliberately no CPU fallback"
        )
    _lib.load()
    return torch.device("cuda", torch.cuda.current_device())


_raw_stream = getattr(torch._C, "_cuda_getCurrentRawStream", None)


def stream_ptr(stream: torch.cuda.Stream | None = None, device_index: int | None = None) -> int:
    """cudaStream_t of ``stream`` or of the current stream (raw pointer; the
    fast path skips building a torch Stream object on every launch)."""
    if stream is not None:
        return int(stream.cuda_stream)
    if _raw_stream is not None:
        return int(_raw_stream(torch.cuda.current_device() if device_index is None else device_index))
    return int(torch.cuda.current_stream().cuda_stream)


def torch_dtype(dtype) -> torch.dtype:
    return _TORCH[np.dtype(dtype)]


def empty(n: int, dtype, device=None) -> torch.Tensor:
    dev = device if device is not None else require_cuda()
    return torch.empty(int(n), dtype=torch_dtype(dtype), device=dev)


def upload(arr: np.ndarray, device=None) -> torch.Tensor:
    dev = device if device is not None else require_cuda()
    a = np.ascontiguousarray(arr)
    t = torch.empty(a.shape, dtype=torch_dtype(a.dtype), device=dev)
    t.copy_(torch.from_numpy(a.copy() if not a.flags.writeable else a))
    return t


def download(t: torch.Tensor) -> np.ndarray:
    return t.detach().cpu().numpy()


class Workspace:
    """Small status block of the build entry points, one per (thread,
    device): concurrent builds on a shared stream must not share it."""

    _tls = threading.local()

    @classmethod
    def get(cls) -> torch.Tensor:
        dev = require_cuda()
        cache = getattr(cls._tls, "ws", None)
        if cache is None:
            cache = cls._tls.ws = {}
        ws = cache.get(dev.index)
        if ws is None:
            nbytes = int(_lib.load().fs_workspace_bytes())
            ws = torch.empty(nbytes, dtype=torch.uint8, device=dev)
            cache[dev.index] = ws
        return ws
