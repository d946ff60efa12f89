"""Query sharding across GPUs: one process per GPU, torch.distributed plumbing.

The reference parallelises with contiguous query spans over a thread pool
(batch.py:385-396, 428-440); here the spans go to ranks.  Queries are
independent and outputs disjoint (batch.py:16-19), so the data path has no
collective: each rank builds X/J locally (the build is deterministic, so
every replica is bit-identical) and searches its own span.  The single
per-batch collective is a MIN all-reduce of the first out-of-domain position
so every rank raises the same OutOfDomain(position) the unsharded call would.
"""

from __future__ import annotations

import torch
import torch.distributed as dist

from .batch import first_bad_of, new_status
from .errors import OutOfDomain

NO_BAD = (1 << 63) - 1  # int64 sentinel ("no out-of-domain query")


def shard_span(m: int, rank: int, world: int, granularity: int = 4) -> tuple[int, int]:
    """Contiguous [start, stop) of ``m`` queries for ``rank`` of ``world``,
    split at ``granularity`` bounds (16-B aligned shards for 4-byte queries),
    the last rank taking the remainder -- batch._spans (batch.py:385-396)
    with ranks for threads."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("need 0 <= rank < world")
    units = m // granularity
    base, extra = divmod(units, world)
    start = (rank * base + min(rank, extra)) * granularity
    stop = start + (base + (rank < extra)) * granularity
    if rank == world - 1:
        stop = m
    return start, stop


def global_first_bad(local_first_bad: int | None, offset: int, group=None, device=None) -> int | None:
    """MIN all-reduce of the first out-of-domain position over ranks.

    ``local_first_bad`` is the rank-local position (None when clean);
    returns the global position, or None when every rank was clean.
    """
    val = NO_BAD if local_first_bad is None else offset + int(local_first_bad)
    if dist.is_available() and dist.is_initialized():
        t = torch.tensor([val], dtype=torch.int64, device=device)
        dist.all_reduce(t, op=dist.ReduceOp.MIN, group=group)
        val = int(t.item())
    return None if val == NO_BAD else val


def sharded_batch_search(prepared, z_local, out_local, offset: int, group=None, status=None) -> int:
    """Search this rank's span on its GPU, then agree on OutOfDomain.

    ``z_local``/``out_local`` are CUDA tensors holding queries
    [offset, offset + len) of the global batch; ``status`` an optional
    reusable workspace (new_status()).  One search kernel that reports
    global positions (fs_search_device_at: status word 3 = first bad
    position XOR 2^63, a signed-int64 key with "clean" = INT64_MAX), one MIN
    all-reduce of that word in place, and a single host read decides:
    OutOfDomain with the global first position on every rank if any rank
    saw a bad query.  Returns the span's length.
    """
    fb = status if status is not None else new_status(z_local.device)
    prepared.launch(z_local, out_local, fb, base=int(offset))
    key = fb[3:4].view(torch.int64)
    if dist.is_available() and dist.is_initialized():
        dist.all_reduce(key, op=dist.ReduceOp.MIN, group=group)
    k = int(key.item())
    if k != NO_BAD:
        raise OutOfDomain(position=k + (1 << 63))
    return z_local.numel()
