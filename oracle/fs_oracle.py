"""CPU oracle: a numpy restatement of the reference's hot path.

TEST INFRASTRUCTURE -- NOT PRODUCT CODE.  Only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py``'s cpu_baseline / ``--impl
reference`` legs may import this module, and only as the checker or as the
timed CPU baseline; the product package (paper_1506_08620_b200) never
imports it and has no CPU fallback.

Every function restates one function of the reference ``fastsearch`` 0.1.0
(/root/reference/pkg/src/fastsearch, pure Python + numpy; numpy is the only
third-party arithmetic, its IEEE-754 RN elementwise ops and PCG64 stream).
The restatement works on plain numpy arrays so it shares no code with the
product.  Parity is PINNED: tests/golden/*.npz were produced by running the
reference itself in the build container (tests/golden/make_golden.py) and
tests/test_oracle_golden.py checks this module against every vector there
(worked example, growth seeds, error cases, K tables/hashes, exhaustive
boundary probes for sizes 2..64, 1e5-query random sweeps, the five configs).
"""

from __future__ import annotations

import os
from concurrent.futures import ThreadPoolExecutor

import numpy as np

# ---------------------------------------------------------------------------
# errors (return codes instead of exception classes, so the oracle does not
# depend on the product's exception module)
# ---------------------------------------------------------------------------


class OracleError(ValueError):
    def __init__(self, kind: str, position=None):
        self.kind = kind  # "not_distinguishable" | "overflow" | "out_of_domain" | "inconsistent"
        self.position = position
        super().__init__(f"{kind} (position={position})")


# ---------------------------------------------------------------------------
# partition.py
# ---------------------------------------------------------------------------


def gen_uniform_gap(size: int, gap_lo: float, gap_hi: float, seed: int, dtype) -> np.ndarray:
    """partition.py:126-147: X_0 = 0, f64 gaps U[gap_lo, gap_hi], f64 cumsum, cast."""
    rng = np.random.default_rng(seed)
    gaps = rng.uniform(gap_lo, gap_hi, size=size - 1)
    return np.concatenate([[0.0], np.cumsum(gaps)]).astype(dtype)


def random_queries(xs: np.ndarray, count: int, seed: int) -> np.ndarray:
    """pkg/tests/helpers.py:42-49 (== partition.gen_queries, partition.py:150-160)."""
    rng = np.random.default_rng(seed)
    z = rng.uniform(float(xs[0]), float(xs[-1]), size=count).astype(xs.dtype)
    top = xs[-1]
    z[z >= top] = np.nextafter(top, xs.dtype.type(-np.inf))
    return z


def boundary_probes(xs: np.ndarray) -> np.ndarray:
    """pkg/tests/helpers.py:31-39: knots, nextafter(knot, +-inf), midpoints, in domain."""
    up = np.nextafter(xs, xs.dtype.type(np.inf))
    down = np.nextafter(xs, xs.dtype.type(-np.inf))
    mids = xs[:-1] + (xs[1:] - xs[:-1]) / xs.dtype.type(2)
    z = np.concatenate([xs, up, down, mids])
    z = z[(z >= xs[0]) & (z < xs[-1])]
    return np.unique(z)


def bucket_edge_probes(xs: np.ndarray, h, r: int, count: int, seed: int) -> np.ndarray:
    """z = cast(X0 + j/h) for random buckets j and
    +-1..3 ulp neighbours, kept in domain."""
    rng = np.random.default_rng(seed)
    t = xs.dtype.type
    j = rng.integers(0, r + 1, size=count).astype(np.float64)
    base = (float(xs[0]) + j / float(h)).astype(xs.dtype)
    out = [base]
    lo, hi = base.copy(), base.copy()
    for _ in range(3):
        lo = np.nextafter(lo, t(-np.inf))
        hi = np.nextafter(hi, t(np.inf))
        out += [lo, hi]
    z = np.concatenate(out)
    return z[(z >= xs[0]) & (z < xs[-1])]


def first_bad(xs: np.ndarray, z: np.ndarray):
    """batch.py:411-413: first j with !(X0 <= z < XN) (NaN included), or None."""
    bad = ~((z >= xs[0]) & (z < xs[-1]))
    return int(np.argmax(bad)) if bad.any() else None


def linear_scan(xs: np.ndarray, z) -> int:
    """partition.py:180-192: walk the knots; max{i : X_i <= z}."""
    if not (xs[0] <= z < xs[-1]):
        raise OracleError("out_of_domain")
    i = 0
    last = len(xs) - 2
    while i < last and xs[i + 1] <= z:
        i += 1
    return i


def linear_scan_batch(xs: np.ndarray, z: np.ndarray) -> np.ndarray:
    """partition.py:195-216: sort the queries, advance one knot cursor."""
    z = np.asarray(z)
    fb = first_bad(xs, z)
    if fb is not None:
        raise OracleError("out_of_domain", fb)
    order = np.argsort(z, kind="stable")
    zs = z[order].tolist()
    xl = xs.tolist()
    out = np.empty(len(zs), dtype=np.int64)
    i = 0
    last = len(xl) - 2
    for pos, q in zip(order.tolist(), zs):
        while i < last and xl[i + 1] <= q:
            i += 1
        out[pos] = i
    return out


def rank_oracle(xs: np.ndarray, z: np.ndarray) -> np.ndarray:
    """max{i : X_i <= z} for large batches: count of knots <= z, minus one
    (the defining property of partition.py:180-192, evaluated by numpy's
    comparison-only searchsorted).  Pinned to linear_scan_batch in tests."""
    fb = first_bad(xs, z)
    if fb is not None:
        raise OracleError("out_of_domain", fb)
    return np.searchsorted(xs, z, side="right").astype(np.int64) - 1


def pad_right_pow2(xs: np.ndarray):
    """partition.py:163-171 -> (padded, p, probe)."""
    n = len(xs) - 1
    bits = n.bit_length()
    padded = np.full(1 << bits, xs[-1], dtype=xs.dtype)
    padded[: n + 1] = xs
    return padded, bits, 1 << (bits - 1)


# ---------------------------------------------------------------------------
# direct.py
# ---------------------------------------------------------------------------


def compute_h_r(xs: np.ndarray, qbits: int = 32, q: int = 1):
    """direct.py:135-191, op for op in the array's precision.

    Returns (h, r, increments, h_start) or raises OracleError.
    """
    if qbits not in (32, 64) or q < 1:
        raise ValueError("qbits must be 32 or 64 and q >= 1")
    n = len(xs) - 1
    scalar = xs.dtype.type
    offsets = xs - xs[0]
    collide = offsets[q:] == offsets[:-q]
    if collide.any():
        raise OracleError("not_distinguishable", int(np.argmax(collide)) + q)
    basis = min(q, n)
    with np.errstate(over="ignore"):
        h = scalar(1.0) / (offsets[basis:] - offsets[:-basis]).min()
        h_start = h
        limit = scalar(2.0 ** qbits)
        span = offsets[-1]
        if not h * span < limit:
            raise OracleError("overflow", 0)
        growth = np.nextafter(h, scalar(np.inf)) - h
        increments = 0
        while True:
            floors = np.floor(h * offsets)
            if (floors[q:] > floors[:-q]).all():
                break
            h = h + growth
            increments += 1
            if not h * span < limit:
                raise OracleError("overflow", increments)
            growth = growth + growth
    return h, int(floors[-1]), increments, h_start


def knot_buckets(xs: np.ndarray, h) -> np.ndarray:
    """direct.py:194-197."""
    return np.floor(h * (xs - xs[0])).astype(np.int64)


def build_table(xs: np.ndarray, h, r: int, q: int = 1) -> np.ndarray:
    """direct.py:200-229: K as np.repeat of knot indices over bucket runs."""
    n = len(xs) - 1
    f = knot_buckets(xs, h)
    if f[-1] != r:
        raise OracleError("inconsistent")
    if q == 1:
        counts = np.concatenate([[1], np.diff(f)])
    else:
        counts = np.concatenate([np.diff(f), [1]])
    k = np.repeat(np.arange(n + 1, dtype=np.uint32), counts)
    assert len(k) == r + 1 and k[-1] == n
    return k


FUSED_DTYPES = {
    np.dtype(np.float32): np.dtype([("idx", "<u4"), ("val", "<f4")]),
    np.dtype(np.float64): np.dtype([("idx", "<u4"), ("pad", "<u4"), ("val", "<f8")]),
}


def fused_records(xs: np.ndarray, k: np.ndarray) -> np.ndarray:
    """direct.py:255-263."""
    rec = np.zeros(len(k), dtype=FUSED_DTYPES[xs.dtype])
    rec["idx"] = k
    rec["val"] = xs[k]
    return rec


# ---------------------------------------------------------------------------
# batch.py lane kernels (vectorised, bit-identical to the scalar kernels)
# ---------------------------------------------------------------------------


def direct_lanes(xs, h, k, z):
    """batch.py:315-317."""
    t = k[(h * (z - xs[0])).astype(np.int64)].astype(np.int64)
    return t - (z < xs[t])


def gap2_lanes(xs, h, k, z):
    """batch.py:321-345 (xpad = [X0] + X)."""
    xp = np.concatenate([xs[:1], xs])
    t = k[(h * (z - xs[0])).astype(np.int64)].astype(np.int64)
    return t - (z < xp[t + 1]) - (z < xp[t])


def generic_lanes(xs, h, k, q, z):
    """direct.py:294-300 vectorised."""
    t = k[(h * (z - xs[0])).astype(np.int64)].astype(np.int64)
    hits = np.zeros_like(t)
    for m in range(q):
        hits += z < xs[np.maximum(t - m, 0)]
    return t - hits


def cache_lanes(xs, h, rec, z):
    """batch.py:368-371."""
    j = (h * (z - xs[0])).astype(np.int64)
    r = rec[j]
    return r["idx"].astype(np.int64) - (z < r["val"])


def bitset2_lanes(padded, probe, z):
    """batch.py:193-200."""
    i = np.zeros(len(z), dtype=np.int64)
    k = probe
    while k:
        r = i | k
        i = np.where(z >= padded[r], r, i)
        k >>= 1
    return i


def bitset1_lanes(xs, probe, z):
    """batch.py:176-185."""
    n = len(xs) - 1
    i = np.zeros(len(z), dtype=np.int64)
    k = probe
    while k:
        r = i | k
        take = (r < n) & (z >= xs[np.minimum(r, n)])
        i = np.where(take, r, i)
        k >>= 1
    return i


def bitset3_lanes(xs, probe, z):
    """batch.py:208-216."""
    n = len(xs) - 1
    i = np.zeros(len(z), dtype=np.int64)
    k = probe
    while k:
        r = i | k
        i = np.where(z >= xs[np.minimum(r, n)], r, i)
        k >>= 1
    return i


def offset_lanes(xs, z):
    """batch.py:224-234 with binsearch.offset_constants (binsearch.py:34-38)."""
    n = len(xs) - 1
    f0 = (n + 1) >> 1
    s = n + 1 - f0
    jn = (n + 1).bit_length() - 1
    i = np.where(z >= xs[f0], f0, 0).astype(np.int64)
    for _ in range(jn):
        half = s >> 1
        f = i + half
        i = np.where(z >= xs[f], f, i)
        s -= half
    return i


def eytzinger_layout(xs: np.ndarray):
    """eytzinger.py:45-63 -> (tree, L)."""
    n = len(xs) - 1
    depth = (n + 1).bit_length()
    size = (1 << depth) - 1
    padded = np.full(size, xs[-1], dtype=xs.dtype)
    padded[: n + 1] = xs
    slots = np.arange(1, size + 1, dtype=np.int64)
    levels = np.frexp(slots.astype(np.float64))[1] - 1
    stride = np.int64(1) << (depth - levels)
    rank = (slots - (np.int64(1) << levels)) * stride + (stride >> 1) - 1
    return padded[rank], depth


def eytzinger_lanes(tree, depth, z):
    """batch.py:242-246."""
    k = np.ones(len(z), dtype=np.int64)
    for _ in range(depth):
        k = 2 * k + (z >= tree[k - 1])
    return k - (1 << depth) - 1


def classic_scalar(xs, z) -> int:
    """binsearch.py:48-57."""
    low, high = 0, len(xs) - 1
    while high - low > 1:
        mid = (low + high) >> 1
        if z < xs[mid]:
            high = mid
        else:
            low = mid
    return low


# ---------------------------------------------------------------------------
# The reference's batch driver (batch.py:385-441) -- the CPU baseline port
# ---------------------------------------------------------------------------


class PreparedPort:
    """prepare() of batch.py:156-255 restated for the lane kernels the bench
    compares (direct, direct-cache, direct-gap2, bitset2)."""

    def __init__(self, algorithm: str, xs: np.ndarray, qbits: int = 32):
        self.algorithm = algorithm
        self.xs = xs
        if algorithm in ("direct", "direct-cache", "direct-gap2"):
            q = 2 if algorithm == "direct-gap2" else 1
            h, r, _, _ = compute_h_r(xs, qbits, q)
            k = build_table(xs, h, r, q)
            self.h, self.r, self.k = h, r, k
            if algorithm == "direct":
                self.lanes = lambda z: direct_lanes(xs, h, k, z)
            elif algorithm == "direct-gap2":
                self.lanes = lambda z: gap2_lanes(xs, h, k, z)
            else:
                rec = fused_records(xs, k)
                self.lanes = lambda z: cache_lanes(xs, h, rec, z)
        elif algorithm == "bitset2":
            padded, _, probe = pad_right_pow2(xs)
            self.lanes = lambda z: bitset2_lanes(padded, probe, z)
        else:
            raise ValueError(f"port covers direct/direct-gap2/direct-cache/bitset2, not {algorithm!r}")


def spans(total: int, parts: int, granularity: int):
    """batch.py:385-396."""
    units = total // granularity
    parts = min(parts, units) or 1
    base, extra = divmod(units, parts)
    start = 0
    for w in range(parts):
        stop = start + (base + (w < extra)) * granularity
        yield start, stop
        start = stop
    if start < total:
        yield start, total


def batch_search_port(prep: PreparedPort, z: np.ndarray, out: np.ndarray, d: int = 65536,
                      threads: int | None = None) -> int:
    """batch.py:399-441 with the lane path on the ⌊M/d⌋·d prefix; the M mod d
    tail also goes through the lanes closure here (the reference's scalar
    closures are bit-identical to the lanes, batch.py:5-10)."""
    m = len(z)
    fb = first_bad(prep.xs, z)
    if fb is not None:
        raise OracleError("out_of_domain", fb)
    nthreads = threads or os.cpu_count() or 1
    lane_stop = (m // d) * d

    def run(a, b):
        if a < b:
            out[a:b] = prep.lanes(z[a:b])

    if nthreads == 1:
        run(0, m)
        return m
    sp = list(spans(lane_stop, nthreads, d)) if lane_stop else []
    if lane_stop < m:
        sp.append((lane_stop, m))
    with ThreadPoolExecutor(max_workers=nthreads) as pool:
        for fut in [pool.submit(run, a, b) for a, b in sp]:
            fut.result()
    return m
