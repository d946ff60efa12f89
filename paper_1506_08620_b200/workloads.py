"""Seeded synthetic workloads for the five BASELINE configs.

No public benchmark or dataset is involved; these recipes
 produce the knot arrays X on the host with numpy's
PCG64 stream (bit-reproducible per seed) and the query streams either on the
host (numpy, exact ``gen_queries`` recipe, for parity tests) or directly on
the device (torch Philox, same distributions, for full-size runs where a
2^30-query host draw would dominate the run).

  cfg1  f32, N+1 = 1,001 sorted U[0,1), whole-array redraw while min gap < 1e-6;
        M = 1e6 uniform queries                                (CPU-runnable)
  cfg2  f64, N+1 = 10,001 sorted U[0,100), redraw while min gap < 1e-9;
        M = 1e8 uniform, 1% overwritten with exact knots X_i, i < N
  cfg3  f32, N+1 = 4,097, gaps 0.5 + U[0,1) summed in f64 from 0;
        M = 2^30 uniform                                      (streaming)
  cfg4  f32, N+1 = 65,537, geometric gaps 1e-4 * 1.0001^i summed in f64;
        M = 2^28: 50% uniform on [X0, XN), 50% on the densest 10% [X0, X_6554)
  cfg5  f64, N+1 in {33, 1025, 32769, 1048577} sorted U[0,1), offenders of
        min gap 1e-7 deleted and redrawn; M = 2^28 uniform.  The unfiltered
        1,048,577 draw is the fallback instance (Overflow -> bitset2).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .partition import SortedPartition, gen_uniform_gap_partition, validate_partition


@dataclass(frozen=True)
class Config:
    name: str
    precision: str
    n1: int
    m: int
    description: str


CONFIGS = {
    "cfg1": Config("cfg1", "single", 1001, 1_000_000, "f32 N+1=1001 sorted U[0,1) min gap 1e-6; M=1e6"),
    "cfg2": Config("cfg2", "double", 10_001, 100_000_000, "f64 N+1=10001 sorted U[0,100) min gap 1e-9; M=1e8 (1% exact knots)"),
    "cfg3": Config("cfg3", "single", 4097, 1 << 30, "f32 N+1=4097 gaps 0.5+U[0,1); M=2^30 uniform"),
    "cfg4": Config("cfg4", "single", 65_537, 1 << 28, "f32 N+1=65537 geometric gaps 1e-4*1.0001^i; M=2^28 50% clustered"),
    "cfg5": Config("cfg5", "double", 1_048_577, 1 << 28, "f64 N+1 in {33,1025,32769,1048577} sorted U[0,1) min gap 1e-7; M=2^28"),
}

CFG5_SIZES = (33, 1025, 32_769, 1_048_577)


def _sorted_redraw(rng, n1, lo, hi, min_gap, dtype):
    """Whole-array redraw until the cast array's min gap (in f64) >= min_gap."""
    while True:
        x = np.sort(rng.uniform(lo, hi, n1)).astype(dtype)
        if np.diff(x.astype(np.float64)).min() >= min_gap:
            return x


def _sorted_repair(rng, n1, min_gap):
    """Sorted U[0,1) with offenders of ``min_gap`` deleted and redrawn."""
    x = np.sort(rng.uniform(0.0, 1.0, n1))
    while True:
        bad = np.diff(x) < min_gap
        if not bad.any():
            return x
        keep = np.concatenate([[True], ~bad])
        x = np.sort(np.concatenate([x[keep], rng.uniform(0.0, 1.0, int(bad.sum()))]))


def knots(name: str, seed: int = 0, n1: int | None = None, filtered: bool = True) -> SortedPartition:
    """The knot array X of config ``name`` (validated SortedPartition)."""
    if name == "cfg1":
        rng = np.random.default_rng(seed)
        return validate_partition(_sorted_redraw(rng, 1001, 0.0, 1.0, 1e-6, np.float32))
    if name == "cfg2":
        rng = np.random.default_rng(seed)
        return validate_partition(_sorted_redraw(rng, 10_001, 0.0, 100.0, 1e-9, np.float64))
    if name == "cfg3":
        return gen_uniform_gap_partition(4097, 0.5, 1.5, seed, "single")
    if name == "cfg4":
        gaps = 1e-4 * 1.0001 ** np.arange(65_536, dtype=np.float64)
        x = np.concatenate([[0.0], np.cumsum(gaps)]).astype(np.float32)
        return validate_partition(x)
    if name == "cfg5":
        size = n1 if n1 is not None else CFG5_SIZES[-1]
        rng = np.random.default_rng(seed)
        if filtered:
            x = _sorted_repair(rng, size, 1e-7)
        else:
            x = np.unique(rng.uniform(0.0, 1.0, size))
            while len(x) < size:  # exact duplicates are astronomically rare
                x = np.unique(np.concatenate([x, rng.uniform(0.0, 1.0, size - len(x))]))
        return validate_partition(x)
    raise ValueError(f"unknown config {name!r}")


def cfg4_dense_top(p: SortedPartition) -> float:
    """Upper end of cfg4's clustered half: X_6554 (the densest 10% of knots)."""
    return float(p.values[min(6554, len(p.values) - 1)])


def queries_host(name: str, p: SortedPartition, m: int, seed: int = 1) -> np.ndarray:
    """Host query stream of config ``name`` (numpy PCG64, gen_queries recipe:
    draw f64 on [X0, XN), cast, pull values rounded onto XN back inside)."""
    rng = np.random.default_rng(seed)
    dtype = p.values.dtype
    x0, xn = float(p.values[0]), float(p.values[-1])
    if name == "cfg4":
        half = m // 2
        a = rng.uniform(x0, xn, size=m - half)
        b = rng.uniform(x0, cfg4_dense_top(p), size=half)
        z = np.concatenate([a, b])[rng.permutation(m)].astype(dtype)
    else:
        z = rng.uniform(x0, xn, size=m).astype(dtype)
    top = dtype.type(p.values[-1])
    z[z >= top] = np.nextafter(top, dtype.type(-np.inf))
    if name == "cfg2" and m >= 100:
        k = m // 100
        pos = rng.choice(m, size=k, replace=False)
        z[pos] = p.values[rng.integers(0, p.n_intervals, size=k)]
    return z


def queries_device(name: str, p: SortedPartition, m: int, seed: int = 1, device=None, chunk: int = 1 << 26):
    """Device query stream with the same distributions (torch Philox)."""
    import torch

    dev = device if device is not None else torch.device("cuda", torch.cuda.current_device())
    tdt = torch.float32 if p.precision == "single" else torch.float64
    g = torch.Generator(device=dev)
    g.manual_seed(seed)
    z = torch.empty(m, dtype=tdt, device=dev)
    x0, xn = float(p.values[0]), float(p.values[-1])
    hi_dense = cfg4_dense_top(p) if name == "cfg4" else xn
    for a in range(0, m, chunk):
        b = min(m, a + chunk)
        u = torch.rand(b - a, dtype=torch.float64, device=dev, generator=g)
        if name == "cfg4":
            coin = torch.rand(b - a, dtype=torch.float64, device=dev, generator=g) < 0.5
            hi = torch.where(coin, torch.full_like(u, hi_dense), torch.full_like(u, xn))
            v = x0 + u * (hi - x0)
        else:
            v = x0 + u * (xn - x0)
        z[a:b] = v.to(tdt)
    top = torch.tensor(p.values[-1], dtype=tdt, device=dev)
    below = torch.nextafter(top, torch.tensor(float("-inf"), dtype=tdt, device=dev))
    z = torch.where(z >= top, below, z)
    if name == "cfg2" and m >= 100:
        k = m // 100
        pos = torch.randperm(m, device=dev, generator=g)[:k]
        xi = p.device_values()[torch.randint(0, p.n_intervals, (k,), device=dev, generator=g)]
        z[pos] = xi
    return z
