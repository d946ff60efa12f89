"""Loader for the golden fixtures (tests/golden/, produced by running the
reference itself: tests/golden/make_golden.py).  Rebuilds every partition
and query set from its recipe and checks it against the recorded SHA-256,
so a drifting recipe fails loudly instead of silently testing other data."""

from __future__ import annotations

import functools
import hashlib
import json
import re
from pathlib import Path

import numpy as np

from oracle import fs_oracle as orc

GOLDEN = Path(__file__).resolve().parent / "golden"
SEED = 20240708


def sha(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


@functools.lru_cache(maxsize=1)
def meta() -> dict:
    return json.loads((GOLDEN / "golden.json").read_text())


@functools.lru_cache(maxsize=1)
def arrays():
    return np.load(GOLDEN / "golden.npz")


def _dtype(s: str):
    return np.dtype(s)


def _cfg_knots(name: str) -> np.ndarray:
    from paper_1506_08620_b200 import workloads

    m = re.match(r"(cfg\d)(?:_s(\d+))?(?:_(\d+))?(_unfiltered)?$", name)
    cfg, seed, n1, unf = m.group(1), m.group(2), m.group(3), m.group(4)
    kw = {}
    if seed is not None:
        kw["seed"] = int(seed)
    if n1 is not None:
        kw["n1"] = int(n1)
    if unf:
        kw["filtered"] = False
    return workloads.knots(cfg, **kw).values


def knots_for(case: dict) -> np.ndarray:
    name = case["name"]
    a = arrays()
    if f"{name}/x" in a:
        x = a[f"{name}/x"]
    elif name.startswith("sweep_"):
        _, prec, size = name.split("_")[:3]
        x = orc.gen_uniform_gap(int(size), 1, 5, SEED + int(size), np.float32 if prec == "single" else np.float64)
    elif name.startswith("probes_"):
        _, prec, size = name.split("_")
        x = orc.gen_uniform_gap(int(size), 1, 5, SEED + int(size), np.float32 if prec == "single" else np.float64)
    elif name.startswith("worked_"):
        prec = name.split("_")[1]
        x = np.array([0.0, 0.5, 0.7, 1.1], dtype=np.float32 if prec == "single" else np.float64)
    elif name.startswith("cfg"):
        base = re.sub(r"_(stream|edges)$", "", name)
        x = _cfg_knots(base)
    else:
        raise KeyError(name)
    if "x_sha" in case:
        assert sha(x) == case["x_sha"], f"recipe drift for {name}"
    return x


def edge_probes(xs: np.ndarray, h, r: int) -> np.ndarray:
    """Same construction as make_golden.py (bucket edges +-3 ulp, knots, knot
    neighbours)."""
    rng = np.random.default_rng(11)
    t = xs.dtype.type
    j = rng.integers(0, r + 1, size=20_000).astype(np.float64)
    base = (float(xs[0]) + j / float(h)).astype(xs.dtype)
    zs = [base]
    lo, hi = base.copy(), base.copy()
    for _ in range(3):
        lo = np.nextafter(lo, t(-np.inf))
        hi = np.nextafter(hi, t(np.inf))
        zs += [lo, hi]
    knots_in = xs[:-1]
    zs += [knots_in, np.nextafter(knots_in, t(np.inf)), np.nextafter(xs[1:], t(-np.inf))]
    ze = np.concatenate(zs)
    return ze[(ze >= xs[0]) & (ze < xs[-1])]


def queries_for(case: dict, xs: np.ndarray) -> np.ndarray:
    name = case["name"]
    a = arrays()
    if f"{name}/z" in a:
        z = a[f"{name}/z"]
    elif name.startswith("sweep_"):
        size = int(name.split("_")[2])
        z = orc.random_queries(xs, 100_000, SEED + size + 1)
    elif name.endswith("_stream"):
        from paper_1506_08620_b200 import workloads
        from paper_1506_08620_b200.partition import validate_partition

        cfg = name.split("_")[0]
        z = workloads.queries_host(cfg, validate_partition(xs), 200_000, seed=7)
    elif name.endswith("_edges"):
        h, r, _, _ = orc.compute_h_r(xs)
        z = edge_probes(xs, h, r)
    else:
        raise KeyError(name)
    assert sha(z) == case["z_sha"], f"query recipe drift for {name}"
    return z


def expected_answers(case: dict):
    """Full answers when stored, else None (compare SHA-256 of int64 answers)."""
    a = arrays()
    key = f"{case['name']}/ans"
    return a[key].astype(np.int64) if key in a else None


def check_answers(case: dict, got: np.ndarray) -> None:
    got = np.asarray(got).astype(np.int64)
    want = expected_answers(case)
    if want is not None:
        bad = np.flatnonzero(got != want)
        assert bad.size == 0, f"{case['name']}: {bad.size} mismatches, first at {bad[:5]}"
    assert sha(got) == case["ans_sha"], f"{case['name']}: answer hash differs from the reference"


def build_cases(filter_fn=None):
    return [c for c in meta()["builds"] if filter_fn is None or filter_fn(c)]


def query_cases(filter_fn=None):
    return [c for c in meta()["queries"] if filter_fn is None or filter_fn(c)]
