"""Hypothesis strategies: adversarial strictly increasing knot arrays."""

import numpy as np
from hypothesis import strategies as st


@st.composite
def partitions(draw, max_size=96):
    """Strictly increasing float32/float64 knots with mixed gap scales:
    near-duplicate gaps (a few ulps), gap ratios up to ~1e6, negative and
    tiny-magnitude origins, and subnormal-neighbourhood values."""
    dtype = draw(st.sampled_from([np.float32, np.float64]))
    n1 = draw(st.integers(min_value=2, max_value=max_size))
    seed = draw(st.integers(min_value=0, max_value=2**32 - 1))
    rng = np.random.default_rng(seed)
    kind = draw(st.sampled_from(["uniform", "geometric", "clustered", "ulp", "tiny", "offset", "collide"]))
    if kind == "uniform":
        gaps = rng.uniform(1.0, 5.0, n1 - 1)
    elif kind == "geometric":
        gaps = 1e-3 * np.exp(rng.uniform(0, np.log(1e4), n1 - 1))
    elif kind == "clustered":
        gaps = np.where(rng.random(n1 - 1) < 0.2, 1e-4, 1.0) * rng.uniform(1, 2, n1 - 1)
    elif kind == "ulp":
        gaps = np.full(n1 - 1, 1.0)
    elif kind == "tiny":
        gaps = rng.uniform(1.0, 3.0, n1 - 1) * (1e-40 if dtype == np.float32 else 1e-310)
    else:
        gaps = rng.uniform(0.5, 1.5, n1 - 1)
    origin = {"offset": draw(st.sampled_from([-1e6, -3.5, 1e3, 12345.678])), "tiny": 0.0}.get(kind, 0.0)
    x = (origin + np.concatenate([[0.0], np.cumsum(gaps)])).astype(dtype)
    if kind == "ulp":
        # consecutive representable values: minimum possible spacing
        start = dtype(draw(st.sampled_from([1.0, 1024.0, -7.0])))
        x = [start]
        for _ in range(n1 - 1):
            x.append(np.nextafter(x[-1], dtype(np.inf)))
        x = np.array(x, dtype=dtype)
    if kind == "collide":
        # a far-away first knot: offsets X_i - X_0 round onto each other
        # (NotDistinguishable), or nearly so (growth, gap-2 rescue)
        far = dtype(-1e9 if dtype == np.float32 else -1e18)
        x = np.concatenate([[far], (np.cumsum(rng.uniform(0.5, 200.0, n1 - 1))).astype(dtype)]).astype(dtype)
    x = np.unique(x)  # casting can merge neighbours
    if len(x) < 2:
        x = np.array([0.0, 1.0], dtype=dtype)
    assert np.all(np.isfinite(x)) and np.all(np.diff(x) > 0)
    return x


@st.composite
def big_partitions(draw):
    """Large strictly increasing knot arrays (2^12 .. 2^20 + 1 knots) that
    reach the big-table device paths: subtree records below the smem top
    and f32 shadow keys (bitset2), the sparse two-level table, group and
    zoned records, the hot window and the L2 rank directory (direct),
    bank-replicated levels with large batches."""
    dtype = draw(st.sampled_from([np.float32, np.float64]))
    n1 = draw(st.sampled_from([(1 << 12) + 1, 5000, (1 << 15) + 1, 70_000, (1 << 17) + 3, 300_000, (1 << 20) + 1]))
    seed = draw(st.integers(min_value=0, max_value=2**32 - 1))
    rng = np.random.default_rng(seed)
    kind = draw(st.sampled_from(["uniform", "geometric", "clustered", "sorted_random", "offset"]))
    if kind == "uniform":
        gaps = rng.uniform(1.0, 5.0, n1 - 1)
    elif kind == "geometric":  # growth capped so float32 stays finite at 2^20 knots
        gaps = 1e-4 * 1.0001 ** (np.arange(n1 - 1) % 60_000) * rng.uniform(0.9, 1.1, n1 - 1)
    elif kind == "clustered":
        gaps = np.where(rng.random(n1 - 1) < 0.3, 1e-3, 1.0) * rng.uniform(1, 2, n1 - 1)
    elif kind == "sorted_random":
        gaps = np.diff(np.sort(rng.uniform(0, 1, n1 + 1)))[: n1 - 1] + 1e-7
    else:
        gaps = rng.uniform(0.5, 1.5, n1 - 1)
    origin = -2.0e4 if kind == "offset" else 0.0
    x = np.unique((origin + np.concatenate([[0.0], np.cumsum(gaps)])).astype(dtype))
    assert len(x) >= 2 and np.all(np.diff(x) > 0)
    return x
