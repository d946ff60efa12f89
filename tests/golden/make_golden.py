"""Generate the golden fixtures by running the REFERENCE itself.

Run in the build container, where the reference package is importable:

    PYTHONPATH=/root/reference/pkg/src:. python tests/golden/make_golden.py

It imports ``fastsearch`` (the unmodified reference, /root/reference/pkg/src)
and records, for every index-build case the reference's own tests pin
(pkg/tests/test_direct.py, test_acceptance.py) plus the five BASELINE
configs, the reference's outputs: h (raw bits), r, increments, h_start bits,
K (in full when small, else SHA-256 + a seeded sample), and query answers
(in full for the small probe sets, SHA-256 for the large sweeps).  The
fixtures travel with the repo; nothing at test time reads /root/reference.
"""

from __future__ import annotations

import hashlib
import json
import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
ROOT = HERE.parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, "/root/reference/pkg/tests")

from fastsearch import batch as ref_batch  # noqa: E402
from fastsearch import direct as ref_direct  # noqa: E402
from fastsearch import errors as ref_errors  # noqa: E402
from fastsearch import partition as ref_partition  # noqa: E402
from helpers import boundary_probes as ref_boundary_probes  # noqa: E402
from helpers import random_queries as ref_random_queries  # noqa: E402

from paper_1506_08620_b200 import workloads  # noqa: E402  (host-side knot recipes only)

SEED = 20240708  # pkg/tests/test_acceptance.py:28
FULL_K_MAX = 4096
K_SAMPLE = 1000


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def bits(v) -> int:
    v = np.asarray(v)
    return int(v.view(np.uint32 if v.dtype == np.float32 else np.uint64))


def build_case(name, p, q=1, qbits=32, arrays=None, store_x=True):
    """Reference compute_h_r + build_index on partition p."""
    case = {"name": name, "dtype": str(p.values.dtype), "n1": len(p.values), "q": q, "qbits": qbits,
            "x_sha": sha(p.values)}
    if store_x:
        arrays[f"{name}/x"] = p.values
    try:
        h, r, st = ref_direct.compute_h_r(p, qbits=qbits, q=q)
    except ref_errors.NotDistinguishable as e:
        case["error"] = "not_distinguishable"
        case["position"] = int(e.position)
        return case
    except ref_errors.Overflow:
        case["error"] = "overflow"
        return case
    case["h_bits"] = bits(h)
    case["h_repr"] = repr(float(h))
    case["r"] = int(r)
    case["increments"] = int(st.increments)
    case["growth_total"] = float(st.growth_total)
    # initial guess exactly as direct.py:454-464 forms it
    xs = p.values
    offs = xs - xs[0]
    basis = min(q, len(xs) - 1)
    with np.errstate(over="ignore"):
        h_start = xs.dtype.type(1.0) / (offs[basis:] - offs[:-basis]).min()
    case["h_start_bits"] = bits(h_start)
    idx = ref_direct.build_index(p, h, r, q=q, qbits=qbits)
    k = idx.k
    case["k_len"] = int(len(k))
    case["k_sha"] = sha(k)
    f = ref_direct.knot_buckets(p, h)
    case["f_sha"] = sha(f)
    if len(k) <= FULL_K_MAX:
        arrays[f"{name}/k"] = k
    rng = np.random.default_rng(len(k))
    pos = np.sort(rng.integers(0, len(k), size=min(K_SAMPLE, len(k))))
    arrays[f"{name}/k_sample_pos"] = pos.astype(np.int64)
    arrays[f"{name}/k_sample"] = k[pos]
    if q == 1 and len(k) <= 1 << 24:
        fused = ref_direct.with_fused(idx, p).fused
        case["fused_sha"] = sha(fused)
    return case


def query_case(name, p, z, arrays, store=True, algorithms=("direct", "bitset2")):
    """Reference answers for queries z: linear-scan oracle (small) and run_batch."""
    case = {"name": name, "dtype": str(p.values.dtype), "m": int(len(z)), "z_sha": sha(z)}
    if len(z) <= 200_000:
        want = ref_partition.linear_scan_oracle_batch(p, z)
    else:
        want = ref_batch.run_batch(ref_batch.prepare("bitset2", p), z, d=65536, threads=8)
    for a in algorithms:
        try:
            got = ref_batch.run_batch(ref_batch.prepare(a, p), z, d=65536, threads=8)
        except ref_errors.InfeasibleError:
            continue
        assert np.array_equal(got, want), (name, a)
    case["ans_sha"] = sha(want.astype(np.int64))
    if store:
        arrays[f"{name}/z"] = z
        arrays[f"{name}/ans"] = want.astype(np.int32)
    return case


def main():
    arrays: dict[str, np.ndarray] = {}
    builds, queries = [], []
    vp = ref_partition.validate_partition
    gp = ref_partition.gen_uniform_gap_partition

    # --- reference test pins (pkg/tests/test_direct.py, test_acceptance.py) ---
    for prec, dt in (("single", np.float32), ("double", np.float64)):
        worked = vp(np.array([0.0, 0.5, 0.7, 1.1], dtype=dt))
        builds.append(build_case(f"worked_{prec}", worked, arrays=arrays))
        builds.append(build_case(f"worked_{prec}_q2", worked, q=2, arrays=arrays))
        queries.append(query_case(f"worked_{prec}", worked, np.array([0.6, 0.0, np.nextafter(dt(1.1), dt(-np.inf))], dtype=dt), arrays))
    builds.append(build_case("unit4", vp([0.0, 1.0, 2.0, 3.0]), arrays=arrays))
    builds.append(build_case("unit4_q2", vp([0.0, 1.0, 2.0, 3.0]), q=2, arrays=arrays))
    builds.append(build_case("two_knots", vp([0.0, 1.0]), arrays=arrays))
    builds.append(build_case("two_knots_q2", vp([0.0, 2.5]), q=2, arrays=arrays))
    collide = vp(np.array([-1e9, 0.0, 1.0], dtype=np.float32))
    builds.append(build_case("collide_f32", collide, arrays=arrays))
    builds.append(build_case("collide_f32_q2", collide, q=2, arrays=arrays))
    builds.append(build_case("subnormal_gap_f32", vp(np.array([0.0, 1.42e-45, 1.0], dtype=np.float32)), arrays=arrays))
    for prec, seeds in (("single", (116, 733, 995, 1216)), ("double", (32, 173, 285, 656))):
        for s in seeds:
            builds.append(build_case(f"growth_{prec}_{s}", gp(15, 1, 5, seed=s, precision=prec), arrays=arrays))
    builds.append(build_case("gap2_33_s21", gp(33, 1, 5, seed=21), q=2, arrays=arrays))
    builds.append(build_case("gap3_63_s8", gp(63, 1, 5, seed=8), q=3, arrays=arrays))
    builds.append(build_case("qbits64_255_s7", gp(255, 1, 5, seed=7), qbits=64, arrays=arrays))
    for prec in ("single", "double"):
        for size in range(2, 65):
            for tag, seed in (("s", size), ("S", SEED + size)):
                p = gp(size, 1, 5, seed=seed, precision=prec)
                builds.append(build_case(f"small_{prec}_{size}_{tag}", p, arrays=arrays))
                if tag == "S":
                    queries.append(query_case(f"probes_{prec}_{size}", p, ref_boundary_probes(p), arrays,
                                              algorithms=ref_batch.ALGORITHMS))
        for size in (15, 255, 4095, 65535):
            p = gp(size, 1, 5, seed=SEED + size, precision=prec)
            builds.append(build_case(f"sweep_{prec}_{size}", p, arrays=arrays, store_x=False))
            if size <= 4095:
                builds.append(build_case(f"sweep_{prec}_{size}_q2", p, q=2, arrays=arrays, store_x=False))
            z = ref_random_queries(p, 100_000, seed=SEED + size + 1)
            queries.append(query_case(f"sweep_{prec}_{size}", p, z, arrays, store=False,
                                      algorithms=ref_batch.ALGORITHMS))

    # --- the five BASELINE configs (knot recipes in paper_1506_08620_b200.workloads) ---
    cfgs = [("cfg1_s0", "cfg1", dict(seed=0)), ("cfg1_s1", "cfg1", dict(seed=1)), ("cfg1_s2", "cfg1", dict(seed=2)),
            ("cfg2_s0", "cfg2", dict(seed=0)), ("cfg2_s1", "cfg2", dict(seed=1)), ("cfg2_s2", "cfg2", dict(seed=2)),
            ("cfg3_s0", "cfg3", dict(seed=0)), ("cfg4", "cfg4", {}),
            ("cfg5_33", "cfg5", dict(n1=33)), ("cfg5_1025", "cfg5", dict(n1=1025)),
            ("cfg5_32769", "cfg5", dict(n1=32769)), ("cfg5_1048577", "cfg5", dict(n1=1048577)),
            ("cfg5_1048577_unfiltered", "cfg5", dict(n1=1048577, filtered=False)),
            ("cfg5_32769_unfiltered", "cfg5", dict(n1=32769, filtered=False))]
    for cname, cfg, kw in cfgs:
        p = workloads.knots(cfg, **kw)
        pr = vp(p.values)
        builds.append(build_case(cname, pr, arrays=arrays, store_x=False))
        if cname.endswith("unfiltered"):
            continue
        # uniform sample of the config's own query stream + bucket-edge probes
        z = workloads.queries_host(cfg, p, 200_000, seed=7)
        queries.append(query_case(f"{cname}_stream", pr, z, arrays, store=False))
        try:
            h, r, _ = ref_direct.compute_h_r(pr)
        except ref_errors.InfeasibleError:
            continue
        rng = np.random.default_rng(11)
        t = pr.values.dtype.type
        j = rng.integers(0, r + 1, size=20_000).astype(np.float64)
        base = (float(pr.values[0]) + j / float(h)).astype(pr.values.dtype)
        zs = [base]
        lo, hi = base.copy(), base.copy()
        for _ in range(3):
            lo = np.nextafter(lo, t(-np.inf))
            hi = np.nextafter(hi, t(np.inf))
            zs += [lo, hi]
        knots_in = pr.values[:-1]
        zs += [knots_in, np.nextafter(knots_in, t(np.inf)), np.nextafter(pr.values[1:], t(-np.inf))]
        ze = np.concatenate(zs)
        ze = ze[(ze >= pr.values[0]) & (ze < pr.values[-1])]
        queries.append(query_case(f"{cname}_edges", pr, ze, arrays, store=False))

    # --- out-of-domain positions (test_batch.py:63-81, test_partition.py:183-187) ---
    ood = []
    p = gp(255, 1, 5, seed=2000, precision="double")
    z = ref_random_queries(p, 10, seed=2001)
    z[3] = p.values[-1]
    z[7] = p.values[0] - 1
    try:
        ref_batch.run_batch(ref_batch.prepare("direct", p), z, d=2)
    except ref_errors.OutOfDomain as e:
        ood.append({"name": "right_endpoint", "position": int(e.position)})
        arrays["ood/right_endpoint/x"] = p.values
        arrays["ood/right_endpoint/z"] = z
    z = ref_random_queries(p, 8, seed=2001)
    z[5] = np.nan
    try:
        ref_batch.run_batch(ref_batch.prepare("bitset2", p), z, d=4)
    except ref_errors.OutOfDomain as e:
        ood.append({"name": "nan", "position": int(e.position)})
        arrays["ood/nan/z"] = z

    meta = {"generator": "tests/golden/make_golden.py", "reference": "fastsearch 0.1.0 (/root/reference/pkg)",
            "numpy": np.__version__, "builds": builds, "queries": queries, "out_of_domain": ood}
    (HERE / "golden.json").write_text(json.dumps(meta, indent=1))
    np.savez_compressed(HERE / "golden.npz", **arrays)
    print(f"{len(builds)} build cases, {len(queries)} query cases, {len(arrays)} arrays")


if __name__ == "__main__":
    main()
