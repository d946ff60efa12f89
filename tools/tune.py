"""Launch-geometry / algorithm sweep for the search kernels (tuning aid, not
part of the product).  Times each variant with CUDA events over device-
resident queries and prints one JSON line per variant.

    python tools/tune.py [--configs cfg3,cfg4] [--geometry] [--steps 10]

Config specs: cfgN (BASELINE recipes), cfg5:<N+1>, cfg2:<seed>, cfg5u (the
unfiltered cfg5 draw, bitset2 fall-back instance), unif32:<size> / unif64:<size> (the throughput sweep's
U[1,5]-gap partitions), big32:<N+1> (sorted f32
U[0,1) knots).  Layout variants: direct-k (plain K), direct-rank (rank
directory only), direct-hot / direct-hot:<KB> / direct-nohot (hot window on, of a given size, off), direct-nozoned (zoned records off), direct-count / direct-nocount (count words forced / excluded), direct-sparse2 / direct-rec / direct-rec8 (two-level sparse table / 16-B / 8-B group
records forced), bitset2-flat (no subtree records),
direct-gap2-k (gap 2 over plain K), fallback (prepare_with_fallback), gap:<q>
(direct with gap q over its count directory).
"""

from __future__ import annotations

import argparse
import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1506_08620_b200 as fs  # noqa: E402
from paper_1506_08620_b200 import workloads  # noqa: E402

PEAK = 6461.2


def time_launch(fn, steps, warmup=3):
    for _ in range(warmup):
        fn()
    torch.cuda.synchronize()
    a = torch.cuda.Event(enable_timing=True)
    b = torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(steps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / 1e3 / steps


def verify(p, z, out):
    x = p.device_values()
    o = out.long().clamp(0, p.n_intervals - 1)
    return bool(((x[o] <= z) & (z < x[o + 1])).all().item())


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="cfg3")
    ap.add_argument("--algos", default="direct,direct-cache,bitset2")
    ap.add_argument("--geometry", action="store_true")
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--m", type=int, default=0)
    ap.add_argument("--out-bytes", type=int, default=4)
    ap.add_argument("--smem-kb", type=int, default=0, help="cap the planners' shared-memory budget (KB)")
    args = ap.parse_args()
    if args.smem_kb:
        from paper_1506_08620_b200 import batch as _bb

        _bb.SMEM_BUDGET_OVERRIDE = args.smem_kb * 1024
    torch.cuda.set_device(0)
    for spec in args.configs.split(","):
        name, _, arg = spec.partition(":")
        kw = {"n1": int(arg)} if name == "cfg5" and arg else ({"seed": int(arg)} if arg else {})
        if name == "cfg5u":  # the unfiltered cfg5 draw: direct raises Overflow, bitset2 is the fallback
            name, kw = "cfg5", {"n1": int(arg or 1048577), "filtered": False}
        if name == "big32":  # f32 sorted U[0,1) with 2^20 / 2^22 knots: bitset2 with several global levels
            n1 = int(arg or 1048577)
            rng = np.random.default_rng(5)
            xs = np.unique(rng.uniform(0, 1, n1 + n1 // 8).astype(np.float32))[:n1]
            p = fs.validate_partition(xs)
            z = (torch.rand(1 << 28, device="cuda", generator=torch.Generator(device="cuda").manual_seed(1))
                 * float(xs[-1] - xs[0]) + float(xs[0])).float()
            z = torch.clamp(z, max=float(np.nextafter(xs[-1], np.float32(0))))
            out = torch.empty(z.numel(), dtype=torch.int32, device="cuda")
            fb = fs.new_status()
            for algo in args.algos.split(","):
                if algo not in ("bitset2",):
                    continue
                prep = fs.prepare(algo, p)
                t = time_launch(lambda: prep.launch(z, out, fb), args.steps)
                ok = fs.first_bad_of(fb) is None and verify(p, z, out)
                print(json.dumps({"config": spec, "algo": algo, "m": z.numel(), "gqs": round(z.numel() / t / 1e9, 2),
                                  "ok": ok, "placement": prep.placement()}), flush=True)
            continue
        if name in ("unif32", "unif64"):  # the throughput sweep's partitions: gaps U[1, 5], seed 42
            prec = "single" if name == "unif32" else "double"
            p = fs.gen_uniform_gap_partition(int(arg), 1.0, 5.0, 42, prec)
            m = args.m or (1 << 28)
            zh = np.array(fs.gen_queries(p, 1 << 24, 43).values)
            z = torch.from_numpy(zh).cuda().repeat(m >> 24)
        else:
            p = workloads.knots(name, **kw)
            m = args.m or workloads.CONFIGS[name].m
            z = workloads.queries_device(name, p, m, seed=1)
        out = torch.empty(m, dtype=torch.int32 if args.out_bytes == 4 else torch.int64, device="cuda")
        fb = fs.new_status()
        qbytes = z.element_size() + out.element_size()
        if name == "cfg3" or args.geometry:
            zi = z.view(torch.int32) if z.element_size() == 4 else z.view(torch.int64)
            oo = out if z.element_size() == out.element_size() else out
            t = time_launch(lambda: oo.copy_(zi[: oo.numel()].to(oo.dtype)) if False else oo.copy_(zi.to(oo.dtype, copy=False)), args.steps)
            print(json.dumps({"config": spec, "variant": "torch copy ceiling", "ms": t * 1e3,
                              "gbs": qbytes * m / t / 1e9, "frac": qbytes * m / t / 1e9 / PEAK}), flush=True)
        for algo in args.algos.split(","):
            try:
                base = {"direct-k": "direct", "direct-rank": "direct", "direct-hot": "direct", "direct-nohot": "direct",
                        "direct-nozoned": "direct", "direct-count": "direct", "direct-nocount": "direct",
                        "direct-nobytes": "direct", "direct-norows": "direct",
                        "bitset2-flat": "bitset2", "direct-gap2-k": "direct-gap2"}.get(algo, algo)
                if algo.startswith("direct-hot:") or algo.startswith("direct-count:"):
                    base = "direct"
                if algo in ("direct-sparse2", "direct-rec", "direct-rec8", "direct-rec12", "direct-rec8x3"):
                    from paper_1506_08620_b200 import batch as _b

                    keep = (_b.SPARSE_FORMATS, _b.SPARSE_RECORDS_MAX_PAST_SIXTH_PPM, _b.SPARSE_RECORDS8_MAX_PAST_PPM)
                    _b.SPARSE_FORMATS = {"direct-sparse2": ("two-level",), "direct-rec": ("records",),
                                         "direct-rec8": ("records8",), "direct-rec12": ("records12",),
                                         "direct-rec8x3": ("records8x3",)}[algo]
                    _b.SPARSE_RECORDS_MAX_PAST_SIXTH_PPM = _b.SPARSE_RECORDS8_MAX_PAST_PPM = 10**6
                    try:
                        prep = fs.prepare("direct", p)
                    finally:
                        (_b.SPARSE_FORMATS, _b.SPARSE_RECORDS_MAX_PAST_SIXTH_PPM,
                         _b.SPARSE_RECORDS8_MAX_PAST_PPM) = keep
                elif algo == "fallback":  # prepare_with_fallback: direct, else gap-q count directory, else bitset2
                    prep = fs.prepare_with_fallback(p)
                elif algo.startswith("gap:"):  # direct with gap q over its count directory
                    prep = fs.prepare_direct_gap(p, int(algo.split(":")[1]))
                else:
                    prep = fs.prepare(base, p)
                if algo == "direct-k":  # plain K table instead of rank directory / records
                    prep.plan.rank = None
                    prep.plan.records = None
                if algo == "direct-rank":
                    prep.plan.records = None
                    prep.plan.sparse = None
                if algo == "direct-hot":
                    prep = fs.prepare("direct", p, hot_window=True)
                if algo == "direct-nohot":
                    prep = fs.prepare("direct", p, hot_window=False)
                if algo.startswith("direct-count:"):  # count words forced within a shared-memory budget (KB)
                    from paper_1506_08620_b200 import batch as _b

                    keep_c = (_b.SPARSE_FORMATS, _b.COUNT_WORDS_MAX_RARE_PPM, _b.COUNT_WORDS_MAX_L2_XREAD_PPM,
                              _b.COUNT_WORDS_MAX_XREAD_PPM, _b.COUNT_WORDS_BUDGET_BYTES)
                    _b.SPARSE_FORMATS = ("count-words",)
                    _b.COUNT_WORDS_MAX_RARE_PPM = _b.COUNT_WORDS_MAX_L2_XREAD_PPM = 10**6
                    _b.COUNT_WORDS_MAX_XREAD_PPM = 10**6
                    _b.COUNT_WORDS_BUDGET_BYTES = int(algo.split(":")[1]) * 1024
                    try:
                        prep = fs.prepare("direct", p)
                    finally:
                        (_b.SPARSE_FORMATS, _b.COUNT_WORDS_MAX_RARE_PPM, _b.COUNT_WORDS_MAX_L2_XREAD_PPM,
                         _b.COUNT_WORDS_MAX_XREAD_PPM, _b.COUNT_WORDS_BUDGET_BYTES) = keep_c
                if algo in ("direct-count", "direct-nocount"):  # count words forced / excluded
                    from paper_1506_08620_b200 import batch as _b

                    keep_c = (_b.SPARSE_FORMATS, _b.COUNT_WORDS_MAX_RARE_PPM, _b.COUNT_WORDS_MAX_L2_XREAD_PPM,
                              _b.COUNT_WORDS_MAX_XREAD_PPM)
                    if algo == "direct-count":
                        _b.SPARSE_FORMATS = ("count-words",)
                        _b.COUNT_WORDS_MAX_RARE_PPM = _b.COUNT_WORDS_MAX_L2_XREAD_PPM = 10**6
                        _b.COUNT_WORDS_MAX_XREAD_PPM = 10**6
                    else:
                        _b.SPARSE_FORMATS = tuple(n for n in keep_c[0] if n != "count-words")
                    try:
                        prep = fs.prepare("direct", p)
                    finally:
                        (_b.SPARSE_FORMATS, _b.COUNT_WORDS_MAX_RARE_PPM, _b.COUNT_WORDS_MAX_L2_XREAD_PPM,
                         _b.COUNT_WORDS_MAX_XREAD_PPM) = keep_c
                if algo == "direct-norows":  # the 8-B rank directory through L2 (no 16-B rank rows)
                    from paper_1506_08620_b200 import batch as _b

                    keep_rr = _b.RANK_ROWS_MIN_KNOT_SHARE
                    _b.RANK_ROWS_MIN_KNOT_SHARE = 0
                    try:
                        prep = fs.prepare("direct", p)
                    finally:
                        _b.RANK_ROWS_MIN_KNOT_SHARE = keep_rr
                if algo == "direct-nobytes":  # the staged directory alone, X through L2 (no knot bytes)
                    from paper_1506_08620_b200 import batch as _b

                    _b.KNOT_BYTES = False
                    try:
                        prep = fs.prepare("direct", p)
                    finally:
                        _b.KNOT_BYTES = True
                if algo == "direct-nozoned":  # no zoned records: the hot window / L2 directory
                    from paper_1506_08620_b200 import batch as _b

                    _b.ZONED = False
                    try:
                        prep = fs.prepare("direct", p)
                    finally:
                        _b.ZONED = True
                if algo.startswith("direct-hot:"):
                    from paper_1506_08620_b200 import batch as _b

                    keep_hw = _b.HOT_WINDOW_BYTES
                    _b.HOT_WINDOW_BYTES = int(algo.split(":")[1]) * 1024
                    try:
                        prep = fs.prepare("direct", p, hot_window=True)
                    finally:
                        _b.HOT_WINDOW_BYTES = keep_hw
                if algo == "bitset2-flat":  # global levels from the padded array (no subtree records)
                    prep.plan.b2_deep = None
                if algo == "direct-gap2-k":  # gap-2 over its plain K table (no rank directory)
                    prep.plan.rank = None
            except fs.InfeasibleError as e:
                print(json.dumps({"config": spec, "algo": algo, "infeasible": type(e).__name__}), flush=True)
                continue
            geos = [0]
            if args.geometry:
                geos = [0] + [thr | (cap << 12) for thr in (256, 512, 1024) for cap in (0, 1, 2, 3, 4, 6, 8)]
            for tune in geos:
                prep.plan.tune = tune
                try:
                    t = time_launch(lambda: prep.launch(z, out, fb), args.steps)
                except Exception as e:  # geometry that does not fit
                    print(json.dumps({"config": spec, "algo": algo, "tune": tune, "error": str(e)[:80]}), flush=True)
                    continue
                ok = fs.first_bad_of(fb) is None and verify(p, z, out)
                gbs = qbytes * m / t / 1e9
                print(json.dumps({
                    "config": spec, "algo": algo, "threads": tune & 0xfff, "cap": tune >> 12, "m": m,
                    "ms": round(t * 1e3, 4), "gqs": round(m / t / 1e9, 2), "gbs": round(gbs, 1),
                    "frac": round(gbs / PEAK, 4), "ok": ok, "placement": prep.placement(),
                    "r": getattr(prep.structure, "r", None), "algorithm": prep.algorithm,
                    "q": getattr(prep.structure, "q", None),
                }), flush=True)
            prep.plan.tune = 0
        del z, out
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
