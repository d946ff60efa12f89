#!/usr/bin/env python
"""Benchmark of the B200 sorted-interval lookup (arXiv 1506.08620 hot path).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

One JSON line on rank 0.  Workload (BASELINE.json configs[2], "cfg3", the
streaming config the >=70%-of-roofline target and the 1/2/4/8-GPU sharding
are quoted on): float32 knots X, N+1 = 4,097, spacing 0.5 + U[0,1) summed
from 0 (seed 0); 2^30 float32 queries Uniform[X0, XN) PER GPU (weak
scaling: each rank owns a 2^30-query shard of an N x 2^30 global stream,
X and J built locally on every GPU, no per-query communication).

A step = one batch search over the rank's 2^30 queries with the direct
search kernel (one launch).  ``value`` = queries/s with queries resident in
HBM (CUDA events on the launching stream, max over ranks); ``e2e`` = the
same metric through the public drop-in API (``batch_search`` on pinned host
numpy arrays: H2D copies, kernel and D2H inside every step); ``bsearch`` =
the branchless binary search (Alg 3, bitset2) timed identically -- the
"direct vs binary search" half of the metric.  Inputs are 4 GiB + 4 GiB of
output per GPU, far larger than the 126 MB L2, so no flush is needed; the
``per_config`` sweep flushes L2 before every launch of a stream that fits in
it (cfg1).

``--impl reference`` times the reference's CPU path (its numpy lane kernel
and thread-span driver, restated in oracle/fs_oracle.py -- the reference
itself is Python and cannot travel to the GPU box) on all host cores, on a
bounded sample of the same workload.
"""

from __future__ import annotations

import argparse
import json
import os
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "queries/sec and achieved HBM GB/s (fraction of roofline), direct vs binary search"
UNIT = "queries/s"
M_PER_GPU = 1 << 30
BYTES_PER_QUERY = 8  # 4 B float32 query read + 4 B int32 index written
SPEC_HBM_GBS = 8000.0  # B200 nominal HBM3e bandwidth (secondary denominator)
CPU_SAMPLE = 1 << 24


def peaks() -> dict:
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return {"hbm_gbs": float(d["hbm_gbs"]), "source": "measured (MEASURED_PEAKS.json)"}
    return {"hbm_gbs": 6650.0, "source": "fallback (B200_PROFILING.md)"}


def ncu_traffic() -> dict | None:
    """DRAM bytes per launch of the direct kernel from the committed ncu
    capture (profiles/ncu_direct_cfg3.json), if one exists."""
    p = ROOT / "profiles" / "ncu_direct_cfg3.json"
    if p.exists():
        try:
            return json.loads(p.read_text())
        except Exception:
            return None
    return None


class ClockSampler:
    """NVML sampling of SM clock and clock-event reasons during a region."""

    REASONS = {
        "gpu_idle": 0x1,
        "applications_clocks_setting": 0x2,
        "sw_power_cap": 0x4,
        "hw_slowdown": 0x8,
        "sync_boost": 0x10,
        "sw_thermal_slowdown": 0x20,
        "hw_thermal_slowdown": 0x40,
        "hw_power_brake_slowdown": 0x80,
        "display_clock_setting": 0x100,
    }

    def __init__(self, index: int):
        self.samples = []
        self.reasons = 0
        self._stop = threading.Event()
        self._h = None
        self.max_mhz = None
        try:
            import pynvml

            pynvml.nvmlInit()
            self._nv = pynvml
            self._h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self._h, pynvml.NVML_CLOCK_SM)
        except Exception:
            self._nv = None

    def _run(self):
        nv = self._nv
        while not self._stop.is_set():
            try:
                self.samples.append(nv.nvmlDeviceGetClockInfo(self._h, nv.NVML_CLOCK_SM))
                self.reasons |= int(nv.nvmlDeviceGetCurrentClocksEventReasons(self._h))
            except Exception:
                pass
            self._first.set()
            time.sleep(0.002)

    def __enter__(self):
        if self._nv is not None:
            self._first = threading.Event()
            self._t = threading.Thread(target=self._run, daemon=True)
            self._t.start()
            self._first.wait(5.0)  # the region starts once the sampler is running
            self.samples.clear()  # (that first sample predates the region)
        return self

    def __exit__(self, *exc):
        self._stop.set()
        if self._nv is not None:
            self._t.join()

    def summary(self) -> dict:
        reasons = [k for k, v in self.REASONS.items() if self.reasons & v and k != "gpu_idle"]
        return {
            "sm_mhz": float(np.median(self.samples)) if self.samples else None,
            "sm_max_mhz": self.max_mhz,
            "samples": len(self.samples),
            "reasons": reasons,
        }


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def cpu_reference_rate(xs: np.ndarray, z: np.ndarray, algo: str, steps: int, warmup: int, min_time: float):
    """Reference CPU lane path (restated) over all host cores: queries/s."""
    from oracle import fs_oracle as orc

    threads = os.cpu_count() or 1
    prep = orc.PreparedPort(algo, xs)
    out = np.empty(len(z), dtype=np.int32)
    for _ in range(max(1, warmup)):
        orc.batch_search_port(prep, z, out, d=65536, threads=threads)
    times = []
    t_total = 0.0
    while len(times) < steps or t_total < min_time:
        t0 = time.perf_counter()
        orc.batch_search_port(prep, z, out, d=65536, threads=threads)
        dt = time.perf_counter() - t0
        times.append(dt)
        t_total += dt
        if len(times) >= 10 * max(steps, 1) and t_total >= 0.5 * min_time:
            break
    rate = len(z) / float(np.median(times))
    return rate, threads, len(times), out


def run_reference(args):
    world, rank, _ = dist_env()
    if rank != 0:
        return 0
    from paper_1506_08620_b200 import workloads

    p = workloads.knots("cfg3", seed=0)
    n = args.ref_sample
    z = workloads.queries_host("cfg3", p, n, seed=1)
    rate, threads, reps, _ = cpu_reference_rate(p.values, z, "direct", args.steps, args.warmup,
                                                min_time=args.ref_min_time)
    sample = (f"cfg3 direct lane path (batch.py:315-317 via oracle/fs_oracle.py), {n} queries "
              f"per step, d=65536, {threads} threads, median of {reps} passes")
    line = {
        "impl": "reference",
        "metric": METRIC,
        "value": rate * 1.0,
        "unit": UNIT,
        "n_gpus": args.gpus,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": 1e3 * n / rate,
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "f32",
        "data": "synthetic (seeded cfg3 recipe)",
        "config": {"workload": "cfg3: f32 N+1=4097 gaps 0.5+U[0,1); uniform queries", "queries_per_step": n,
                   "algorithm": "direct"},
        "cpu_baseline": {"value": rate, "unit": UNIT, "cores": threads, "kind": "port", "sample": sample},
        "e2e": {"value": rate, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "gpu_launches": 0,
    }
    print(json.dumps(line), flush=True)
    return 0


def time_device(prep, z, out, fb, steps: int, warmup: int, barrier, flush=None):
    """Warm up, then time exactly ``steps`` launches with CUDA events on the
    launching stream, bracketed by barrier + synchronize.  With ``flush`` (a
    device buffer larger than L2), every launch is preceded by an untimed
    write of that buffer and timed by its own event pair, so a stream that
    fits in L2 is read cold each time."""
    import torch

    for _ in range(warmup):
        prep.launch(z, out, fb)
    torch.cuda.synchronize()
    barrier()
    torch.cuda.synchronize()
    s = torch.cuda.current_stream()
    if flush is not None:
        pairs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
        for a, b in pairs:
            flush.zero_()
            a.record(s)
            prep.launch(z, out, fb)
            b.record(s)
        torch.cuda.synchronize()
        barrier()
        torch.cuda.synchronize()
        return sum(a.elapsed_time(b) for a, b in pairs) / 1e3
    start = torch.cuda.Event(enable_timing=True)
    stop = torch.cuda.Event(enable_timing=True)
    start.record(s)
    for _ in range(steps):
        prep.launch(z, out, fb)
    stop.record(s)
    torch.cuda.synchronize()
    barrier()
    torch.cuda.synchronize()
    return start.elapsed_time(stop) / 1e3  # seconds for `steps` launches


L2_FLUSH_BYTES = 512 << 20  # > 4x the 126 MB L2


PER_CONFIG = (
    # (label, config, knot-recipe kwargs, queries per GPU): BASELINE.json configs[0..4]
    ("cfg1", "cfg1", {"seed": 0}, 1_000_000),
    ("cfg2_s0", "cfg2", {"seed": 0}, 100_000_000),
    ("cfg3", "cfg3", {"seed": 0}, 1 << 30),
    ("cfg4", "cfg4", {}, 1 << 28),
    ("cfg5_33", "cfg5", {"n1": 33}, 1 << 28),
    ("cfg5_1025", "cfg5", {"n1": 1025}, 1 << 28),
    ("cfg5_32769", "cfg5", {"n1": 32_769}, 1 << 28),
    ("cfg5_1048577", "cfg5", {"n1": 1_048_577}, 1 << 28),
)


def per_config(steps: int, barrier, world: int):
    """Every BASELINE config on this GPU: direct (or its fall-back) vs
    bitset2, device-resident, CUDA events, answers verified by the bracket
    property.  Returns {label: {...}} with per-rank times max-reduced."""
    import torch
    import torch.distributed as dist

    import paper_1506_08620_b200 as fs
    from paper_1506_08620_b200 import workloads

    pk = peaks()["hbm_gbs"]
    res = {}
    for label, cfg, kw, m in PER_CONFIG:
        p = workloads.knots(cfg, **kw)
        z = workloads.queries_device(cfg, p, m, seed=11)
        out = torch.empty(m, dtype=torch.int32, device=z.device)
        fb = fs.new_status(z.device)
        qb = z.element_size() + 4
        row = {"queries_per_gpu": m, "dtype": "f32" if p.precision == "single" else "f64", "bytes_per_query": qb}
        # streams that fit in L2 are read cold: the L2 is flushed before every launch
        flush = torch.empty(L2_FLUSH_BYTES, dtype=torch.uint8, device=z.device) if qb * m < L2_FLUSH_BYTES else None
        row["l2"] = "flushed before each launch" if flush is not None else "stream > L2, no flush"
        for name in ("direct", "bitset2"):
            prep = fs.prepare_with_fallback(p) if name == "direct" else fs.prepare("bitset2", p)
            n = steps * (1 if m >= (1 << 30) else 4) * (1 if m >= (1 << 26) else 10)
            t = time_device(prep, z, out, fb, n, 3, barrier, flush) / n
            ok = fs.first_bad_of(fb) is None and verify_bracket(p, z, out)
            tt = torch.tensor([t, 0.0 if ok else 1.0], dtype=torch.float64, device=z.device)
            if world > 1:
                dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            t, bad = tt.tolist()
            row[name] = {
                "algorithm": prep.algorithm,
                "gqs": world * m / t / 1e9,
                "ms": 1e3 * t,
                "roofline_frac": qb * m / t / 1e9 / pk,
                "placement": prep.placement(),
                "verified": bad == 0,
            }
            if name == "direct" and prep.algorithm.startswith("direct"):
                row["R"] = prep.structure.r
        res[label] = row
        del z, out, flush
        torch.cuda.empty_cache()
    return res


def verify_bracket(p, z, out) -> bool:
    """X[out] <= z < X[out+1] for every query (unique answer => equals the
    oracle's max{i : X_i <= z}); exact float compares on the device."""
    import torch

    x = p.device_values()
    o = out.long()
    ok = (o >= 0) & (o < p.n_intervals)
    o = o.clamp(0, p.n_intervals - 1)
    ok &= (x[o] <= z) & (z < x[o + 1])
    return bool(ok.all().item())


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--e2e-steps", type=int, default=None)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--m", type=int, default=M_PER_GPU, help="queries per GPU")
    ap.add_argument("--no-configs", action="store_true", help="skip the per-config sweep (cfg1..cfg5)")
    ap.add_argument("--ref-sample", type=int, default=CPU_SAMPLE, help="--impl reference: queries per step")
    ap.add_argument("--ref-min-time", type=float, default=10.0, help="--impl reference: minimum seconds sampled")
    args = ap.parse_args()
    args.warmup = max(3, args.warmup)
    if args.impl == "reference":
        return run_reference(args)

    import torch
    import torch.distributed as dist

    world, rank, local = dist_env()
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))

        def barrier():
            dist.barrier()
    else:
        def barrier():
            pass

    import paper_1506_08620_b200 as fs
    from paper_1506_08620_b200 import workloads

    m = args.m
    p = workloads.knots("cfg3", seed=0)
    t0 = time.perf_counter()
    prep = fs.prepare("direct", p)
    torch.cuda.synchronize()
    build_ms = 1e3 * (time.perf_counter() - t0)
    prep_b = fs.prepare("bitset2", p)
    z = workloads.queries_device("cfg3", p, m, seed=1 + rank)
    out = torch.empty(m, dtype=torch.int32, device=z.device)
    fb = fs.new_status(z.device)

    with ClockSampler(local) as clk:
        t_dir = time_device(prep, z, out, fb, args.steps, args.warmup, barrier)
    clocks = clk.summary()
    bad = -1 if fs.first_bad_of(fb) is None else 0
    verified = bad == -1 and verify_bracket(p, z, out)
    t_bs = time_device(prep_b, z, out, fb, max(3, args.steps // 5), 3, barrier)
    verified &= verify_bracket(p, z, out)

    # end-to-end through the public API on pinned host buffers (per rank: the
    # full 2^30 shard at N=1; 2^28 at N>1 so N ranks' host buffers stay bounded)
    e2e_steps = args.e2e_steps or max(3, min(args.steps, 10))
    me = m if world == 1 else min(m, 1 << 28)
    zh_t = torch.empty(me, dtype=torch.float32, pin_memory=True)
    zh_t.copy_(z[:me])
    oh_t = torch.empty(me, dtype=torch.int32, pin_memory=True)
    zh, oh = zh_t.numpy(), oh_t.numpy()
    cfg = fs.LaneConfig(d=65536, kernel="direct", structure=prep)
    del z, out
    torch.cuda.empty_cache()
    def timed_calls(call, n):
        """Median seconds of n synchronous public-API calls, each bracketed by
        CUDA events on the current stream (device clock; the call returns only
        after its results are in host memory)."""
        call()  # warm-up (allocator, copy stream, pinned staging slots)
        barrier()
        ts = []
        for _ in range(n):
            torch.cuda.synchronize()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            call()
            b.record()
            b.synchronize()
            ts.append(a.elapsed_time(b) / 1e3)
        barrier()
        return float(np.median(ts))

    t_e2e = timed_calls(lambda: fs.batch_search(cfg, zh, oh), e2e_steps)
    # opt-in speculative write-back (atomic=False): both PCIe directions overlap
    t_e2e_ov = timed_calls(lambda: fs.batch_search(cfg, zh, oh, atomic=False), e2e_steps)
    # what a drop-in numpy user passes: ordinary pageable arrays (staged by the library)
    zpg = zh.copy()
    opg = np.empty_like(oh)
    t_e2e_pg = timed_calls(lambda: fs.batch_search(cfg, zpg, opg), 3)
    del zpg, opg

    times = torch.tensor([t_dir, t_bs, t_e2e, t_e2e_ov, t_e2e_pg], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(times, op=dist.ReduceOp.MAX)
        v = torch.tensor([1 if verified else 0], device="cuda")
        dist.all_reduce(v, op=dist.ReduceOp.MIN)
        verified = bool(v.item())
    t_dir, t_bs, t_e2e, t_e2e_ov, t_e2e_pg = times.tolist()
    z_cpu, o_cpu = zh[:CPU_SAMPLE].copy(), oh[:CPU_SAMPLE].copy()
    del zh_t, oh_t, zh, oh
    torch.cuda.empty_cache()
    configs = None if args.no_configs else per_config(max(3, min(args.steps, 10)), barrier, world)

    if rank == 0:
        total = m * world
        step = t_dir / args.steps
        value = total / step
        bs_steps = max(3, args.steps // 5)
        pk = peaks()
        achieved = BYTES_PER_QUERY * m / step / 1e9  # per GPU GB/s
        traffic = ncu_traffic()
        line = {
            "metric": METRIC,
            "value": value,
            "unit": UNIT,
            "n_gpus": world,
            "steps": args.steps,
            "warmup": args.warmup,
            "ms_per_step": 1e3 * step,
            "higher_is_better": True,
            "scaling": "weak",
            "vs_baseline": None,
            "dtype": "f32",
            "data": "synthetic (seeded cfg3 recipe; queries generated on device, Philox)",
            "config": {
                "workload": "cfg3: f32 X N+1=4097, dX=0.5+U[0,1) (seed 0); 2^30 f32 queries U[X0,XN) per GPU",
                "queries_per_gpu": m,
                "global_queries": total,
                "algorithm": "direct (gap 1, X+J staged in smem)",
                "placement": prep.placement(),
                "R": prep.structure.r,
                "h": float(prep.structure.h),
                "index_build_ms": build_ms,
                "l2": "inputs 4 GiB + outputs 4 GiB per GPU >> 126 MB L2; no flush needed",
                "parallelism": f"query shards x{world}, X/J replicated (built locally)",
                "verified": verified,
            },
            "roofline": {
                "bound": "hbm",
                "achieved": achieved,
                "peak": pk["hbm_gbs"],
                "unit": "GB/s",
                "frac": achieved / pk["hbm_gbs"],
                "traffic": (traffic or {}).get("dram_bytes_per_launch"),
                "peak_source": pk["source"],
                "frac_of_spec": achieved / SPEC_HBM_GBS,  # the ~8 TB/s nominal peak the north star cites
                "algorithmic_bytes_per_query": BYTES_PER_QUERY,
            },
            "bsearch": {
                "algorithm": "bitset2 (Alg 3, padded, smem)",
                "value": total / (t_bs / bs_steps),
                "ms_per_step": 1e3 * t_bs / bs_steps,
                "roofline_frac": BYTES_PER_QUERY * m / (t_bs / bs_steps) / 1e9 / pk["hbm_gbs"],
                "direct_speedup": (t_bs / bs_steps) / step,
            },
            "e2e": {
                "value": me * world / t_e2e,
                "unit": UNIT,
                "h2d_bytes_per_step": 4 * me,
                "d2h_bytes_per_step": 4 * me,
                "queries_per_gpu": me,
                "api": "paper_1506_08620_b200.batch_search(LaneConfig(d=65536,'direct'), pinned numpy z, pinned numpy int32 out)",
                "ms_per_step": 1e3 * t_e2e,
                "contract": "reference batch_search guarantee kept: nothing written to out on OutOfDomain "
                            "(host threads check the domain while chunks upload; write-back starts once "
                            "no query is bad, overlapping the remaining uploads)",
                "pageable": {
                    "value": me * world / t_e2e_pg,
                    "ms_per_step": 1e3 * t_e2e_pg,
                    "api": "batch_search on ordinary (pageable) numpy arrays: library pinned staging ring",
                },
                "overlapped": {
                    "value": me * world / t_e2e_ov,
                    "ms_per_step": 1e3 * t_e2e_ov,
                    "api": "batch_search(..., atomic=False): chunk results written back while later chunks upload",
                },
            },
            "gpu_launches": args.steps * prep.launches_per_batch(m),
            "clocks": clocks,
        }
        if configs is not None:
            line["per_config"] = configs
        if not args.no_cpu_baseline and world == 1:  # rank 0 at N=1 only
            from oracle import fs_oracle as orc  # noqa: F401  (cpu_baseline leg only)

            zs = z_cpu
            rate, threads, reps, outc = cpu_reference_rate(p.values, zs, "direct", 3, 1, min_time=10.0)
            line["cpu_baseline"] = {
                "value": rate,
                "unit": UNIT,
                "cores": threads,
                "kind": "port",
                "sample": f"first {CPU_SAMPLE} queries of rank 0's stream, reference direct lane path "
                          f"(batch.py:315-317, restated in oracle/fs_oracle.py), d=65536, {threads} threads, "
                          f"median of {reps} passes",
            }
            line["config"]["cpu_sample_matches_gpu"] = bool(np.array_equal(outc, o_cpu))
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
