"""Per-launch cost of small batches: eager launches vs CUDA-graph replay,
smem-staged vs L2 tables (tuning aid)."""

import json
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

import paper_1506_08620_b200 as fs  # noqa: E402
from paper_1506_08620_b200 import workloads  # noqa: E402

torch.cuda.set_device(0)
p = workloads.knots("cfg1", seed=0)
for m in (10_000, 100_000, 1_000_000, 10_000_000):
    z = workloads.queries_device("cfg1", p, m, seed=1)
    out = torch.empty(m, dtype=torch.int32, device="cuda")
    fb = fs.new_status()
    for algo in ("direct", "direct-cache", "bitset2"):
        prep = fs.prepare(algo, p)
        for policy in (0, 1):
            prep.plan.smem_policy = policy
            for _ in range(5):
                prep.launch(z, out, fb)
            torch.cuda.synchronize()
            n = 200
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            t0 = time.perf_counter()
            a.record()
            for _ in range(n):
                prep.launch(z, out, fb)
            b.record()
            cpu = (time.perf_counter() - t0) / n
            torch.cuda.synchronize()
            eager = a.elapsed_time(b) / n * 1e3
            g = torch.cuda.CUDAGraph()
            s = torch.cuda.Stream()
            s.wait_stream(torch.cuda.current_stream())
            with torch.cuda.stream(s):
                with torch.cuda.graph(g):
                    for _ in range(10):
                        prep.launch(z, out, fb)
            torch.cuda.current_stream().wait_stream(s)
            g.replay()
            torch.cuda.synchronize()
            a.record()
            for _ in range(n // 10):
                g.replay()
            b.record()
            torch.cuda.synchronize()
            graph = a.elapsed_time(b) / n * 1e3
            print(json.dumps({"m": m, "algo": algo, "policy": policy, "cpu_us": round(cpu * 1e6, 2),
                              "eager_us": round(eager, 2), "graph_us": round(graph, 2),
                              "graph_gqs": round(m / graph / 1e3, 1), "eager_gqs": round(m / eager / 1e3, 1)}),
                  flush=True)
