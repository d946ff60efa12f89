"""Index-build (setup) time per config, warm, and end-to-end batch_search on
pageable vs pinned host arrays (measurement aid)."""

import json
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1506_08620_b200 as fs  # noqa: E402
from paper_1506_08620_b200 import workloads  # noqa: E402

torch.cuda.set_device(0)
for label, cfg, kw in (("cfg1", "cfg1", {"seed": 0}), ("cfg2_s0", "cfg2", {"seed": 0}), ("cfg2_s1", "cfg2", {"seed": 1}),
                       ("cfg3", "cfg3", {"seed": 0}), ("cfg4", "cfg4", {}), ("cfg5_1048577", "cfg5", {"n1": 1048577})):
    p = workloads.knots(cfg, **kw)
    p.device_values()
    for algo in ("direct", "bitset2"):
        fs.prepare(algo, p)  # warm (module load, allocator)
        torch.cuda.synchronize()
        ts = []
        for _ in range(5):
            t0 = time.perf_counter()
            prep = fs.prepare(algo, p)
            torch.cuda.synchronize()
            ts.append(time.perf_counter() - t0)
            del prep
        t = float(np.median(ts))
        print(json.dumps({"config": label, "algo": algo, "n1": len(p.values), "build_ms": round(1e3 * t, 3),
                          "ns_per_knot": round(1e9 * t / len(p.values), 2)}), flush=True)
    torch.cuda.empty_cache()

p = workloads.knots("cfg3", seed=0)
prep = fs.prepare("direct", p)
cfgl = fs.LaneConfig(65536, "direct", prep)
for m in (1 << 24, 1 << 28):
    z = workloads.queries_host("cfg3", p, m, seed=1)
    for kind in ("pageable", "pinned"):
        if kind == "pinned":
            zt = torch.empty(m, dtype=torch.float32, pin_memory=True)
            zt.copy_(torch.from_numpy(z))
            ot = torch.empty(m, dtype=torch.int32, pin_memory=True)
            zz, oo = zt.numpy(), ot.numpy()
        else:
            zz, oo = z, np.empty(m, dtype=np.int32)
        for atomic in (True, False):
            fs.batch_search(cfgl, zz, oo, atomic=atomic)
            ts = []
            for _ in range(3):
                t0 = time.perf_counter()
                fs.batch_search(cfgl, zz, oo, atomic=atomic)
                ts.append(time.perf_counter() - t0)
            t = float(np.median(ts))
            print(json.dumps({"m": m, "host": kind, "atomic": atomic, "ms": round(1e3 * t, 2),
                              "gqs": round(m / t / 1e9, 2), "pcie_gbs": round(8 * m / t / 1e9, 1)}), flush=True)
