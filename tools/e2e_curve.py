"""End-to-end batch_search throughput on host arrays vs batch size, 1 MB to
4 GiB of float32 queries (cfg3 partition), pageable numpy arrays (what a
drop-in caller passes) beside pinned ones, atomic contract on.  Wall-clock
per call (the call is synchronous), median of the repetitions; the library's
persistent host pool and pinned staging ring are warm (measurement aid)."""

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
p = workloads.knots("cfg3", seed=0)
prep = fs.prepare("direct", p)
cfg = fs.LaneConfig(65536, "direct", prep)
top = 1 << 30
rng = np.random.default_rng(1)
z_all = rng.uniform(float(p.x0), float(p.xn), size=top).astype(np.float32)
z_all[z_all >= p.values[-1]] = np.nextafter(p.values[-1], np.float32(0))
out_all = np.empty(top, dtype=np.int32)
zp = torch.empty(top, dtype=torch.float32, pin_memory=True)
zp.numpy()[:] = z_all
op = torch.empty(top, dtype=torch.int32, pin_memory=True)
for lg in range(18, 31, 2):  # 2^18 queries = 1 MB ... 2^30 = 4 GiB
    m = 1 << lg
    for kind in ("pageable", "pinned"):
        zz, oo = (z_all[:m], out_all[:m]) if kind == "pageable" else (zp.numpy()[:m], op.numpy()[:m])
        fs.batch_search(cfg, zz, oo)  # warm
        reps = 20 if m <= 1 << 24 else 5
        ts = []
        for _ in range(reps):
            t0 = time.perf_counter()
            fs.batch_search(cfg, zz, oo)
            ts.append(time.perf_counter() - t0)
        t = float(np.median(ts))
        print(json.dumps({"queries": m, "mbytes_in": 4 * m >> 20, "host": kind, "ms": round(1e3 * t, 3),
                          "gqs": round(m / t / 1e9, 3), "pcie_gbs_both_ways": round(8 * m / t / 1e9, 1)}),
              flush=True)
assert np.array_equal(out_all[: 1 << 20], fs.run_batch(prep, z_all[: 1 << 20]).astype(np.int32))
