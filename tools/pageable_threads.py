"""End-to-end batch_search on ordinary (pageable) numpy arrays, cfg3, as a
function of the staging thread count (FSG_COPY_THREADS is read per call).
Tuning aid."""

import json
import os
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1506_08620_b200 as fs  # noqa: E402
from paper_1506_08620_b200 import workloads  # noqa: E402

torch.cuda.set_device(0)
p = workloads.knots("cfg3")
m = 1 << 28
z = workloads.queries_host("cfg3", p, m, seed=3)
out = np.empty(m, dtype=np.int32)
cfg = fs.LaneConfig(65536, "direct", fs.prepare("direct", p))
fs.batch_search(cfg, z, out)
for threads in [int(a) for a in (sys.argv[1:] or ["4", "8", "12", "16"])]:
    os.environ["FSG_COPY_THREADS"] = str(threads)
    ts = []
    for _ in range(4):
        t0 = time.perf_counter()
        fs.batch_search(cfg, z, out)
        ts.append(time.perf_counter() - t0)
    t = float(np.median(ts))
    print(json.dumps({"copy_threads": threads, "ms": round(1e3 * t, 1), "gqs": round(m / t / 1e9, 2)}), flush=True)
