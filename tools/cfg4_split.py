"""cfg4 diagnostics: rank-directory (L2, with its hot window), sparse+dense
table, zoned records (mixed slot/rank) and striped rank words on the uniform and the clustered halves of the query
stream separately (tuning aid)."""

import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

import paper_1506_08620_b200 as fs  # noqa: E402
from paper_1506_08620_b200 import batch, workloads  # noqa: E402

torch.cuda.set_device(0)
p = workloads.knots("cfg4")
m = 1 << 27
x0, xn, hi = float(p.values[0]), float(p.values[-1]), workloads.cfg4_dense_top(p)
g = torch.Generator(device="cuda")
g.manual_seed(1)
streams = {
    "uniform": (x0 + torch.rand(m, dtype=torch.float64, device="cuda", generator=g) * (xn - x0)).float(),
    "clustered": (x0 + torch.rand(m, dtype=torch.float64, device="cuda", generator=g) * (hi - x0)).float(),
}
for k, z in streams.items():
    streams[k] = torch.where(z >= xn, torch.nextafter(torch.tensor(xn, device="cuda").float(),
                                                      torch.tensor(0.0, device="cuda")), z)
out = torch.empty(m, dtype=torch.int32, device="cuda")
st = fs.new_status()
only = sys.argv[1:]  # optional: variant stream (profiling a single case)
for variant in ("rank-l2", "sparse-dense", "zoned", "zoned-rank"):
    if only and variant != only[0]:
        continue
    batch.SPARSE_MAX_DENSE_KNOT_FRACTION = 1.0 if variant == "sparse-dense" else 0.25
    batch.ZONED = variant.startswith("zoned")
    batch.ZONED_RANK_MAX_XREAD_PPM = 150_000 if variant == "zoned-rank" else 0  # striped rank words / mixed records
    prep = fs.prepare("direct", p)
    for k, z in streams.items():
        if only and k != only[1]:
            continue
        for _ in range(3):
            prep.launch(z, out, st)
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(10):
            prep.launch(z, out, st)
        b.record()
        torch.cuda.synchronize()
        t = a.elapsed_time(b) / 10 / 1e3
        print(json.dumps({"variant": variant, "stream": k, "gqs": round(m / t / 1e9, 1),
                          "placement": prep.placement(), "ndense": prep.plan.sparse_ndense,
                          "shift": prep.plan.sparse_shift}), flush=True)
