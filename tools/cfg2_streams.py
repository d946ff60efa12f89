"""cfg2 seeds 0 and 1: the direct search on the config's stream (1% of the
queries exact knots) vs a uniform-only stream of the same size, to separate
the cost of X reads through L2 (exact-knot queries) from the record decode
(measurement aid; profiles/r02/records19_rejected.txt)."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch, json
import paper_1506_08620_b200 as fs
from paper_1506_08620_b200 import workloads
torch.cuda.set_device(0)
for seed in (0, 1):
    p = workloads.knots("cfg2", seed=seed)
    prep = fs.prepare("direct", p)
    m = 100_000_000
    zk = workloads.queries_device("cfg2", p, m, seed=1)
    g = torch.Generator(device="cuda"); g.manual_seed(5)
    zu = (float(p.values[0]) + torch.rand(m, dtype=torch.float64, device="cuda", generator=g) * float(p.values[-1] - p.values[0]))
    zu = torch.clamp(zu, max=float(p.values[-2]))
    out = torch.empty(m, dtype=torch.int32, device="cuda"); st = fs.new_status()
    for name, z in (("with 1% knots", zk), ("uniform only", zu)):
        for _ in range(3): prep.launch(z, out, st)
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(20): prep.launch(z, out, st)
        b.record(); torch.cuda.synchronize()
        t = a.elapsed_time(b) / 20 / 1e3
        print(json.dumps({"seed": seed, "stream": name, "gqs": round(m / t / 1e9, 1), "fmt": prep.placement()["sparse_format"], "smem_x": prep.placement()["smem_x"]}))
