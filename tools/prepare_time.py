"""Wall time of prepare("direct") per config (certification, tables and the
layout planners), warm, mean of 3 (tuning aid)."""
import time, sys
sys.path.insert(0, '.')
import torch, paper_1506_08620_b200 as fs
from paper_1506_08620_b200 import workloads
torch.cuda.set_device(0)
for name, kw in (("cfg3", {}), ("cfg2", {}), ("cfg2", {"seed": 1}), ("cfg4", {}), ("cfg5", {"n1": 33}), ("cfg5", {"n1": 1025}), ("cfg5", {"n1": 32769}), ("cfg5", {"n1": 1048577})):
    p = workloads.knots(name, **kw)
    fs.prepare("direct", p); torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(3):
        prep = fs.prepare("direct", p)
    torch.cuda.synchronize()
    print(name, kw, "prepare ms", round((time.perf_counter() - t) / 3 * 1e3, 2), prep.placement().get("sparse_format"), prep.placement()["smem_hot"])
