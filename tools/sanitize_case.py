"""Small end-to-end exercise of every kernel for compute-sanitizer runs."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np
import torch

import paper_1506_08620_b200 as fs
from oracle import fs_oracle as orc
from paper_1506_08620_b200 import persist, workloads

torch.cuda.set_device(0)
for prec, size in (("single", 4097), ("double", 1025), ("single", 65537), ("double", 33)):
    p = fs.gen_uniform_gap_partition(size, 0.5, 1.5, seed=1, precision=prec)
    z = orc.random_queries(p.values, 10_007, seed=2)
    want = orc.rank_oracle(p.values, z)
    for algo in fs.ALGORITHMS:
        prep = fs.prepare(algo, p)
        for policy in (0, 1):
            prep.plan.smem_policy = policy
            assert np.array_equal(fs.run_batch(prep, z), want), (algo, prep, policy)
        zt = torch.from_numpy(z).cuda()
        out = torch.empty(len(z) - 1, dtype=torch.int32, device="cuda")
        fs.batch_search(fs.LaneConfig(1, algo, prep), zt[1:], out)
        assert np.array_equal(out.cpu().numpy(), want[1:])
    bad = z.copy(); bad[5] = np.nan
    try:
        fs.run_batch(fs.prepare("direct", p), bad)
        raise SystemExit("expected OutOfDomain")
    except fs.OutOfDomain as e:
        assert e.position == 5
p = workloads.knots("cfg4")
z = workloads.queries_host("cfg4", p, 100_003, seed=1)
assert np.array_equal(fs.run_batch(fs.prepare("direct", p), z), orc.rank_oracle(p.values, z))
assert np.array_equal(fs.run_batch(fs.prepare("bitset2", p), z), orc.rank_oracle(p.values, z))
t = torch.randint(0, 255, (100_003,), dtype=torch.uint8, device="cuda")
persist.device_crc32(t)
print("sanitize case ok")
