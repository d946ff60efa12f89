"""cfg1 (10^6 f32 queries) under bench.py's per-config timing (L2 flushed
before each launch, CUDA events around the launch): the search kernel vs a
copy of the same 4 MB stream into a 4 MB output, and vs the same search with
warm L2 (measurement aid)."""

import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

import paper_1506_08620_b200 as fs  # noqa: E402
from paper_1506_08620_b200 import workloads  # noqa: E402

torch.cuda.set_device(0)
p = workloads.knots("cfg1", seed=0)
m = 1_000_000
z = workloads.queries_device("cfg1", p, m, seed=11)
out = torch.empty(m, dtype=torch.int32, device="cuda")
zi = z.view(torch.int32)
fb = fs.new_status()
flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")


def timed(fn, n=50, cold=True):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    pairs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(n)]
    for a, b in pairs:
        if cold:
            flush.zero_()
        a.record()
        fn()
        b.record()
    torch.cuda.synchronize()
    return sorted(a.elapsed_time(b) * 1e3 for a, b in pairs)[n // 2]


for name in ("direct", "bitset2"):
    prep = fs.prepare(name, p)
    for cold in (True, False):
        us = timed(lambda: prep.launch(z, out, fb), cold=cold)
        print(json.dumps({"kernel": name, "l2": "flushed" if cold else "warm", "us": round(us, 2),
                          "gqs": round(m / us / 1e3, 1), "placement": prep.placement()}))
for cold in (True, False):
    us = timed(lambda: out.copy_(zi), cold=cold)
    print(json.dumps({"kernel": "torch copy 4 MB -> 4 MB", "l2": "flushed" if cold else "warm", "us": round(us, 2),
                      "gqs_equiv": round(m / us / 1e3, 1)}))
