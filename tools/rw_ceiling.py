"""HBM ceiling for the stream shapes of the search kernel (tuning aid):
torch copies with the same read:write byte mix as f32->int32 (1:1),
f32->int64 (1:2) and f64->int32 (2:1) searches."""
import json
import torch

torch.cuda.set_device(0)
n = 1 << 30
for src, dst in ((torch.float32, torch.int32), (torch.float32, torch.int64), (torch.float64, torch.int32),
                 (torch.float64, torch.int64)):
    a = torch.rand(n if src == torch.float32 else n // 2, device="cuda").to(src)
    b = torch.empty(a.numel(), device="cuda", dtype=dst)
    for _ in range(3):
        b.copy_(a)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10):
        b.copy_(a)
    e1.record()
    torch.cuda.synchronize()
    t = e0.elapsed_time(e1) / 10 / 1e3
    byt = a.numel() * (a.element_size() + b.element_size())
    print(json.dumps({"read": str(src), "write": str(dst), "gbs": round(byt / t / 1e9, 1)}), flush=True)
    del a, b
