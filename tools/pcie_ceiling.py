"""PCIe ceilings for the end-to-end leg (tuning aid): pinned host->device and
device->host copies of 4 GiB, alone and concurrently on two streams (CUDA
events around each); the e2e step moves 4 GiB each way."""
import torch

n = 1 << 30  # int32 elements = 4 GiB
h_in = torch.empty(n, dtype=torch.int32, pin_memory=True)
h_out = torch.empty(n, dtype=torch.int32, pin_memory=True)
d_a = torch.empty(n, dtype=torch.int32, device="cuda")
d_b = torch.empty(n, dtype=torch.int32, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def timed(fn, reps=3):
    best = 1e9
    for _ in range(reps):
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        best = min(best, a.elapsed_time(b) / 1e3)
    return best


gb = 4 * n / 1e9
t_h2d = timed(lambda: d_a.copy_(h_in, non_blocking=True))
t_d2h = timed(lambda: h_out.copy_(d_b, non_blocking=True))


def both():
    cur = torch.cuda.current_stream()
    s1.wait_stream(cur)
    s2.wait_stream(cur)
    with torch.cuda.stream(s1):
        d_a.copy_(h_in, non_blocking=True)
    with torch.cuda.stream(s2):
        h_out.copy_(d_b, non_blocking=True)
    cur.wait_stream(s1)
    cur.wait_stream(s2)


t_both = timed(both)
print(f"H2D {gb / t_h2d:.1f} GB/s ({t_h2d * 1e3:.1f} ms), D2H {gb / t_d2h:.1f} GB/s ({t_d2h * 1e3:.1f} ms), "
      f"both concurrently {2 * gb / t_both:.1f} GB/s aggregate ({t_both * 1e3:.1f} ms for 4 GiB each way; "
      f"an e2e ceiling of {n / t_both / 1e9:.2f} G queries/s)")
