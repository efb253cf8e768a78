"""Host<->device copy ceiling on this box: pinned H2D, D2H, and both at once (the e2e leg's bound)."""
import torch

n = 1 << 28  # 1 GiB of fp32
h_in = torch.empty(n, dtype=torch.float32, pin_memory=True)
h_out = torch.empty(n, dtype=torch.float32, pin_memory=True)
d_a = torch.empty(n, dtype=torch.float32, device="cuda")
d_b = torch.empty(n, dtype=torch.float32, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def timed(fn, reps=5):
    best = 1e9
    for _ in range(reps):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record(torch.cuda.current_stream())
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    return best


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


gb = n * 4 / 1e9
t = timed(lambda: d_a.copy_(h_in, non_blocking=True))
print(f"H2D pinned  {gb / t * 1e3:.1f} GB/s")
t = timed(lambda: h_out.copy_(d_b, non_blocking=True))
print(f"D2H pinned  {gb / t * 1e3:.1f} GB/s")
t = timed(both)
print(f"H2D+D2H concurrent  {gb / t * 1e3:.1f} GB/s each direction")
