"""Probe: pinned H2D / D2H bandwidth alone and concurrently (dev tool)."""
import torch, time
n = 1 << 30  # 1 GiB per buffer (float32 x 256M)
h1 = torch.empty(n // 4, dtype=torch.float32, pin_memory=True)
h2 = torch.empty(n // 4, dtype=torch.float32, pin_memory=True)
d1 = torch.empty(n // 4, dtype=torch.float32, device="cuda")
d2 = torch.empty(n // 4, dtype=torch.float32, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
def timed(fn, reps=4):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    for _ in range(reps): fn()
    torch.cuda.synchronize(); return (time.perf_counter() - t0) / reps
h2d = timed(lambda: d1.copy_(h1, non_blocking=True))
d2h = timed(lambda: h2.copy_(d2, non_blocking=True))
def both():
    with torch.cuda.stream(s1): d1.copy_(h1, non_blocking=True)
    with torch.cuda.stream(s2): h2.copy_(d2, non_blocking=True)
bi = timed(both)
print(f"H2D alone {n/h2d/1e9:.1f} GB/s, D2H alone {n/d2h/1e9:.1f} GB/s, concurrent: {2*n/bi/1e9:.1f} GB/s total ({n/bi/1e9:.1f} each)")
