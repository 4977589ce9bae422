"""Probe: H2D bandwidth with 1, 2, 4 concurrent copy streams, contiguous and
2D-pitched (4096 x 4096 fp32 blocks out of a 32768-wide host matrix).  Dev tool."""
import ctypes, time
import torch

cudart = ctypes.CDLL("libcudart.so.12") if False else None
n = 1 << 30
hs = [torch.empty(n // 4, dtype=torch.float32, pin_memory=True) for _ in range(4)]
ds = [torch.empty(n // 4, dtype=torch.float32, device="cuda") for _ in range(4)]
ss = [torch.cuda.Stream() for _ in range(4)]

def timed(fn, reps=3):
    fn(); torch.cuda.synchronize(); t0 = time.perf_counter()
    for _ in range(reps): fn()
    torch.cuda.synchronize(); return (time.perf_counter() - t0) / reps

for k in (1, 2, 4):
    def go():
        for i in range(k):
            with torch.cuda.stream(ss[i]):
                ds[i].copy_(hs[i], non_blocking=True)
    t = timed(go)
    print(f"contiguous H2D, {k} streams: {k * n / t / 1e9:.1f} GB/s", flush=True)

# pitched: 4096 x 4096 blocks out of an 8192-wide pinned host matrix (rows of 16 KB at a 32 KB pitch)
H = torch.empty((8192, 8192), dtype=torch.float32, pin_memory=True)
D = [torch.empty((4096, 4096), dtype=torch.float32, device="cuda") for _ in range(4)]
blocks = [H[r:r + 4096, c:c + 4096] for r in (0, 4096) for c in (0, 4096)]
for k in (1, 2, 4):
    def go():
        for i, b in enumerate(blocks):
            with torch.cuda.stream(ss[i % k]):
                D[i].copy_(b, non_blocking=True)
    t = timed(go)
    print(f"pitched 4096^2 blocks, {k} streams: {4 * 64 * 2**20 / t / 1e9:.1f} GB/s", flush=True)
