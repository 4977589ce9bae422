"""Probe: how does the tcgen05 fp32 accumulator round?  (dev tool, not a test)"""
import torch
from paper_1511_04348_b200 import dense_gemm

torch.manual_seed(0)
def split(x):
    hi = x.to(torch.bfloat16).double()
    lo = (x.double() - hi).float().to(torch.bfloat16).double()
    return hi, lo

for K in (256, 1024, 4096, 16384, 32768):
    M = N = 512
    a = torch.randn(M, K, dtype=torch.float32, device="cuda")
    b = torch.randn(K, N, dtype=torch.float32, device="cuda")
    ref = a.double() @ b.double()
    c = dense_gemm(a, b, precision="fp32acc")
    ah, al = split(a); bh, bl = split(b)
    ideal = ah @ bh + ah @ bl + al @ bh
    e = (c.double() - ref)
    bias = float((e * torch.sign(ref)).mean() / ref.abs().mean())
    print(f"K={K:6d} gpu_err={float(e.norm()/ref.norm()):.3e} split_only={float((ideal-ref).norm()/ref.norm()):.3e} "
          f"signed_bias={bias:+.3e}", flush=True)
    cb = dense_gemm(a, b, precision="bf16")
    print(f"          bf16_err={float((cb.double()-ref).norm()/ref.norm()):.3e}", flush=True)

# deterministic: ones @ (1+2^-7) for K = 2^18: exact sum 264192
K = 1 << 18
a = torch.ones(128, K, device="cuda")
b = torch.full((K, 256), 1.0078125, device="cuda")
c = dense_gemm(a, b, precision="bf16")
print("ones@(1+2^-7) K=2^18 -> gpu", float(c[0, 0]), "exact 264192.0; fp32 RNE sequential ->",
      float(torch.cumsum(torch.full((K,), 1.0078125, dtype=torch.float32), 0)[-1]))
# sum of 16 products then accumulate: emulate RZ vs RNE at 16-chunk granularity
import numpy as np
acc_rne = np.float32(0); acc_rz = 0.0
for i in range(K // 16):
    acc_rne = np.float32(acc_rne + np.float32(16 * 1.0078125))
print("16-chunk RNE emulation ->", float(acc_rne))
