"""Probe for ncu: cuBLAS bf16 GEMM at cfg2 shape (N = 32768), three launches (the third is captured)."""
import torch
n = 32768
A = torch.randn(n, n, device="cuda").bfloat16()
B = torch.randn(n, n, device="cuda").bfloat16()
for _ in range(3):
    C = torch.matmul(A, B)
torch.cuda.synchronize()
