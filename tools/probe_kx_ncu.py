"""Probe for ncu: one KX (precision "exact") launch, 4096^2 x 4096 float64 (argv[1] = f32 for float32)."""
import sys

import torch

from paper_1511_04348_b200.dense import dense_gemm

dt = torch.float32 if len(sys.argv) > 1 and sys.argv[1] == "f32" else torch.float64
a = torch.randn(4096, 4096, dtype=dt, device="cuda")
b = torch.randn(4096, 4096, dtype=dt, device="cuda")
for _ in range(2):
    dense_gemm(a, b, precision="exact")
torch.cuda.synchronize()
