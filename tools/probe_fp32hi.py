"""fp32hi (split-bf16x6) vs fp32acc (x3): relative Frobenius error against float64
over K, and the warm cfg2-shaped rate of both (N = 32768, T = 4096)."""
import sys

import numpy as np
import torch

import paper_1511_04348_b200 as tr
from paper_1511_04348_b200.dense import dense_gemm

g = torch.Generator(device="cuda").manual_seed(0)
for k in (256, 4096, 32768, 131072):
    m = n = 1024
    a = torch.randn(m, k, device="cuda", generator=g)
    b = torch.randn(k, n, device="cuda", generator=g)
    ref = a.double() @ b.double()
    row = [f"K={k}"]
    for p in ("fp32acc", "fp32hi", "bf16"):
        c = dense_gemm(a, b, precision=p)
        row.append(f"{p} {float(torch.linalg.norm(c.double() - ref) / torch.linalg.norm(ref)):.2e}")
    print("  ".join(row), flush=True)
    del a, b, ref
n = int(sys.argv[1]) if len(sys.argv) > 1 else 32768
A = torch.randn(n, n, device="cuda", generator=g)
B = torch.randn(n, n, device="cuda", generator=g)
C = torch.empty(n, n, device="cuda")
m = tr.homogeneous_machine(1, dtype=np.float32)
for p in ("fp32acc", "fp32hi"):
    with tr.Runtime(m, 4096, precision=p) as rt:
        for _ in range(2):
            rt.multiply(A, B, a_uid="A", b_uid="B", out=C)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(3):
            _, s = rt.multiply(A, B, a_uid="A", b_uid="B", out=C)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 3
        print(f"{p}: {ms:.1f} ms per N={n} product = {2 * n**3 / ms / 1e9:.1f} TF/s, "
              f"launch {sum(s.kernel_ms.values()) / s.gpu_launches:.2f} ms x {s.gpu_launches}", flush=True)
