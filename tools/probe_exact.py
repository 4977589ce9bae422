"""Throughput of precision "exact" (KX, CUDA cores, k-ascending rounded mul+add)
against fp32acc on the same dense product; and the scheduled run() in exact mode."""
import time

import numpy as np
import torch

from paper_1511_04348_b200 import homogeneous_machine, run
from paper_1511_04348_b200.dense import dense_gemm

for dt in (torch.float64, torch.float32):
    n = 4096
    a = torch.randn(n, n, dtype=dt, device="cuda")
    b = torch.randn(n, n, dtype=dt, device="cuda")
    for prec in ("exact", "fp32acc"):
        dense_gemm(a, b, precision=prec)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(3):
            dense_gemm(a, b, precision=prec)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 3
        print(f"dense {dt} {prec}: {ms:.2f} ms  {2 * n**3 / ms / 1e9:.1f} TF/s")
rng = np.random.default_rng(0)
a, b = rng.standard_normal((8192, 8192)), rng.standard_normal((8192, 8192))
for prec in ("exact", "fp32acc"):
    run(homogeneous_machine(1), a[:1024, :1024], b[:1024, :1024], 1024, precision=prec)
    t = time.perf_counter()
    c, s = run(homogeneous_machine(1), a, b, 2048, precision=prec)
    w = time.perf_counter() - t
    print(f"run f64 8192 tile 2048 {prec}: {w * 1e3:.0f} ms wall, kernel {sum(s.kernel_ms.values()):.1f} ms, "
          f"{2 * 8192**3 / w / 1e12:.2f} TF/s e2e")
