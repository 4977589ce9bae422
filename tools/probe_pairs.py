"""Probe: warm cfg2 product rate vs CTA-pair variant and in-flight tasks.  Dev tool."""
import numpy as np
import torch
import paper_1511_04348_b200 as tr
from paper_1511_04348_b200.dense import set_gemm_pairs

n, T = 32768, 4096
g = torch.Generator(device="cuda").manual_seed(1)
A = torch.randn((n, n), device="cuda", generator=g); B = torch.randn((n, n), device="cuda", generator=g)
C = torch.empty((n, n), device="cuda")
for prec in ("fp32acc", "bf16"):
    rt = tr.Runtime(tr.homogeneous_machine(1, dtype=np.float32), T, precision=prec)
    for pairs in (0, 1):
        set_gemm_pairs(bool(pairs))
        for infl in (1, 2, 3, 4):
            rt.set_inflight(infl)
            for _ in range(2):
                rt.multiply(A, B, a_uid="A", b_uid="B", out=C)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(3):
                rt.multiply(A, B, a_uid="A", b_uid="B", out=C)
            e1.record(); torch.cuda.synchronize()
            t = e0.elapsed_time(e1) / 3 / 1e3
            print(f"{prec:8s} pairs={pairs} inflight={infl}: {2 * n**3 / t / 1e12:7.1f} TF/s", flush=True)
    rt.close()
