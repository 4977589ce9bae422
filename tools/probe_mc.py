"""Probe: grouped K1 launches of the cfg4 shape (4 tasks, K = 131072, warm) with
CTA pairs vs TMA-multicast clusters of two pairs (tr_set_gemm_multicast)."""
import numpy as np
import torch
import paper_1511_04348_b200 as tr
from paper_1511_04348_b200 import _native as N

K, T = 131072, 4096
g = torch.Generator(device="cuda")
A = torch.randn((T, K), generator=g.manual_seed(1), device="cuda")
B = torch.randn((K, 4 * T), generator=g.manual_seed(2), device="cuda")
C = torch.empty((T, 4 * T), device="cuda")
ref = None
for rnd in range(2):
    for mc in (0, 1):
        N.call("tr_set_gemm_multicast", mc)
        for prec in ("fp32acc", "bf16"):
            with tr.Runtime(tr.homogeneous_machine(1, dtype=np.float32), T, precision=prec) as rt:
                rt.multiply(A, B, a_uid="A", b_uid="B", out=C)
                ms = []
                for _ in range(3):
                    _, s = rt.multiply(A, B, a_uid="A", b_uid="B", out=C)
                    ms.append(sum(s.kernel_ms.values()))
            rows = torch.arange(0, T, 97, device="cuda")
            r = A[rows].double() @ B.double()
            err = float(torch.linalg.norm(C[rows].double() - r) / torch.linalg.norm(r))
            print(f"round {rnd} mc={mc} {prec}: ms {[round(x, 1) for x in ms]} -> "
                  f"{2.0 * T * 4 * T * K / (min(ms) / 1e3) / 1e12:.0f} TF/s, err {err:.2e}", flush=True)
N.call("tr_set_gemm_multicast", 0)
