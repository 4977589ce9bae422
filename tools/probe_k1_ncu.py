"""Probe for ncu: warm cfg2 products (N=32768, T=4096, inputs in HBM) in the
FP32-accurate mode then in bf16 -- 2 products (32 grouped K1 launches) each.
`ncu -k regex:tile_gemm -s 20 -c 1` captures an fp32acc launch, `-s 52 -c 1` a bf16 one.
Optional second argument: a comma list of precisions to run instead (e.g. fp32hi)."""
import sys
import numpy as np
import torch
import paper_1511_04348_b200 as tr

n = int(sys.argv[1]) if len(sys.argv) > 1 else 32768
T = 4096
g = torch.Generator(device="cuda")
A = torch.randn((n, n), generator=g.manual_seed(1), device="cuda")
B = torch.randn((n, n), generator=g.manual_seed(2), device="cuda")
C = torch.empty((n, n), device="cuda")
m = tr.homogeneous_machine(1, dtype=np.float32)
precs = sys.argv[2].split(",") if len(sys.argv) > 2 else ["fp32acc", "bf16"]
for prec in precs:
    with tr.Runtime(m, T, precision=prec) as rt:
        for _ in range(2):
            _, s = rt.multiply(A, B, a_uid="A", b_uid="B", out=C)
        print(prec, s.gpu_launches, sum(s.kernel_ms.values()) / max(1, s.gpu_launches), "ms/launch", flush=True)
