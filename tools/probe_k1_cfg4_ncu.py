"""Probe for ncu: ONE grouped K1 launch of the cfg4 headline's shape -- 4 tasks
(4096 x 4096 outputs of one row block) over K = 131072 (32 k-steps), warm
(operand tiles resident), fp32-accurate.  A = 4096 x 131072, B = 131072 x 16384
on the device (20 GiB in all instead of cfg4's 206 GB, so ncu's kernel replay
can save and restore device memory).  3 products = 3 launches:
`ncu -k regex:tile_gemm -s 2 -c 1` captures the third."""
import sys
import numpy as np
import torch
import paper_1511_04348_b200 as tr

prec = sys.argv[1] if len(sys.argv) > 1 else "fp32acc"
K, T = 131072, 4096
g = torch.Generator(device="cuda")
A = torch.randn((T, K), generator=g.manual_seed(1), device="cuda")
B = torch.randn((K, 4 * T), generator=g.manual_seed(2), device="cuda")
C = torch.empty((T, 4 * T), device="cuda")
with tr.Runtime(tr.homogeneous_machine(1, dtype=np.float32), T, precision=prec) as rt:
    for i in range(3):
        _, s = rt.multiply(A, B, a_uid="A", b_uid="B", out=C)
        print(prec, "launches", s.gpu_launches, "kernel ms", round(sum(s.kernel_ms.values()), 3),
              "TF/s", round(2.0 * T * 4 * T * K / (sum(s.kernel_ms.values()) / 1e3) / 1e12, 1), flush=True)
