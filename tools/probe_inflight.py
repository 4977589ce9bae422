"""Probe: warm cfg2 product time vs launches in flight per device.  Dev tool."""
import numpy as np
import torch
import paper_1511_04348_b200 as tr

n, T = 32768, 4096
g = torch.Generator(device="cuda").manual_seed(1)
A = torch.randn(n, n, device="cuda", generator=g)
B = torch.randn(n, n, device="cuda", generator=g)
C = torch.empty(n, n, device="cuda")
rt = tr.Runtime(tr.homogeneous_machine(1, dtype=np.float32), T)
for _ in range(3):
    rt.multiply(A, B, a_uid="A", b_uid="B", out=C)
for rep in range(2):
    for inflight in (1, 2, 1, 2):
        rt.set_inflight(inflight)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(3):
            _, s = rt.multiply(A, B, a_uid="A", b_uid="B", out=C)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 3
        print(f"inflight={inflight} {ms:8.2f} ms/product  {2 * n ** 3 / ms / 1e9:6.1f} TF/s  launches={s.gpu_launches}", flush=True)
