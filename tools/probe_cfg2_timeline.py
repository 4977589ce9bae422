"""Probe: CUPTI kernel timeline of warm cfg2 products (N=32768, T=4096) through
Runtime.multiply (torch.profiler).  Dev tool."""
import sys
import numpy as np
import torch
import paper_1511_04348_b200 as tr
from torch.profiler import ProfilerActivity, profile

n, T = 32768, 4096
g = torch.Generator(device="cuda").manual_seed(1)
A = torch.randn(n, n, device="cuda", generator=g)
B = torch.randn(n, n, device="cuda", generator=g)
C = torch.empty(n, n, device="cuda")
rt = tr.Runtime(tr.homogeneous_machine(1, dtype=np.float32), T)
if len(sys.argv) > 1:
    rt.set_inflight(int(sys.argv[1]))
for _ in range(3):
    rt.multiply(A, B, a_uid="A", b_uid="B", out=C)
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    for _ in range(2):
        _, s = rt.multiply(A, B, a_uid="A", b_uid="B", out=C)
    torch.cuda.synchronize()
print("span_ms", s.span_ms, "launches", s.gpu_launches)
prof.export_chrome_trace("gpurun_out/cfg2_trace.json")
