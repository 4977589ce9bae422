"""Probe: kernel variant (CTA pairs vs single) on the warm product, and task
order x in-flight depth on the cold (host-buffer) product.  Dev tool."""
import time
import numpy as np
import torch
import paper_1511_04348_b200 as tr
from paper_1511_04348_b200.dense import set_gemm_pairs

n, T = 32768, 4096
dev = torch.device("cuda", 0)
g = torch.Generator(device=dev)
g.manual_seed(1); A = torch.randn((n, n), generator=g, device=dev)
g.manual_seed(2); B = torch.randn((n, n), generator=g, device=dev)
C = torch.empty((n, n), device=dev)
m = tr.homogeneous_machine(1, dtype=np.float32, gpus=[0])
rows = torch.tensor([0, 4095, 4096, 20000, 32767], device=dev)
ref = (A[rows].double() @ B.double())
set_gemm_pairs(False)
a_host = tr.matrix.pinned_empty((n, n), np.float32); a_host[...] = A.cpu().numpy()
b_host = tr.matrix.pinned_empty((n, n), np.float32); b_host[...] = B.cpu().numpy()
del A, B, C
torch.cuda.empty_cache()
for order in ("row-major", "banded", "shells"):
    for fa, inflight in ((True, 2), (True, 3)):
        rt = tr.Runtime(m, T, fetch_ahead=fa)
        rt.set_order(order); rt.set_inflight(inflight)
        ts = []
        for _ in range(3):
            t0 = time.perf_counter(); c, s = rt.multiply(a_host, b_host); ts.append(time.perf_counter() - t0); del c
        print(f"order={order} fetch_ahead={fa} inflight={inflight}: cold multiply {1e3*np.median(ts):.1f} ms "
              f"(span {s.span_ms[0]:.1f}) -> {2*n**3/np.median(ts)/1e12:.1f} TF/s", flush=True)
        rt.close()
ts = []
for _ in range(4):
    t0 = time.perf_counter(); c, s = tr.run(m, a_host, b_host, T); ts.append(time.perf_counter() - t0); del c
print("run():", [round(1e3 * t, 1) for t in ts], flush=True)
