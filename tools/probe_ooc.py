"""Probe: out-of-core product (operands larger than the tile cache) at N=65536.  Dev tool."""
import sys, time
import numpy as np
import torch
import paper_1511_04348_b200 as tr

n, T = int(sys.argv[1]) if len(sys.argv) > 1 else 65536, 4096
t0 = time.perf_counter()
a = tr.matrix.pinned_empty((n, n), np.float32)
b = tr.matrix.pinned_empty((n, n), np.float32)
c = tr.matrix.pinned_empty((n, n), np.float32)
print(f"pinned alloc {time.perf_counter() - t0:.1f} s", flush=True)
g = torch.Generator(device="cuda").manual_seed(1)
rows = 8192
for m in (a, b):
    for r in range(0, n, rows):
        m[r:r + rows] = torch.randn((rows, n), device="cuda", generator=g).cpu().numpy()
print(f"filled {time.perf_counter() - t0:.1f} s", flush=True)
m = tr.homogeneous_machine(1, dtype=np.float32)
flops = 2.0 * n ** 3
cases = [(16, "auto"), (24, "auto"), (24, "auto"), (24, "blocked"), (32, "auto")]
for budget_gb, order in cases:
    rt = tr.Runtime(m, T, hbm_budget_bytes=int(budget_gb * 2**30), trace=(budget_gb == 24))
    rt.set_order(order)
    t1 = time.perf_counter()
    _, s = rt.multiply(a, b, out=c)
    dt = time.perf_counter() - t1
    cs = s.cache
    if s.trace:
        import json
        json.dump(s.trace, open("gpurun_out/trace_ooc24.json", "w"))
    print(f"budget {budget_gb} GiB {order}: {dt*1e3:.0f} ms wall, span {s.span_ms[0]:.0f} ms -> {flops/dt/1e12:.1f} TF/s; "
          f"host fetches {cs.host_fetches} ({cs.bytes_host/1e9:.1f} GB), evictions {cs.evictions}, kernels {s.kernel_ms[0]:.0f} ms",
          flush=True)
    rt.close()
rows_i = np.array([0, 4095, 4096, n // 2 + 7, n - 1]); cols_i = np.array([1, 4097, n // 3, n - 2, n - 1])
from oracle import tilerun_oracle as O
ref = O.c_oracle().gemm(a[rows_i].astype(np.float64), b[:, cols_i].astype(np.float64))
got = c[rows_i][:, cols_i].astype(np.float64)
print("sampled rel err", float(np.linalg.norm(got - ref) / np.linalg.norm(ref)))
