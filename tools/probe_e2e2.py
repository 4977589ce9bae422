"""Probe: replicate bench.py's e2e sequence with a per-phase breakdown (dev tool)."""
import time
import numpy as np
import torch
import paper_1511_04348_b200 as tr

n, T = 32768, 4096
dev = torch.device("cuda", 0)
g = torch.Generator(device=dev)
g.manual_seed(1); A = torch.randn((n, n), generator=g, device=dev)
g.manual_seed(2); B = torch.randn((n, n), generator=g, device=dev)
C = torch.empty((n, n), device=dev)
m = tr.homogeneous_machine(1, dtype=np.float32, gpus=[0])
rt = tr.Runtime(m, T)
for _ in range(3):
    rt.multiply(A, B, a_uid="A", b_uid="B", out=C)
rt.close(); del rt
torch.cuda.empty_cache()
t0 = time.perf_counter()
a_host = tr.matrix.pinned_empty((n, n), np.float32)
b_host = tr.matrix.pinned_empty((n, n), np.float32)
a_host[...] = A.cpu().numpy(); b_host[...] = B.cpu().numpy()
print(f"host staging {time.perf_counter()-t0:.2f}s", flush=True)
del A, B, C
torch.cuda.empty_cache()
for i in range(5):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    rt = tr.Runtime(m, T)
    t1 = time.perf_counter()
    out = tr.scheduler._zeros_like_output(rt.operand(a_host, "A"), n, n, pinned=True, zero=False)
    t2 = time.perf_counter()
    c, s = rt.multiply(a_host, b_host, a_uid="A", b_uid="B", c_uid="C", out=out)
    t3 = time.perf_counter()
    rt.close()
    t4 = time.perf_counter()
    del c, out
    t5 = time.perf_counter()
    print(f"step {i}: create {1e3*(t1-t0):.1f} alloc_out {1e3*(t2-t1):.1f} multiply {1e3*(t3-t2):.1f} "
          f"(native {1e3*s.wall_elapsed:.1f}) close {1e3*(t4-t3):.1f} free_out {1e3*(t5-t4):.1f} ms", flush=True)
for i in range(3):
    t0 = time.perf_counter()
    c, s = tr.run(m, a_host, b_host, T)
    t1 = time.perf_counter()
    del c
    print(f"run(): {1e3*(t1-t0):.1f} ms (native {1e3*s.wall_elapsed:.1f})", flush=True)
