"""Probe: where does the end-to-end (host-buffer) product spend its time? (dev tool)"""
import time
import numpy as np
import torch
import paper_1511_04348_b200 as tr

n, T = 32768, 4096
a = tr.matrix.pinned_empty((n, n), np.float32)
b = tr.matrix.pinned_empty((n, n), np.float32)
g = torch.Generator(device="cuda").manual_seed(1)
a[...] = torch.randn((n, n), device="cuda", generator=g).cpu().numpy()
b[...] = torch.randn((n, n), device="cuda", generator=g).cpu().numpy()
ta = torch.from_numpy(a)
for i in range(2):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    d = ta.to("cuda", non_blocking=True); torch.cuda.synchronize()
    print(f"torch H2D 4 GiB pinned: {4 * 2**30 / (time.perf_counter() - t0) / 1e9:.1f} GB/s", flush=True)
    t0 = time.perf_counter(); h = d.cpu(); print(f"torch D2H (pageable dst) {4*2**30/(time.perf_counter()-t0)/1e9:.1f} GB/s")
    del d, h
m = tr.homogeneous_machine(1, dtype=np.float32)
for i in range(3):
    t0 = time.perf_counter()
    rt = tr.Runtime(m, T)
    t1 = time.perf_counter()
    c, s = rt.multiply(a, b, a_uid="A", b_uid="B", c_uid="C")
    t2 = time.perf_counter()
    rt.close()
    t3 = time.perf_counter()
    print(f"run {i}: create {1e3*(t1-t0):.1f} ms, multiply {1e3*(t2-t1):.1f} ms (native wall {1e3*s.wall_elapsed:.1f}, "
          f"span {s.span_ms[0]:.1f}, kernels {s.kernel_ms[0]:.1f}), close {1e3*(t3-t2):.1f} ms", flush=True)
    del c
rt = tr.Runtime(m, T)
for i in range(3):
    t1 = time.perf_counter()
    c, s = rt.multiply(a, b)  # fresh uids: cold tiles on a persistent session
    t2 = time.perf_counter()
    print(f"persistent-session cold multiply {i}: {1e3*(t2-t1):.1f} ms (span {s.span_ms[0]:.1f}, host {s.cache.host_fetches} tiles)", flush=True)
    del c
for inflight in (1, 2, 4):
    rt.set_inflight(inflight)
    t1 = time.perf_counter(); c, s = rt.multiply(a, b); t2 = time.perf_counter()
    print(f"inflight={inflight}: cold multiply {1e3*(t2-t1):.1f} ms", flush=True)
    del c
