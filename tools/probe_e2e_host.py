"""Probe: host-side phases of the one-shot run() (event time vs native wall).  Dev tool."""
import gc, time
import numpy as np
import torch
import paper_1511_04348_b200 as tr
from paper_1511_04348_b200 import scheduler as S

n, T = 32768, 4096
a = tr.matrix.pinned_empty((n, n), np.float32); b = tr.matrix.pinned_empty((n, n), np.float32)
a[...] = 1.0; b[...] = 1.0
m = tr.homogeneous_machine(1, dtype=np.float32)
orig_alloc = S._zeros_like_output
log = {}
def timed_alloc(*x, **k):
    t0 = time.perf_counter(); r = orig_alloc(*x, **k); log["alloc"] = 1e3 * (time.perf_counter() - t0); return r
S._zeros_like_output = timed_alloc
gc_t = []
gc.callbacks.append(lambda phase, info: gc_t.append((phase, time.perf_counter(), info.get("generation"))))
c = None
for i in range(8):
    c = None
    gc_t.clear()
    t0 = time.perf_counter()
    rt = tr.Runtime(m, T)
    t1 = time.perf_counter()
    c, s = rt.multiply(a, b, a_uid="A", b_uid="B", c_uid="C")
    t2 = time.perf_counter()
    rt.close()
    t3 = time.perf_counter()
    gcs = [(p, g) for p, _, g in gc_t]
    print(f"{i}: create {1e3*(t1-t0):6.1f}  multiply {1e3*(t2-t1):6.1f} (native {1e3*s.wall_elapsed:6.1f}, alloc {log['alloc']:5.1f})"
          f"  close {1e3*(t3-t2):5.1f}  gc {gcs}", flush=True)
