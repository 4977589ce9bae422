"""Probe: cold cfg2 run() step times in isolation vs after warm device sessions
(the bench's order).  Dev tool."""
import time
import numpy as np
import torch
import paper_1511_04348_b200 as tr

n, T = 32768, 4096
machine = tr.homogeneous_machine(1, dtype=np.float32)
a = tr.matrix.pinned_empty((n, n), np.float32)
b = tr.matrix.pinned_empty((n, n), np.float32)
g = torch.Generator(device="cuda").manual_seed(1)
for m in (a, b):
    for r in range(0, n, 4096):
        m[r:r + 4096] = torch.randn((4096, n), device="cuda", generator=g).cpu().numpy()


def steps(tag, k=4):
    out = []
    c = None
    for _ in range(k):
        c = None
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t0 = time.perf_counter()
        e0.record()
        c, s = tr.run(machine, a, b, T)
        e1.record()
        torch.cuda.synchronize()
        out.append((round(e0.elapsed_time(e1), 1), round((time.perf_counter() - t0) * 1e3, 1), round(s.span_ms[0], 1)))
    print(tag, out, flush=True)


steps("isolated")
A = torch.from_numpy(a).cuda()
B = torch.from_numpy(b).cuda()
C = torch.empty_like(A)
for prec in ("fp32acc", "bf16"):
    with tr.Runtime(machine, T, precision=prec) as rt:
        for _ in range(4):
            rt.multiply(A, B, a_uid="A", b_uid="B", out=C)
steps("after warm sessions (torch cache held)")
del A, B, C
tr.release_cached_memory()
torch.cuda.empty_cache()
steps("after release")
