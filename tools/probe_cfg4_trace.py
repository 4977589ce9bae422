"""Probe: device timeline of one cold cfg4 product (N=131072 from pinned host,
B aliasing A as in bench.py) -- GEMM / H2D / convert / D2H busy per 0.5 s bin,
first launch, last H2D.  Dev tool."""
import sys
import numpy as np
import torch
import paper_1511_04348_b200 as tr

n = int(sys.argv[1]) if len(sys.argv) > 1 else 131072
T = 4096
torch._C._host_emptyCache()
a = tr.matrix.pinned_empty((n, n), np.float32)
c = tr.matrix.pinned_empty((n, n), np.float32)
g = torch.Generator(device="cuda").manual_seed(4)
at = torch.from_numpy(a)
for r in range(0, n, 4096):
    at[r:r + 4096].copy_(torch.randn((min(4096, n - r), n), device="cuda", generator=g))
torch.cuda.synchronize()
m = tr.homogeneous_machine(1, dtype=np.float32)
with tr.Runtime(m, T) as rt:  # warm-up (pools)
    rt.multiply(a, a, a_uid="A", b_uid="B", c_uid="C", out=c)
with tr.Runtime(m, T, trace=True) as rt:
    _, s = rt.multiply(a, a, a_uid="A", b_uid="B", c_uid="C", out=c)
ev = s.trace
span = max(e["end_ms"] for e in ev)
print(f"span {span:.0f} ms, wall {s.wall_elapsed * 1e3:.0f} ms, launches {s.gpu_launches}")
kinds = ("gemm", "h2d", "convert", "d2h", "peer")
binw = 500.0
nb = int(span // binw) + 1
busy = {k: np.zeros(nb) for k in kinds}
for e in ev:
    t0, t1 = e["start_ms"], e["end_ms"]
    b = int(t0 // binw)
    while t0 < t1 and b < nb:
        be = (b + 1) * binw
        busy[e["kind"]][b] += min(t1, be) - t0
        t0 = be
        b += 1
first_gemm = min(e["start_ms"] for e in ev if e["kind"] == "gemm")
last_h2d = max(e["end_ms"] for e in ev if e["kind"] == "h2d")
last_gemm = max(e["end_ms"] for e in ev if e["kind"] == "gemm")
print(f"first gemm {first_gemm:.0f} ms, last h2d {last_h2d:.0f} ms, last gemm {last_gemm:.0f} ms")
print("bin(ms)  gemm  h2d  conv  d2h  (busy fraction of the bin; gemm launches may overlap)")
for i in range(nb):
    print(f"{i * binw:7.0f} " + " ".join(f"{busy[k][i] / binw:5.2f}" for k in kinds[:4]))
