"""Probe: split-K correctness diagnostics + MLP step time with/without split-K.  Dev tool."""
import time
import numpy as np
import torch
import paper_1511_04348_b200 as tr
from paper_1511_04348_b200.dense import set_splitk

g = torch.Generator().manual_seed(11)
f = lambda *s: torch.randn(*s, generator=g, dtype=torch.float64)
x, w, bias = f(1000, 8192), f(8192, 10), f(10)
dev = lambda t: t.float().cuda().contiguous()
ref0 = x @ w
for S in (1, 8):
    set_splitk(S)
    for post in (None, "bias_act"):
        rt = tr.Runtime(tr.homogeneous_machine(1, dtype=np.float32), 4096)
        o1 = torch.empty(1000, 10, device="cuda")
        pr = dict(a=dev(x), b=dev(w), out=o1)
        if post:
            pr["post"] = ("bias_act", dev(bias), "sigmoid")
        s = rt.multiply_batch([pr])
        ref = torch.sigmoid(ref0 + bias) if post else ref0
        o = o1.double().cpu()
        err = (o - ref).norm() / ref.norm()
        bad = (o - ref).abs().max()
        print(f"S={S} post={post}: rel {err:.3e} maxabs {bad:.3e} launches {s.gpu_launches} kernel_ms {s.kernel_ms[0]:.3f}",
              flush=True)
        if err > 1e-5:
            d = (o - ref).abs()
            idx = torch.nonzero(d > 1e-3 * ref.abs().max())
            print("   bad rows", sorted(set(idx[:, 0].tolist()))[:20], "cols", sorted(set(idx[:, 1].tolist())))
        rt.close()
set_splitk(8)
