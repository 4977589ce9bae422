"""Probe: cold cfg2 run() time vs (k-steps per finishing unit, k-major panels):
COMBOS="F:P,..." (TR_PANEL_FINISH / TR_PANELS, read per run).  Dev tool."""
import os
import numpy as np
import torch
import paper_1511_04348_b200 as tr

n, T = 32768, 4096
a = tr.matrix.pinned_empty((n, n), np.float32)
b = tr.matrix.pinned_empty((n, n), np.float32)
g = torch.Generator(device="cuda").manual_seed(1)
for m in (a, b):
    for r in range(0, n, 4096):
        m[r:r + 4096] = torch.randn((4096, n), device="cuda", generator=g).cpu().numpy()
machine = tr.homogeneous_machine(1, dtype=np.float32)
for _ in range(2):
    c, s = tr.run(machine, a, b, T)
    del c
res = {}
for rep in range(3):
    for f in os.environ.get("COMBOS", "8:2,1:2,2:2,3:2").split(","):
        os.environ["TR_PANEL_FINISH"], os.environ["TR_PANELS"] = f.split(":")
        c = None
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        c, s = tr.run(machine, a, b, T)
        e1.record()
        torch.cuda.synchronize()
        res.setdefault(f, []).append(e0.elapsed_time(e1))
for f, v in res.items():
    print(f"F={f}: {np.round(v, 1).tolist()}  median {np.median(v):.1f} ms")
