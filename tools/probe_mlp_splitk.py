"""Probe: cfg3 step time with split-K on (8) / off (1), alternating in one
process on one model.  Dev tool."""
import sys
import numpy as np
import torch
import paper_1511_04348_b200 as tr
from paper_1511_04348_b200.dense import set_splitk

sys.path.insert(0, ".")
from bench import train_steps  # noqa: E402

sizes = [784, 8192, 8192, 8192, 10]
batch = 8192
g = torch.Generator(device="cuda").manual_seed(1)
xs = (torch.rand(batch, sizes[0], device="cuda", generator=g) * 2 - 1).cpu().pin_memory()
ts = (torch.rand(batch, sizes[-1], device="cuda", generator=g) * 2 - 1).cpu().pin_memory()
m = tr.GpuMLP.random(sizes, seed=0)
res = {8: [], 1: []}
for rep in range(12):
    for sk in (8, 1):
        set_splitk(sk)
        train_steps(torch, m, xs, ts, 1)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        train_steps(torch, m, xs, ts, 3)
        e1.record()
        torch.cuda.synchronize()
        res[sk].append(e0.elapsed_time(e1) / 3)
for sk, v in res.items():
    print(f"splitk={sk}: median {np.median(v):.3f} ms/step  {np.round(v, 2).tolist()}")
