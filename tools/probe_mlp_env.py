"""Probe: cfg3 step time A/B over an environment switch read per launch
(e.g. TR_SPLIT_REDUCE_COST=0/1), alternating in one process.  Dev tool.
usage: probe_mlp_env.py NAME VAL_A VAL_B"""
import os
import sys
import numpy as np
import torch
import paper_1511_04348_b200 as tr

sys.path.insert(0, ".")
from bench import train_steps  # noqa: E402

name, va, vb = sys.argv[1:4]
sizes = [784, 8192, 8192, 8192, 10]
batch = 8192
g = torch.Generator(device="cuda").manual_seed(1)
xs = (torch.rand(batch, sizes[0], device="cuda", generator=g) * 2 - 1).cpu().pin_memory()
ts = (torch.rand(batch, sizes[-1], device="cuda", generator=g) * 2 - 1).cpu().pin_memory()
m = tr.GpuMLP.random(sizes, seed=0)
res = {va: [], vb: []}
for rep in range(12):
    for v in (va, vb):
        os.environ[name] = v
        train_steps(torch, m, xs, ts, 1)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        train_steps(torch, m, xs, ts, 3)
        e1.record()
        torch.cuda.synchronize()
        res[v].append(e0.elapsed_time(e1) / 3)
for v, t in res.items():
    print(f"{name}={v}: median {np.median(t):.3f} ms/step  {np.round(t, 2).tolist()}")
