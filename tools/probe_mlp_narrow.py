"""Probe: cfg3 step time with the narrow output layer on the tensor cores
(transposed product) vs on CUDA cores, alternating in one process.  Dev tool.
usage: probe_mlp_narrow.py [fp32acc|bf16]"""
import sys
import numpy as np
import torch
import paper_1511_04348_b200 as tr
from paper_1511_04348_b200.dense import set_narrow_tc

sys.path.insert(0, ".")
from bench import train_steps  # noqa: E402

prec = sys.argv[1] if len(sys.argv) > 1 else "fp32acc"
sizes = [784, 8192, 8192, 8192, 10]
batch = 8192
g = torch.Generator(device="cuda").manual_seed(1)
xs = (torch.rand(batch, sizes[0], device="cuda", generator=g) * 2 - 1).cpu().pin_memory()
ts = (torch.rand(batch, sizes[-1], device="cuda", generator=g) * 2 - 1).cpu().pin_memory()
m = tr.GpuMLP.random(sizes, seed=0, precision=prec)
res = {True: [], False: []}
for rep in range(12):
    for on in (True, False):
        set_narrow_tc(on)
        train_steps(torch, m, xs, ts, 1)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        train_steps(torch, m, xs, ts, 3)
        e1.record()
        torch.cuda.synchronize()
        res[on].append(e0.elapsed_time(e1) / 3)
for on, t in res.items():
    print(f"{prec} narrow_tc={int(on)}: median {np.median(t):.3f} ms/step  {np.round(t, 2).tolist()}")
