"""Probe: N plain cfg3 training steps (for ncu captures of single kernels).  Dev tool.
usage: probe_mlp_steps.py [steps]"""
import sys
import torch
import paper_1511_04348_b200 as tr

steps = int(sys.argv[1]) if len(sys.argv) > 1 else 2
sizes = [784, 8192, 8192, 8192, 10]
g = torch.Generator(device="cuda").manual_seed(1)
x = torch.rand(8192, sizes[0], device="cuda", generator=g) * 2 - 1
t = torch.rand(8192, sizes[-1], device="cuda", generator=g) * 2 - 1
m = tr.GpuMLP.random(sizes, seed=0)
for _ in range(steps):
    print(m.train_step(x, t, 0.1))
