"""Probe: CUPTI kernel/memcpy timeline of cfg3 MLP steps (torch.profiler).  Dev tool."""
import json, sys
import numpy as np
import torch
import paper_1511_04348_b200 as tr
from torch.profiler import ProfilerActivity, profile

ordered = sys.argv[1] == "1" if len(sys.argv) > 1 else True
prec = sys.argv[2] if len(sys.argv) > 2 else "fp32acc"
sizes = [784, 8192, 8192, 8192, 10]; batch = 8192
rng = np.random.default_rng(0)
layers = [tr.Layer.random(sizes[i], sizes[i + 1], rng, scale=1 / np.sqrt(sizes[i]), tag=f"layer{i}") for i in range(4)]
x, t = tr.ann.random_regression(rng, batch, 784, 10)
mlp = tr.GpuMLP(layers, tile_size=4096, precision=prec, stream_ordered=ordered)
xd = torch.as_tensor(x, dtype=torch.float32).cuda(); td = torch.as_tensor(t, dtype=torch.float32).cuda()
for _ in range(3):
    mlp.train_step(xd, td, 0.1)
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
    for _ in range(2):
        mlp.train_step(xd, td, 0.1)
    torch.cuda.synchronize()
prof.export_chrome_trace(f"gpurun_out/mlp_trace_{int(ordered)}_{prec}.json")
print("exported")
