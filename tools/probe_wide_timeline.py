"""Probe: CUPTI kernel timeline of one cfg5 (65536-wide) MLP step with the tile
cache capped (torch.profiler).  Dev tool.  usage: probe_wide_timeline.py [cache_gib]"""
import sys
import numpy as np
import torch
import paper_1511_04348_b200 as tr
from torch.profiler import ProfilerActivity, profile

gib = float(sys.argv[1]) if len(sys.argv) > 1 else 24.0
sizes = [784, 65536, 65536, 65536]
batch = 8192
rt = tr.Runtime(tr.homogeneous_machine(1, dtype=np.float32), 4096, hbm_budget_bytes=int(gib * 2**30))
import os
mlp = tr.GpuMLP.random(sizes, seed=0, runtime=rt, write_through_weights=os.environ.get("WTW", "1") == "1")
g = torch.Generator(device="cuda").manual_seed(1)
x = torch.rand(batch, sizes[0], device="cuda", generator=g) * 2 - 1
t = torch.rand(batch, sizes[-1], device="cuda", generator=g) * 2 - 1
mlp.train_step(x, t, 0.1)
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    mlp.train_step(x, t, 0.1)
    torch.cuda.synchronize()
prof.export_chrome_trace("gpurun_out/wide_trace.json")
print("counts", mlp.cache_counts)
