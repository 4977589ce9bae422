"""Probe: A/B of GpuMLP options on cfg3 in one process (alternating, same
clocks): ms/step for each variant.  Dev tool.  usage: probe_mlp_ab.py opt=val,... opt=val,..."""
import sys
import numpy as np
import torch
import paper_1511_04348_b200 as tr

sys.path.insert(0, ".")
from bench import train_steps  # noqa: E402

sizes = [784, 8192, 8192, 8192, 10]
batch = 8192
variants = []
for spec in sys.argv[1:] or ["fused_sgd=1", "fused_sgd=0"]:
    kw = {}
    for item in spec.split(","):
        k, v = item.split("=")
        kw[k] = bool(int(v))
    variants.append((spec, kw))
g = torch.Generator(device="cuda").manual_seed(1)
xs = (torch.rand(batch, sizes[0], device="cuda", generator=g) * 2 - 1).cpu().pin_memory()
ts = (torch.rand(batch, sizes[-1], device="cuda", generator=g) * 2 - 1).cpu().pin_memory()
mlps = {spec: tr.GpuMLP.random(sizes, seed=0, **kw) for spec, kw in variants}
res = {spec: [] for spec, _ in variants}
for rep in range(int(__import__("os").environ.get("REPS", "10"))):
    for spec, _ in variants:
        m = mlps[spec]
        train_steps(torch, m, xs, ts, 1)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        train_steps(torch, m, xs, ts, 3)
        e1.record()
        torch.cuda.synchronize()
        res[spec].append(e0.elapsed_time(e1) / 3)
for spec, v in res.items():
    print(f"{spec:30s} ms/step {np.median(v):7.3f}  all {np.round(v, 2).tolist()}")
