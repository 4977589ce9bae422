"""Probe: CUPTI timeline of pipelined cfg3 steps exactly as bench.py runs them
(train_steps: async steps, batch prefetch, loss read one step late); prints the
GPU-idle gaps with the kernels on either side.  Dev tool."""
import sys

import numpy as np
import torch
from torch.profiler import ProfilerActivity, profile

import bench
import paper_1511_04348_b200 as tr

prec = sys.argv[1] if len(sys.argv) > 1 else "bf16"
sizes, batch = [784, 8192, 8192, 8192, 10], 8192
layers, x, t = bench.cfg3_problem(tr, sizes, batch)
xh = tr.matrix.pinned_empty(x.shape, np.float32)
th = tr.matrix.pinned_empty(t.shape, np.float32)
xh[...] = x
th[...] = t
mlp = tr.GpuMLP(layers, machine=tr.homogeneous_machine(1, dtype=np.float32), tile_size=4096, precision=prec)
xs, ts = torch.from_numpy(xh), torch.from_numpy(th)
bench.train_steps(torch, mlp, xs, ts, 3)
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    bench.train_steps(torch, mlp, xs, ts, 4)
    torch.cuda.synchronize()
ev = [e for e in prof.events() if e.device_type.name == "CUDA"]
ev.sort(key=lambda e: e.time_range.start)
t0 = ev[0].time_range.start
span = max(e.time_range.end for e in ev) - t0
busy, cur0, cur1, gaps = 0, ev[0].time_range.start, ev[0].time_range.end, []
prev = ev[0]
for e in ev[1:]:
    s, en = e.time_range.start, e.time_range.end
    if s > cur1:
        busy += cur1 - cur0
        gaps.append((s - cur1, (cur1 - t0) / 1e3, prev.name[:60], e.name[:60]))
        cur0, cur1 = s, en
    else:
        cur1 = max(cur1, en)
    prev = e if en >= cur1 else prev
busy += cur1 - cur0
print(f"{prec}: 4 steps span {span / 1e3:.2f} ms ({span / 4e3:.2f} ms/step), GPU busy {busy / 4e3:.2f} ms/step")
gaps.sort(reverse=True)
for g in gaps[:12]:
    print(f"gap {g[0]:7.1f} us at {g[1]:8.2f} ms after [{g[2]}] before [{g[3]}]")
