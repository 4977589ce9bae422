"""Probe: cold one-shot run() of cfg2 (N=32768, T=4096) from pinned host buffers,
1 warm-up + 5 timed (CUDA events); for A/B runs of two library builds.  Dev tool."""
import numpy as np
import torch

import paper_1511_04348_b200 as tr

n, T = 32768, 4096
a = tr.matrix.pinned_empty((n, n), np.float32)
b = tr.matrix.pinned_empty((n, n), np.float32)
g = torch.Generator(device="cuda").manual_seed(1)
torch.from_numpy(a).copy_(torch.randn((n, n), device="cuda", generator=g))
torch.from_numpy(b).copy_(torch.randn((n, n), device="cuda", generator=g))
m = tr.homogeneous_machine(1, dtype=np.float32)
ts = []
for i in range(6):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    c, s = tr.run(m, a, b, T)
    e1.record()
    torch.cuda.synchronize()
    if i:
        ts.append(e0.elapsed_time(e1))
    del c
print(f"e2e ms {['%.1f' % t for t in ts]} mean {np.mean(ts):.1f} -> {2 * n**3 / np.mean(ts) / 1e9:.1f} TF/s", flush=True)
