"""Probe: where does one cfg3 MLP training step spend its time?  Dev tool."""
import time
import numpy as np
import torch
import paper_1511_04348_b200 as tr

sizes = [784, 8192, 8192, 8192, 10]; batch = 8192
rng = np.random.default_rng(0)
layers = [tr.Layer.random(sizes[i], sizes[i + 1], rng, scale=1 / np.sqrt(sizes[i]), tag=f"layer{i}") for i in range(4)]
x, t = tr.ann.random_regression(rng, batch, 784, 10)
import sys
T = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
mlp = tr.GpuMLP(layers, tile_size=T)
xd = torch.as_tensor(x, dtype=torch.float32).cuda(); td = torch.as_tensor(t, dtype=torch.float32).cuda()
for _ in range(2):
    mlp.train_step(xd, td, 0.1)
# instrument the product calls
orig = mlp.rt.multiply_batch
log = []
def timed(*a, **k):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    out = orig(*a, **k)
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    s = out
    shape = [(tuple(p["a"].shape), tuple(p["b"].shape), p.get("post", (None,))[0]) for p in a[0]]
    log.append((1e3 * (t1 - t0), s.span_ms[0], s.kernel_ms[0], s.total_tasks, s.gpu_launches, shape))
    return out
mlp.rt.multiply_batch = timed
torch.cuda.synchronize(); t0 = time.perf_counter()
mlp.train_step(xd, td, 0.1)
torch.cuda.synchronize(); step = 1e3 * (time.perf_counter() - t0)
print(f"T={T} step {step:.2f} ms; products wall {sum(l[0] for l in log):.2f} ms, span {sum(l[1] for l in log):.2f}, kernels {sum(l[2] for l in log):.2f}")
for l in log:
    print(f"  wall {l[0]:6.2f} span {l[1]:6.2f} kern {l[2]:6.2f} tasks {l[3]} launches {l[4]}  {l[5]}")
