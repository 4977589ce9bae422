"""Probe: cfg3 MLP step time with / without write-through of operand tiles.  Dev tool."""
import numpy as np
import torch
import paper_1511_04348_b200 as tr

sizes = [784, 8192, 8192, 8192, 10]; batch = 8192
for prec in ("fp32acc", "bf16"):
    for wt in (False, True, False, True):
        rng = np.random.default_rng(0)
        layers = [tr.Layer.random(sizes[i], sizes[i + 1], rng, scale=1 / np.sqrt(sizes[i]), tag=f"layer{i}")
                  for i in range(4)]
        x, t = tr.ann.random_regression(rng, batch, 784, 10)
        mlp = tr.GpuMLP(layers, tile_size=4096, precision=prec, write_through=wt)
        xd = torch.as_tensor(x, dtype=torch.float32).cuda(); td = torch.as_tensor(t, dtype=torch.float32).cuda()
        for _ in range(3):
            mlp.train_step(xd, td, 0.1)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        ls = [mlp.train_step(xd, td, 0.1) for _ in range(10)]
        e1.record(); torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 10
        print(f"{prec:8s} write_through={wt}: {ms:.2f} ms/step  {batch / ms * 1e3:,.0f} samples/s  loss {ls[-1]:.6f}",
              flush=True)
        mlp.close()
