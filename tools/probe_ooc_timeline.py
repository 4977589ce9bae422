"""Probe: CUPTI timeline of one out-of-core product (N=65536 from pinned host,
tile cache capped at 24 GiB): kernel time by variant / grid, H2D and D2H busy.
Dev tool."""
import collections
import json
import os
import numpy as np
import torch
import paper_1511_04348_b200 as tr
from torch.profiler import ProfilerActivity, profile

n, T = 65536, 4096
a = tr.matrix.pinned_empty((n, n), np.float32)
b = tr.matrix.pinned_empty((n, n), np.float32)
c = tr.matrix.pinned_empty((n, n), np.float32)
g = torch.Generator(device="cuda").manual_seed(3)
for m in (a, b):
    for r in range(0, n, 4096):
        m[r:r + 4096] = torch.randn((4096, n), device="cuda", generator=g).cpu().numpy()
machine = tr.homogeneous_machine(1, dtype=np.float32)
budget = int(24 * 2**30)


def step():
    with tr.Runtime(machine, T, hbm_budget_bytes=budget) as rt:
        return rt.multiply(a, b, a_uid="A", b_uid="B", c_uid="C", out=c)[1]


step()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    s = step()
    torch.cuda.synchronize()
prof.export_chrome_trace("gpurun_out/ooc_trace.json")
ev = json.load(open("gpurun_out/ooc_trace.json"))["traceEvents"]
os.remove("gpurun_out/ooc_trace.json")
k = [e for e in ev if e.get("cat") in ("kernel", "gpu_memcpy") and "dur" in e]
t0 = min(e["ts"] for e in k)
t1 = max(e["ts"] + e["dur"] for e in k)
print(f"span {(t1 - t0) / 1e3:.1f} ms  wall {s.wall_elapsed * 1e3:.1f} ms")
agg = collections.defaultdict(lambda: [0, 0.0])
for e in k:
    name = e["name"]
    if "tile_gemm" in name:
        name = name[name.index("tile_gemm"):name.index(">") + 1] + f" grid={e.get('args', {}).get('grid')}"
    elif "Memcpy" in name:
        name = name.split("(")[0]
    else:
        name = name[:60]
    agg[name][0] += 1
    agg[name][1] += e["dur"]
for name, (cnt, d) in sorted(agg.items(), key=lambda x: -x[1][1])[:20]:
    print(f"{d / 1e3:9.1f} ms {cnt:6d}  {name}")
kern = sorted((e["ts"], e["ts"] + e["dur"]) for e in k if e["cat"] == "kernel")
busy, cs, ce = 0.0, None, None
for s0, s1 in kern:
    if ce is None or s0 > ce:
        if ce is not None:
            busy += ce - cs
        cs, ce = s0, s1
    else:
        ce = max(ce, s1)
busy += ce - cs
print(f"kernel busy union {busy / 1e3:.1f} ms")
