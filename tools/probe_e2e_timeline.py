"""Probe: CUPTI timeline of the one-shot cold run() (cfg2 from pinned host):
H2D / kernels / D2H occupancy over time.  Dev tool."""
import json
import numpy as np
import torch
import paper_1511_04348_b200 as tr
from torch.profiler import ProfilerActivity, profile

n, T = 32768, 4096
a = tr.matrix.pinned_empty((n, n), np.float32)
b = tr.matrix.pinned_empty((n, n), np.float32)
g = torch.Generator(device="cuda").manual_seed(1)
for m in (a, b):
    for r in range(0, n, 4096):
        m[r:r + 4096] = torch.randn((4096, n), device="cuda", generator=g).cpu().numpy()
machine = tr.homogeneous_machine(1, dtype=np.float32)
for _ in range(2):
    c, s = tr.run(machine, a, b, T)
    del c
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    c, s = tr.run(machine, a, b, T)
    torch.cuda.synchronize()
prof.export_chrome_trace("gpurun_out/e2e_trace.json")
ev = json.load(open("gpurun_out/e2e_trace.json"))["traceEvents"]
k = [e for e in ev if e.get("cat") in ("kernel", "gpu_memcpy") and "dur" in e]
t0 = min(e["ts"] for e in k)
t1 = max(e["ts"] + e["dur"] for e in k)
print(f"span {(t1 - t0) / 1e3:.1f} ms")
bins = np.zeros((int((t1 - t0) / 5000) + 1, 3))  # 5 ms bins: h2d, kernel, d2h busy fraction (union per kind)
for e in k:
    kind = 1 if e["cat"] == "kernel" else (0 if "HtoD" in e["name"] else 2)
    s0, s1 = e["ts"] - t0, e["ts"] - t0 + e["dur"]
    b0 = int(s0 // 5000)
    while s0 < s1:
        be = (b0 + 1) * 5000
        bins[b0, kind] += min(s1, be) - s0
        s0 = be
        b0 += 1
first_k = min(e["ts"] for e in k if e["cat"] == "kernel") - t0
last_k = max(e["ts"] + e["dur"] for e in k if e["cat"] == "kernel") - t0
h2d = [e for e in k if e["cat"] == "gpu_memcpy" and "HtoD" in e["name"]]
d2h = [e for e in k if e["cat"] == "gpu_memcpy" and "DtoH" in e["name"]]
print(f"first kernel at {first_k / 1e3:.1f} ms, last kernel ends {last_k / 1e3:.1f} ms")
print(f"h2d: {len(h2d)} copies, {sum(e['dur'] for e in h2d) / 1e3:.1f} ms busy, last ends {max(e['ts'] + e['dur'] for e in h2d) / 1e3 - t0 / 1e3:.1f}")
print(f"d2h: {len(d2h)} copies, {sum(e['dur'] for e in d2h) / 1e3:.1f} ms busy, first at {(min(e['ts'] for e in d2h) - t0) / 1e3:.1f}")
print("bin(5ms) h2d kern d2h (us of busy time, summed over overlapping events)")
for i, r in enumerate(bins):
    print(f"{i * 5:4d} {r[0] / 1e3:5.2f} {r[1] / 1e3:5.2f} {r[2] / 1e3:5.2f}")
