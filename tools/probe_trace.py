"""Probe: device timeline of a cold (host-buffer) cfg2 product.  Dev tool."""
import json, sys
import numpy as np
import torch
import paper_1511_04348_b200 as tr

n, T = 32768, 4096
g = torch.Generator(device="cuda").manual_seed(1)
a = tr.matrix.pinned_empty((n, n), np.float32); a[...] = torch.randn((n, n), device="cuda", generator=g).cpu().numpy()
b = tr.matrix.pinned_empty((n, n), np.float32); b[...] = torch.randn((n, n), device="cuda", generator=g).cpu().numpy()
m = tr.homogeneous_machine(1, dtype=np.float32)

def union(iv):
    iv = sorted(iv); tot = 0.0; cur = None
    for s, e in iv:
        if cur is None or s > cur[1]:
            if cur: tot += cur[1] - cur[0]
            cur = [s, e]
        else:
            cur[1] = max(cur[1], e)
    return tot + (cur[1] - cur[0] if cur else 0.0)

for inflight in (2, 4):
    rt = tr.Runtime(m, T, trace=True)
    rt.set_inflight(inflight)
    rt.multiply(a, b)  # warm-up (slab sizing)
    c, s = rt.multiply(a, b)
    ev = s.trace
    by = {}
    for e in ev:
        by.setdefault(e["kind"], []).append((e["start_ms"], e["end_ms"]))
    print(f"inflight={inflight}: span {s.span_ms[0]:.1f} ms, {len(ev)} events", flush=True)
    for k, iv in by.items():
        print(f"  {k:8s} n={len(iv):4d} busy(union)={union(iv):7.1f} ms  first {min(x[0] for x in iv):7.1f}  "
              f"last_end {max(x[1] for x in iv):7.1f}  mean dur {np.mean([x[1]-x[0] for x in iv]):.3f}", flush=True)
    gem = sorted(by["gemm"])
    print("  first gemms:", [(round(x[0], 1), round(x[1], 1)) for x in gem[:6]])
    h2d = sorted(by["h2d"])
    print("  h2d gaps > 0.5 ms:", sum(1 for p, q in zip(h2d, h2d[1:]) if q[0] - p[1] > 0.5),
          "total gap", round(sum(max(0, q[0] - p[1]) for p, q in zip(h2d, h2d[1:])), 1))
    json.dump(ev, open(f"gpurun_out/trace_cold_inflight{inflight}.json", "w"))
    rt.close()
