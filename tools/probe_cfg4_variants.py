"""Probe: schedule variants of the full-size cfg4 product (N = 131072, B aliases
A's host buffer under its own uid, see probe_cfg4_full.py), cold one-shot
sessions, one process (the 128 GiB of pinned host memory is allocated once).
Dev tool."""
import os
import subprocess
import sys
import time

import numpy as np
import torch

import paper_1511_04348_b200 as tr

n = int(sys.argv[1]) if len(sys.argv) > 1 else 131072
T = 4096
variants = [v for v in (sys.argv[2] if len(sys.argv) > 2 else "default").split(";")]
a = tr.matrix.pinned_empty((n, n), np.float32)
c = tr.matrix.pinned_empty((n, n), np.float32)
g = torch.Generator(device="cuda").manual_seed(1)
at = torch.from_numpy(a)
for r in range(0, n, 4096):
    at[r:r + 4096].copy_(torch.randn((4096, n), device="cuda", generator=g))
torch.cuda.synchronize()
machine = tr.homogeneous_machine(1, dtype=np.float32)
knobs = ("TR_PANELS", "TR_PANEL_GROUP", "TR_PANEL_FINISH")
for v in variants:
    # "order=shells,TR_PANELS=2,..." ; keys not given are unset
    kv = dict(x.split("=") for x in v.split(",") if "=" in x)
    for k in knobs:
        os.environ.pop(k, None)
    for k, val in kv.items():
        if k.startswith("TR_"):
            os.environ[k] = val
    smi = subprocess.Popen(["nvidia-smi", "--query-gpu=clocks.sm,power.draw", "--format=csv,noheader,nounits",
                            "-lms", "250"], stdout=subprocess.PIPE, text=True)
    with tr.Runtime(machine, T, precision="fp32acc", trace="trace" in kv) as rt:
        if "order" in kv:
            rt.set_order(kv["order"])
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record()
        st = rt.multiply(a, a, a_uid="A", b_uid="B", c_uid="C", out=c)[1]
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1)
    smi.terminate()
    clk = sorted(float(x.split(",")[0]) for x in smi.communicate()[0].split("\n") if x.strip())
    clk = [x for x in clk if x < 1965] or clk  # samples under the power cap
    print(f"{v:40s} {ms:8.0f} ms sm_mhz~{clk[len(clk) // 2]:.0f} {2.0 * n ** 3 / ms / 1e9:6.1f} TF/s  launches {st.gpu_launches} "
          f"kernel_ms {st.kernel_ms[0]:.0f} span_ms {st.span_ms[0]:.0f}", flush=True)
    if st.trace:
        ev = st.trace
        g = sorted((e for e in ev if e["kind"] == "gemm"), key=lambda e: e["start_ms"])
        h = sorted((e for e in ev if e["kind"] in ("h2d", "fill", "copy")), key=lambda e: e["start_ms"])
        kinds = sorted({e["kind"] for e in ev})
        print("  kinds", kinds, "gemm events", len(g))
        t0 = min(e["start_ms"] for e in ev)
        if h:
            print(f"  h2d first {h[0]['start_ms'] - t0:.0f} last end {max(e['end_ms'] for e in h) - t0:.0f} ms")
        gaps, end = [], g[0]["end_ms"]
        print(f"  first gemm at {g[0]['start_ms'] - t0:.1f} ms")
        for e in g[1:]:
            if e["start_ms"] > end + 0.05:
                gaps.append((e["start_ms"] - end, end - t0, e["task"]))
            end = max(end, e["end_ms"])
        print(f"  gemm idle total {sum(x[0] for x in gaps):.0f} ms in {len(gaps)} gaps; last gemm end {end - t0:.0f}, "
              f"span {max(e['end_ms'] for e in ev) - t0:.0f}")
        for lo, hi in ((0, 1000), (1000, 3000), (3000, 6000), (6000, 20000)):
            print(f"   idle in [{lo},{hi}) ms: {sum(x[0] for x in gaps if lo <= x[1] < hi):.0f}")
        cv = [e for e in ev if e["kind"] == "convert"]
        busy = [(e["start_ms"], e["end_ms"]) for e in g]
        in_gemm = sum(any(a <= e["start_ms"] < b for a, b in busy) for e in cv)
        print(f"  converts {len(cv)}: {in_gemm} start while a GEMM runs; mean dur "
              f"{sum(e['end_ms'] - e['start_ms'] for e in cv) / max(1, len(cv)):.2f} ms")
        for x in sorted(gaps, reverse=True)[:6]:
            print(f"   gap {x[0]:.1f} ms at {x[1]:.0f} ms, next task {x[2]}")
