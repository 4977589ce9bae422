"""Probe: BASELINE cfg4 at its full size, N = 131072 fp32-accurate, on one B200.

The three distinct operands need 206 GB of pinned host memory and the GPU boxes
have ~196 GB, so B aliases A's host buffer (C = A.A) but is registered under its
own uid "B": the tile cache keys, fetches, evicts and converts B's tiles exactly
as it would a distinct matrix, so the H2D traffic, HBM footprint and compute are
those of cfg4 (A, B, C = 64 GiB each; 2 x 32^2 first-touch input tiles, 1024 C
writebacks).  Refuses to run when the host cannot pin 2 x 64 GiB with headroom.

Prints one JSON line (rank 0, N = 1).  Dev tool; the numbers go to profiles/.
"""
import json
import sys
import time

import numpy as np
import torch

import paper_1511_04348_b200 as tr

n = int(sys.argv[1]) if len(sys.argv) > 1 else 131072
T = 4096
budget_gib = float(sys.argv[2]) if len(sys.argv) > 2 else 0.0  # 0 = runtime default (80% of free HBM)
steps = int(sys.argv[3]) if len(sys.argv) > 3 else 1
mat_bytes = n * n * 4


def mem_available() -> int:
    for line in open("/proc/meminfo"):
        if line.startswith("MemAvailable:"):
            return int(line.split()[1]) * 1024
    return 0


avail = mem_available()
need = 2 * mat_bytes + 24 * 2**30
print(f"MemAvailable {avail / 2**30:.1f} GiB, need {need / 2**30:.1f} GiB", flush=True)
if avail < need:
    print(json.dumps({"skipped": f"host MemAvailable {avail / 2**30:.1f} GiB < {need / 2**30:.1f} GiB"}))
    sys.exit(0)

t0 = time.perf_counter()
a = tr.matrix.pinned_empty((n, n), np.float32)
c = tr.matrix.pinned_empty((n, n), np.float32)
print(f"pinned alloc {time.perf_counter() - t0:.1f} s", flush=True)
g = torch.Generator(device="cuda").manual_seed(1)
rows = 4096
at = torch.from_numpy(a)
for r in range(0, n, rows):
    at[r:r + rows].copy_(torch.randn((rows, n), device="cuda", generator=g))
torch.cuda.synchronize()
print(f"filled {time.perf_counter() - t0:.1f} s", flush=True)

machine = tr.homogeneous_machine(1, dtype=np.float32)
budget = int(budget_gib * 2**30)


mode = sys.argv[4] if len(sys.argv) > 4 else "cold"  # "cold": one-shot sessions; "warm": + a re-multiply


def step():
    with tr.Runtime(machine, T, precision="fp32acc", hbm_budget_bytes=budget) as rt:
        if order := (sys.argv[5] if len(sys.argv) > 5 else None):
            rt.set_order(order)
        st = rt.multiply(a, a, a_uid="A", b_uid="B", c_uid="C", out=c)[1]
        print(f"  cold: launches {st.gpu_launches}, kernel_ms {st.kernel_ms[0]:.0f}, span_ms {st.span_ms[0]:.0f}, "
              f"host fetches {st.cache.host_fetches}, evictions {st.cache.evictions}", flush=True)
        if mode == "warm":
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            w = rt.multiply(a, a, a_uid="A", b_uid="B", c_uid="C2", out=c)[1]
            e1.record()
            torch.cuda.synchronize()
            wt = e0.elapsed_time(e1)
            print(f"  warm: {wt:.0f} ms ({2.0 * n ** 3 / wt / 1e9:.1f} TF/s), launches {w.gpu_launches}, "
                  f"kernel_ms {w.kernel_ms[0]:.0f}, span_ms {w.span_ms[0]:.0f}, host fetches {w.cache.host_fetches}",
                  flush=True)
        return st


import subprocess  # noqa: E402

smi = subprocess.Popen(["nvidia-smi", "--query-gpu=timestamp,clocks.sm,power.draw,clocks_throttle_reasons.active",
                        "--format=csv,noheader", "-lms", "500"], stdout=open("gpurun_out/c4_clocks.csv", "w"))
times, stats = [], None
for i in range(steps + 1):  # the first is the warm-up (pools, pinned registration)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    w0 = time.perf_counter()
    e0.record()
    stats = step()
    e1.record()
    torch.cuda.synchronize()
    dt = e0.elapsed_time(e1) / 1e3
    print(f"step {i}: {dt * 1e3:.0f} ms event, {(time.perf_counter() - w0) * 1e3:.0f} ms wall, "
          f"{2.0 * n ** 3 / dt / 1e12:.1f} TF/s", flush=True)
    if i:
        times.append(dt)
smi.terminate()

t = float(np.mean(times))
flops = 2.0 * n ** 3
cs = stats.cache
peaks = json.load(open("MEASURED_PEAKS.json"))
peak_tf = float(peaks.get("bf16_tflops", 1645.7))
h2d_bw, d2h_bw = 55.6e9, 56e9
t_roof = max(flops / (peak_tf * 1e12 / 3), cs.bytes_host / h2d_bw, cs.bytes_writeback / d2h_bw)

from oracle import tilerun_oracle as O  # noqa: E402  (checker only)

ri = np.array([0, T - 1, T, n // 2 + 7, n - 1])
ci = np.array([1, T + 1, n // 3, n - 2, n - 1])
ref = O.c_oracle().gemm(a[ri].astype(np.float64), a[:, ci].astype(np.float64))
parity = float(np.linalg.norm(c[ri][:, ci].astype(np.float64) - ref) / np.linalg.norm(ref))
print(json.dumps({
    "workload": f"cfg4 full size: out-of-core GEMM N={n} fp32-accurate from pinned host, T={T}, "
                f"B aliases A's host buffer under its own uid (206 GB of distinct operands exceed the box's RAM)",
    "value": flops / t / 1e12, "unit": "TFLOP/s", "ms_per_step": t * 1e3, "steps": len(times),
    "step_ms": [x * 1e3 for x in times],
    "hbm_budget_gib": budget_gib or "default (80% of free HBM)",
    "host_fetches": cs.host_fetches, "bytes_host": cs.bytes_host, "l1_hits": cs.l1_hits,
    "evictions": cs.evictions, "writebacks": cs.writebacks, "bytes_writeback": cs.bytes_writeback,
    "tasks_completed": int(sum(d.tasks_completed for d in stats.devices.values())),
    "roofline": {"time_ms": t_roof * 1e3, "frac": t_roof / t,
                 "frac_vs_sustained_peak": max(flops / (float(peaks.get("bf16_tflops_sustained", peak_tf)) * 1e12 / 3),
                                               cs.bytes_host / h2d_bw, cs.bytes_writeback / d2h_bw) / t,
                 "def": f"max(2N^3 / (bf16 burst peak {peak_tf:.1f} / 3), bytes_host / 55.6 GB/s, "
                        f"bytes_writeback / 56 GB/s)"},
    "parity_rel_fro_sampled": parity,
    "parity_sample": "rows {0,T-1,T,n/2+7,n-1} x cols {1,T+1,n/3,n-2,n-1} vs the f64 C oracle",
}), flush=True)
