"""Sustained (power-capped) K1 rate for the current TR_K1_ORDER / TR_K1_HINTS:
cfg2 warm products for ~12 s per precision, median SM clock and board power
sampled by NVML every 5 ms, K1 launch time from the session's timing pairs."""
import statistics
import sys
import threading
import time

import numpy as np
import pynvml
import torch

import paper_1511_04348_b200 as tr

pynvml.nvmlInit()
H = pynvml.nvmlDeviceGetHandleByIndex(0)
samples, on = [], [False]


def loop():
    while True:
        if on[0]:
            samples.append((pynvml.nvmlDeviceGetClockInfo(H, pynvml.NVML_CLOCK_SM),
                            pynvml.nvmlDeviceGetPowerUsage(H) / 1e3))
        time.sleep(0.005)


threading.Thread(target=loop, daemon=True).start()
n, T = 32768, 4096
g = torch.Generator(device="cuda")
A = torch.randn((n, n), generator=g.manual_seed(1), device="cuda")
B = torch.randn((n, n), generator=g.manual_seed(2), device="cuda")
C = torch.empty((n, n), device="cuda")
m = tr.homogeneous_machine(1, dtype=np.float32)
secs = float(sys.argv[1]) if len(sys.argv) > 1 else 12.0
for prec in ("fp32acc", "bf16"):
    with tr.Runtime(m, T, precision=prec) as rt:
        rt.multiply(A, B, a_uid="A", b_uid="B", out=C)
        torch.cuda.synchronize()
        samples.clear()
        on[0] = True
        t0, ms, launches = time.perf_counter(), 0.0, 0
        while time.perf_counter() - t0 < secs:
            _, s = rt.multiply(A, B, a_uid="A", b_uid="B", out=C)
            ms += sum(s.kernel_ms.values())
            launches += s.gpu_launches
        torch.cuda.synchronize()
        on[0] = False
        mhz = statistics.median(x[0] for x in samples)
        w = statistics.median(x[1] for x in samples)
        per = ms / launches
        tf = 2.0 * n ** 3 / 16 / (per / 1e3) / 1e12
        print(f"{prec}: launch {per:.3f} ms = {tf:.1f} TF/s at {mhz:.0f} MHz, {w:.0f} W, {tf / mhz * 1e3:.1f} TF/s per GHz",
              flush=True)
