"""K1 against cuBLAS on the same box, same shape, interleaved (so clocks and
power state are shared): cfg2's N = 32768 product.

  ours bf16      Runtime(precision="bf16") warm multiply, fp32 A/B/C resident
  ours fp32acc   the same in split-bf16x3 (FP32-accurate)
  cublas bf16    torch.matmul on bf16 copies (bf16 out)
  cublas fp32    torch.matmul fp32, TF32 off (SGEMM)
  cublas tf32    torch.matmul fp32, TF32 on
"""
import json
import statistics
import sys

import torch

import paper_1511_04348_b200 as tr

import threading
import time

import pynvml

pynvml.nvmlInit()
H = pynvml.nvmlDeviceGetHandleByIndex(0)


class Sampler:
    """SM clock (MHz) and board power (W) every 5 ms while active."""

    def __init__(self):
        self.on, self.samples = False, []
        threading.Thread(target=self._loop, daemon=True).start()

    def _loop(self):
        while True:
            if self.on:
                self.samples.append((pynvml.nvmlDeviceGetClockInfo(H, pynvml.NVML_CLOCK_SM),
                                     pynvml.nvmlDeviceGetPowerUsage(H) / 1e3))
            time.sleep(0.005)

    def start(self):
        self.samples = []
        self.on = True

    def stop(self):
        self.on = False
        s = self.samples or [(-1, -1)]
        return statistics.median(x[0] for x in s), statistics.median(x[1] for x in s)


SAMPLER = Sampler()

n = int(sys.argv[1]) if len(sys.argv) > 1 else 32768
T = 4096
flops = 2.0 * n ** 3
g = torch.Generator(device="cuda")
A = torch.randn((n, n), generator=g.manual_seed(1), device="cuda")
B = torch.randn((n, n), generator=g.manual_seed(2), device="cuda")
C = torch.empty((n, n), device="cuda")
Ah, Bh = A.bfloat16(), B.bfloat16()
machine = tr.homogeneous_machine(1, dtype="float32") if False else tr.homogeneous_machine(1)
rts = {p: tr.Runtime(machine, T, precision=p) for p in ("bf16", "fp32acc")}


def time_it(fn, reps=3):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    SAMPLER.start()
    e0.record()
    for _ in range(reps):
        r = fn()
    e1.record()
    torch.cuda.synchronize()
    mhz, watts = SAMPLER.stop()
    extra = {}
    if isinstance(r, tuple):  # ours: per-launch K1 time from the session's timing pairs
        s = r[1]
        extra = {"launches": s.gpu_launches, "avg_launch_ms": sum(s.kernel_ms.values()) / max(1, s.gpu_launches)}
    return e0.elapsed_time(e1) / reps, mhz, watts, extra


def ours(p):
    return lambda: rts[p].multiply(A, B, a_uid="A", b_uid="B", out=C)


def cublas(kind):
    def f():
        if kind == "bf16":
            torch.matmul(Ah, Bh)
        else:
            torch.backends.cuda.matmul.allow_tf32 = kind == "tf32"
            torch.matmul(A, B)
    return f


arms = {"ours_bf16": ours("bf16"), "cublas_bf16": cublas("bf16"), "ours_fp32acc": ours("fp32acc"),
        "cublas_fp32": cublas("fp32"), "cublas_tf32": cublas("tf32")}
res = {k: [] for k in arms}
for rnd in range(3):
    for k, fn in arms.items():
        res[k].append(time_it(fn, reps=2 if "fp32" in k and "cublas" in k else 8))
out = {}
for k, v in res.items():
    ms = statistics.median(x[0] for x in v)
    out[k] = {"ms": round(ms, 2), "tflops": round(flops / ms / 1e9, 1), "sm_mhz": [x[1] for x in v],
              "watts": [round(x[2]) for x in v], **v[-1][3]}
    if "launches" in v[-1][3]:
        out[k]["launch_tflops"] = round(flops / v[-1][3]["launches"] / v[-1][3]["avg_launch_ms"] / 1e9, 1)
with torch.profiler.profile(activities=[torch.profiler.ProfilerActivity.CUDA]) as prof:
    cublas("bf16")()
    torch.cuda.synchronize()
out["cublas_bf16_kernels"] = sorted({e.name for e in prof.events() if e.device_type.name == "CUDA"})
out["ratio_bf16_ours_over_cublas"] = round(out["cublas_bf16"]["ms"] / out["ours_bf16"]["ms"], 3)
out["ratio_fp32acc_over_sgemm"] = round(out["cublas_fp32"]["ms"] / out["ours_fp32acc"]["ms"], 2)
print(json.dumps({"n": n, "tile": T, **out}, indent=1))
