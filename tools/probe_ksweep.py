"""Probe: tile-GEMM launch time vs K (fixed 4096x4096 output) -> per-launch fixed cost.  Dev tool."""
import numpy as np
import torch
import paper_1511_04348_b200 as tr

T = 4096
for prec in ("fp32acc", "bf16"):
    rows = []
    for K in (64, 256, 1024, 4096, 8192, 16384, 32768):
        a = torch.randn(T, K, device="cuda"); b = torch.randn(K, T, device="cuda"); c = torch.empty(T, T, device="cuda")
        rt = tr.Runtime(tr.homogeneous_machine(1, dtype=np.float32), T, precision=prec)
        rt.set_inflight(1)
        ms = []
        for it in range(4):
            _, s = rt.multiply(a, b, a_uid="A", b_uid="B", out=c)
            ms.append(s.kernel_ms[0])
        rt.close()
        t = float(np.median(ms[1:]))
        rows.append((K, t))
        print(f"{prec:8s} K={K:6d}  {t*1e3:8.1f} us  {2*T*T*K/t/1e9:7.1f} TF/s", flush=True)
    K = np.array([r[0] for r in rows], float); t = np.array([r[1] for r in rows])
    A = np.vstack([np.ones_like(K), K]).T
    (a0, a1), *_ = np.linalg.lstsq(A[2:], t[2:], rcond=None)
    print(f"{prec}: fit t = {a0*1e3:.1f} us + K * {a1*1e6:.3f} ns  -> asymptotic {2*T*T/a1/1e9:.0f} TF/s")
