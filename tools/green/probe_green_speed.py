"""Probe: product time on one green-context device of various SM counts.  Dev tool."""
import numpy as np
import torch
import paper_1511_04348_b200 as tr
from paper_1511_04348_b200 import DeviceSpec, Machine, ProximityMatrix
from paper_1511_04348_b200.dense import set_task_group

n, T = 16384, 2048
a = torch.randn(n, n, device="cuda"); b = torch.randn(n, n, device="cuda"); c = torch.empty(n, n, device="cuda")
for grp in (4, 1):
    set_task_group(grp)
    for sms in (None, 64, 32, 16):
        rt = tr.Runtime(Machine([DeviceSpec(0, gpu=0, sms=sms)], ProximityMatrix.uniform(1), dtype=np.float32), T)
        rt.multiply(a, b, a_uid="A", b_uid="B", out=c)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(3):
            rt.multiply(a, b, a_uid="A", b_uid="B", out=c)
        e1.record(); torch.cuda.synchronize()
        print(f"group={grp} sms={sms}: {e0.elapsed_time(e1) / 3:.2f} ms", flush=True)
        rt.close()
