"""Probe: task shares of 8/16/24/32-SM green devices.  Dev tool."""
import numpy as np
import torch
import paper_1511_04348_b200 as tr
from paper_1511_04348_b200 import DeviceSpec, Machine, ProximityMatrix
from paper_1511_04348_b200.dense import set_task_group

n, T = 16384, 2048
a = torch.randn(n, n, device="cuda"); b = torch.randn(n, n, device="cuda"); c = torch.empty(n, n, device="cuda")
for grp in (4, 2, 1):
    set_task_group(grp)
    m = Machine([DeviceSpec(i, gpu=0, sms=8 * (i + 1)) for i in range(4)], ProximityMatrix.uniform(4), dtype=np.float32)
    rt = tr.Runtime(m, T)
    rt.multiply(a, b, a_uid="A", b_uid="B", out=c)
    tot = np.zeros(4)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(3):
        _, s = rt.multiply(a, b, a_uid="A", b_uid="B", out=c)
        tot += [s.tasks_by_device[d] for d in range(4)]
    e1.record(); torch.cuda.synchronize()
    print(f"group={grp}: shares {np.round(tot / tot.sum(), 3)}  {e0.elapsed_time(e1) / 3:.1f} ms/product", flush=True)
    rt.close()
