"""Probe: which sequence breaks green-context sessions.  Dev tool."""
import sys
import numpy as np
import paper_1511_04348_b200 as tr
from paper_1511_04348_b200 import DeviceSpec, Machine, ProximityMatrix

seq = sys.argv[1]
if len(sys.argv) > 3 and sys.argv[3] == "torch_first":
    import torch
    torch.zeros(1, device="cuda")
    torch.empty(4, pin_memory=True)
cfg = sys.argv[2] if len(sys.argv) > 2 else "64,32"
specs = [DeviceSpec(i, gpu=0, sms=(int(v) or None)) for i, v in enumerate(cfg.split(","))]
m = Machine(specs, ProximityMatrix.uniform(len(specs)), dtype=np.float32)
rt = tr.Runtime(m, 512)
h = np.ones((2048, 2048), np.float32)
dev = None
for step, kind in enumerate(seq):
    try:
        if kind == "h":
            _, s = rt.multiply(h, h)
        elif kind == "u":  # same uids: no slab growth
            _, s = rt.multiply(h, h, a_uid="HA", b_uid="HB")
        elif kind == "t":
            import torch
            dev = torch.ones((2048, 2048), device="cuda")
            s = None
        elif kind == "d":
            import torch
            out = torch.empty((2048, 2048), device="cuda")
            _, s = rt.multiply(dev, dev, out=out)
        elif kind == "s":
            import torch
            torch.cuda.synchronize()
            s = None
        print(seq, step, kind, "OK", None if s is None else s.tasks_by_device, flush=True)
    except Exception as e:
        print(seq, step, kind, "FAIL", str(e)[:100], flush=True)
        break
