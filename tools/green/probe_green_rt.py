"""Probe: green-context logical devices through the Runtime.  Dev tool."""
import sys
import numpy as np
import paper_1511_04348_b200 as tr
from paper_1511_04348_b200 import DeviceSpec, Machine, ProximityMatrix

variant = sys.argv[1]
if variant == "torch_first":
    import torch
    torch.zeros(1, device="cuda")
m = Machine([DeviceSpec(0, gpu=0, sms=64), DeviceSpec(1, gpu=0, sms=32)], ProximityMatrix.uniform(2), dtype=np.float32)
rt = tr.Runtime(m, 512)
a = np.ones((2048, 2048), np.float32)
if variant == "torch_after":
    import torch
    ad = torch.ones((2048, 2048), device="cuda")
    cd = torch.empty((2048, 2048), device="cuda")
    try:
        _, s = rt.multiply(ad, ad, out=cd)
        print(variant, "device OK", float(cd[0, 0]), s.tasks_by_device)
    except Exception as e:
        print(variant, "device FAIL", e)
try:
    c, s = rt.multiply(a, a)
    print(variant, "OK", c[0, 0], s.tasks_by_device)
except Exception as e:
    print(variant, "FAIL", e)
