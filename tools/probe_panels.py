"""Probe: cold cfg2 product span vs the number of k-major panels (TR_PANELS).  Dev tool."""
import os
import numpy as np
import torch
import paper_1511_04348_b200 as tr

n, T = 32768, 4096
g = torch.Generator(device="cuda").manual_seed(1)
a = tr.matrix.pinned_empty((n, n), np.float32); a[...] = torch.randn((n, n), device="cuda", generator=g).cpu().numpy()
b = tr.matrix.pinned_empty((n, n), np.float32); b[...] = torch.randn((n, n), device="cuda", generator=g).cpu().numpy()
m = tr.homogeneous_machine(1, dtype=np.float32)
c, s = tr.run(m, a, b, T)  # warm-up: pools
import itertools
cases = [("shells", None, None, "")] + [("k-panels", P, GB, "") for P in (2, 3) for GB in (1, 2)]
for order, P, GB, SCHED in cases:
        os.environ["TR_PANEL_SCHED"] = SCHED
        if P is not None:
            os.environ["TR_PANELS"] = str(P)
            os.environ["TR_PANEL_GROUP"] = str(GB)
        spans = []
        for _ in range(3):
            c = None
            with tr.Runtime(m, T) as rt:  # fresh session: a cold product, like run()
                rt.set_order(order)
                c, s = rt.multiply(a, b, a_uid="A", b_uid="B", c_uid="C")
            spans.append(s.span_ms[0])
        print(f"{order:9s} P={P} GB={GB} {SCHED}: span {np.mean(spans):6.1f} ms  ({', '.join(f'{x:.1f}' for x in spans)})", flush=True)
