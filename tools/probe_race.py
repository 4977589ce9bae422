"""Probe: repeat small multi-device products and require bitwise-identical results
(the product is deterministic), bisecting over fetch-ahead and task order.  Dev tool."""
import json, sys
import numpy as np
import paper_1511_04348_b200 as tr
from oracle import tilerun_oracle as O

meta = json.loads(open("tests/golden/runs.json").read()); arr = np.load("tests/golden/runs.npz")
cases = [n for n in meta if n not in ("session_reuse", "transpose")]
for fa in (True, False):
    for order in ("auto", "row-major"):
        bad = 0
        for rep in range(12):
            for name in cases:
                m = meta[name]
                a, b, cref = arr[name + "_a"], arr[name + "_b"], arr[name + "_c"]
                rt = tr.Runtime(tr.homogeneous_machine(m["devices"], capacity_tiles=m["capacity"]), m["tile"],
                                coherence=m["coherence"], fetch_ahead=fa)
                rt.set_order(order)
                c, s = rt.multiply(a, b, a_uid="A", b_uid="B", c_uid="C")
                rt.close()
                err = float(np.linalg.norm(c - cref) / np.linalg.norm(cref))
                if err > 1e-5:
                    bad += 1
                    if bad <= 3:
                        d = np.abs(c - cref)
                        i, j = np.unravel_index(np.argmax(d), d.shape)
                        print(f"  BAD fa={fa} order={order} {name} rep {rep}: err {err:.3e} worst ({i},{j}) "
                              f"got {c[i,j]:.6g} want {cref[i,j]:.6g}", flush=True)
        print(f"fetch_ahead={fa} order={order}: {bad} bad of {12*len(cases)}", flush=True)
