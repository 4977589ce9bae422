"""Probe: the bench's inhomogeneous leg alone (shares vs standalone rates)."""
import json, sys
import torch
import paper_1511_04348_b200 as tr
sys.path.insert(0, ".")
import bench
for prec in ("fp32acc",):
    r = bench.bench_inhomogeneous(tr, torch, prec, 0)
    print(json.dumps(r), flush=True)
