"""Probe: the bench's cfg5 hetero leg alone (args as bench.py, e.g. --tile 2048)."""
import json, sys
import torch
import paper_1511_04348_b200 as tr
sys.path.insert(0, ".")
import bench
args = bench.parse(sys.argv[1:])
r = bench.bench_wide_hetero(args, tr, torch, [0])
r.pop("loss", None)
print(json.dumps(r), flush=True)
