"""Probe: run single bench legs by name (dev tool): python tools/probe_legs.py coherence inhomogeneous"""
import json, sys
import torch
import paper_1511_04348_b200 as tr
sys.path.insert(0, ".")
import bench
args = bench.parse([])
for leg in sys.argv[1:]:
    if leg == "coherence":
        r = bench.bench_coherence(args, tr, torch, 0)
    elif leg == "inhomogeneous":
        r = bench.bench_inhomogeneous(tr, torch, args.precision, 0)
    print(leg, json.dumps(r), flush=True)
    tr.release_cached_memory()
    torch.cuda.empty_cache()
