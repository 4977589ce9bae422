"""Summarise a CUPTI trace (tools/probe_mlp_timeline.py): per-kernel time and
the GPU-idle gaps of the last step.  Dev tool."""
import json, sys, collections
ev = json.load(open(sys.argv[1]))["traceEvents"]
k = sorted([e for e in ev if e.get("cat") in ("kernel", "gpu_memcpy", "gpu_memset") and "dur" in e], key=lambda e: e["ts"])
t0, t1 = k[0]["ts"], max(e["ts"] + e["dur"] for e in k)
span = (t1 - t0) / 2  # two steps
agg = collections.defaultdict(lambda: [0, 0.0])
for e in k:
    n = e["name"].replace("(anonymous namespace)::", "").split("(")[0][:90]
    agg[n][0] += 1
    agg[n][1] += e["dur"] / 2
busy = 0.0
cur0, cur1 = k[0]["ts"], k[0]["ts"] + k[0]["dur"]
gaps = []
for e in k[1:]:
    if e["ts"] > cur1:
        busy += cur1 - cur0
        gaps.append((e["ts"] - cur1, e["name"][:50]))
        cur0, cur1 = e["ts"], e["ts"] + e["dur"]
    else:
        cur1 = max(cur1, e["ts"] + e["dur"])
busy += cur1 - cur0
print(f"per step: span {span / 1e3:.2f} ms, GPU busy {busy / 2 / 1e3:.2f} ms")
for n, (c, t) in sorted(agg.items(), key=lambda x: -x[1][1])[:16]:
    print(f"{t / 1e3:8.3f} ms {c / 2:6.0f}x  {n}")
gaps.sort(reverse=True)
print("largest gaps (us):", [(round(g, 1), n) for g, n in gaps[:8]])
