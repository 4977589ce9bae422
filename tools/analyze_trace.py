"""Dev tool: summarise a torch.profiler chrome trace -- GPU time per kernel name,
busy union, idle gaps (largest first)."""
import json, sys
from collections import defaultdict

ev = json.load(open(sys.argv[1]))["traceEvents"]
k = [e for e in ev if e.get("cat") in ("kernel", "gpu_memcpy", "gpu_memset") and "dur" in e]
k.sort(key=lambda e: e["ts"])
per = defaultdict(lambda: [0, 0.0])
for e in k:
    n = e["name"][:70]
    per[n][0] += 1
    per[n][1] += e["dur"]
t0, t1 = k[0]["ts"], max(e["ts"] + e["dur"] for e in k)
busy, cur_s, cur_e, gaps = 0.0, None, None, []
for e in k:
    s, f = e["ts"], e["ts"] + e["dur"]
    if cur_e is None or s > cur_e:
        if cur_e is not None:
            busy += cur_e - cur_s
            gaps.append((s - cur_e, cur_e - t0, e["name"][:50]))
        cur_s, cur_e = s, f
    else:
        cur_e = max(cur_e, f)
busy += cur_e - cur_s
print(f"span {(t1 - t0) / 1e3:.2f} ms, busy union {busy / 1e3:.2f} ms, events {len(k)}")
for n, (c, d) in sorted(per.items(), key=lambda x: -x[1][1])[:25]:
    print(f"{d / 1e3:9.3f} ms {c:5d}  {n}")
gaps.sort(reverse=True)
print("largest gaps (us, at ms, next):")
for g in gaps[:15]:
    print(f"  {g[0]:8.1f}  {g[1] / 1e3:8.3f}  {g[2]}")
if len(sys.argv) > 2:  # per-event listing of the last N events
    print("events:")
    for e in k[-int(sys.argv[2]):]:
        a = e.get("args", {})
        print(f"  {(e['ts'] - t0) / 1e3:8.3f} {e['dur']:9.1f}us grid={a.get('grid')} {e['name'][:60]}")
