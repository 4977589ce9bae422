"""Probe: directory-lock cost (tr_session_lock_stats) with 1, 4 and 8 logical
devices (worker threads) on one GPU -- cold cfg2-shaped product from pinned host
(every fill, peer copy and launch goes through the lock) and a warm one."""
import sys
import numpy as np
import torch
import paper_1511_04348_b200 as tr

n = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
T = int(sys.argv[2]) if len(sys.argv) > 2 else 2048
a = tr.matrix.pinned_empty((n, n), np.float32)
b = tr.matrix.pinned_empty((n, n), np.float32)
g = torch.Generator(device="cuda").manual_seed(1)
for m in (a, b):
    for r in range(0, n, 4096):
        m[r:r + 4096] = torch.randn((min(4096, n - r), n), device="cuda", generator=g).cpu().numpy()
for nd in (1, 4, 8):
    mach = tr.homogeneous_machine(nd, dtype=np.float32, gpus=[0] * nd)
    for rep in range(2):
        with tr.Runtime(mach, T) as rt:
            rt.lock_stats(reset=True)
            torch.cuda.synchronize()
            _, s = rt.multiply(a, b, a_uid="A", b_uid="B", c_uid="C")
            cold = rt.lock_stats(reset=True)
            _, s2 = rt.multiply(a, b, a_uid="A", b_uid="B", c_uid="C2")
            warm = rt.lock_stats(reset=True)
        if rep:
            print(f"devices {nd}: cold wall {s.wall_elapsed * 1e3:.1f} ms, lock held {cold['held_s'] * 1e3:.2f} ms "
                  f"({cold['held_s'] / s.wall_elapsed:.1%}), waited {cold['waited_s'] * 1e3:.2f} ms, "
                  f"{cold['acquisitions']} acq, max hold {cold['max_hold_us']:.0f} us, l2 {s.cache.l2_hits}, "
                  f"served {[d.peer_copies_served for d in s.devices.values()]} | warm wall {s2.wall_elapsed * 1e3:.1f} ms, "
                  f"held {warm['held_s'] * 1e3:.2f} ms, waited {warm['waited_s'] * 1e3:.2f} ms, {warm['acquisitions']} acq",
                  flush=True)
