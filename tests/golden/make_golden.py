"""Generate golden vectors by running the REAL reference (tilerun) in this container.

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden.py

Imports /root/reference/pkg/src/tilerun (read-only; pure Python + numpy) and
writes small fixtures next to this script.  The GPU box never has the
reference: tests read only these committed files.

Fixtures
  tiles.npz        known-answer products (tests/test_tiles.py:147-195) and random
                   reference_gemm / accumulate_product results (f64, bitwise)
  plans.json       plan() task lists for several shapes (scheduler.py:165-197)
  runs.npz/.json   full run() products + CacheStats/RunStats for small configs
                   (sim engine: deterministic), incl. capacity-3, bypass, multi-device
  directory.json   random op sequences on CacheDirectory and its answers
  ann.npz          DenseBackend MLP: forward/backward/grad values and training
                   trajectories (xor 50 steps; per-layer-scaled 24-40-40-6 net)
  sim_runs.json    the reference's SIMULATED engine (scheduler.py:432-464): makespans
                   (float.hex, bitwise), sim clocks, steal events with times, per-device
                   task counts and counters for heterogeneous / bounded / host-worker /
                   bypass / no-steal / non-uniform-fabric machines and multi-call sessions
  cfg1.npz         cfg1 (N=2048, T=512, float32 machine): the reference's own
                   threaded run -- stats, sampled output blocks and per-tile checksums,
                   plus the float64 reference_gemm checksums of the same inputs
"""

from __future__ import annotations

import json
import sys
import time
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
sys.path.insert(0, "/root/reference/pkg/src")

import tilerun as ref  # noqa: E402
from tilerun import ann as ref_ann  # noqa: E402
from tilerun.scheduler import plan as ref_plan  # noqa: E402


def int_matrix(rng, rows, cols, lo=-4, hi=4):
    return rng.integers(lo, hi + 1, size=(rows, cols)).astype(np.float64)


def stats_dict(stats):
    return {
        "cache": stats.cache.as_dict(),
        "per_device": {str(d): s.as_dict() for d, s in stats.cache_per_device.items()},
        "tasks_by_device": {str(d): v for d, v in stats.tasks_by_device.items()},
        "total_tasks": stats.total_tasks,
        "grid": [stats.grid_rows, stats.grid_cols, stats.k_steps],
        "steals": len(stats.steal_events),
    }


def gen_tiles():
    out = {}
    out["hand_a"] = np.array([[1.0, 2.0], [3.0, 4.0]])
    out["hand_b"] = np.array([[5.0, 6.0], [7.0, 8.0]])
    out["hand_c"] = ref.gemm_tile(out["hand_a"], out["hand_b"], np.zeros((2, 2)))
    out["acc_c"] = ref.gemm_tile(np.array([[1.0, 1.0]]), np.array([[2.0], [3.0]]), np.array([[10.0]]))
    rng = np.random.default_rng(1234)
    shapes = [(1, 1, 1), (4, 5, 3), (9, 11, 6), (17, 33, 9), (30, 18, 25), (64, 64, 64), (5, 130, 7)]
    for idx, (m, k, n) in enumerate(shapes):
        a = rng.standard_normal((m, k))
        b = rng.standard_normal((k, n))
        out[f"rand{idx}_a"], out[f"rand{idx}_b"] = a, b
        out[f"rand{idx}_c"] = ref.reference_gemm(a, b)
        a32, b32 = a.astype(np.float32), b.astype(np.float32)
        out[f"rand{idx}_a32"], out[f"rand{idx}_b32"] = a32, b32
        out[f"rand{idx}_c32"] = ref.reference_gemm(a32, b32)
        acc = rng.standard_normal((m, n))
        out[f"rand{idx}_acc0"] = acc.copy()
        out[f"rand{idx}_acc"] = ref.accumulate_product(a, b, acc)
    census = []
    for n_ in range(1, 14):
        for t in range(1, n_ + 2):
            tm = ref.partition(np.zeros((n_, n_ + 3)), t)
            census.append([n_, n_ + 3, t, tm.grid_rows, tm.grid_cols, tm.full_tile_count, tm.ragged_tile_count])
    out["census"] = np.array(census, dtype=np.int64)
    np.savez_compressed(HERE / "tiles.npz", **out)


def gen_plans():
    cases = []
    for (m, k, n, t) in [(4, 4, 4, 2), (6, 4, 6, 2), (2, 2, 2, 4), (7, 5, 3, 2), (13, 9, 21, 4), (5, 5, 5, 1),
                         (8192, 784, 8192, 4096), (2048, 2048, 2048, 512), (32768, 32768, 32768, 4096)]:
        p = ref_plan(ref.partition(np.zeros((m, k)) if m * k < 1e7 else np.zeros((1, 1)), t),
                     ref.partition(np.zeros((k, n)) if k * n < 1e7 else np.zeros((1, 1)), t)) \
            if m * k < 1e7 and k * n < 1e7 else None
        if p is not None:
            tasks = [[tk.task_id, tk.row, tk.col, tk.k_steps] for tk in p.tasks]
            grid = [p.grid_rows, p.grid_cols, p.k_steps]
        else:  # shapes too big to allocate here: the planner only needs the grid
            gr, gc, ks = -(-m // t), -(-n // t), -(-k // t)
            tasks = [[i * gc + j, i, j, ks] for i in range(gr) for j in range(gc)]
            grid = [gr, gc, ks]
        cases.append({"m": m, "k": k, "n": n, "tile": t, "grid": grid, "tasks": tasks})
    (HERE / "plans.json").write_text(json.dumps(cases))


RUN_CASES = [
    # name, m, k, n, tile, devices, capacity, coherence, kind, seed
    ("int_12_t4_1dev", 12, 12, 12, 4, 1, None, True, "int", 1),
    ("int_12_t4_3dev", 12, 12, 12, 4, 3, None, True, "int", 1),
    ("float_30x18x25_t7_2dev", 30, 18, 25, 7, 2, None, True, "float", 2),
    ("int_24_t4_cap6_3dev", 24, 24, 24, 4, 3, 6, True, "int", 4),
    ("int_16_t4_cap3_1dev", 16, 16, 16, 4, 1, 3, True, "int", 5),
    ("int_16_t4_cap3_2dev", 16, 16, 16, 4, 2, 3, True, "int", 5),
    ("int_24_t4_g6_1dev", 24, 24, 24, 4, 1, None, True, "int", 8),
    ("int_24_t4_g6_3dev", 24, 24, 24, 4, 3, None, True, "int", 8),
    ("int_24_t4_bypass_2dev", 24, 24, 24, 4, 2, None, False, "int", 8),
    ("float_ragged_37x53x29_t8", 37, 53, 29, 8, 2, None, True, "float", 9),
    ("int_40_t5_cap3_2dev", 40, 40, 40, 5, 2, 3, True, "int", 10),
    ("float_t1_9x7x5", 9, 7, 5, 1, 2, None, True, "float", 11),
    ("float_512x384x512_t16", 512, 384, 512, 16, 2, None, True, "uniform", 12),
]


def gen_runs():
    arrays, meta = {}, {}
    for name, m, k, n, t, ndev, cap, coh, kind, seed in RUN_CASES:
        rng = np.random.default_rng(seed)
        if kind == "int":
            a, b = int_matrix(rng, m, k), int_matrix(rng, k, n)
        elif kind == "uniform":
            a, b = rng.uniform(0.0, 1.0, size=(m, k)), rng.uniform(0.0, 1.0, size=(k, n))
        else:
            a, b = rng.standard_normal((m, k)), rng.standard_normal((k, n))
        machine = ref.homogeneous_machine(ndev, capacity_tiles=cap)
        c, stats = ref.run(machine, a, b, tile_size=t, mode="sim", coherence=coh)
        arrays[name + "_a"], arrays[name + "_b"], arrays[name + "_c"] = a, b, c
        meta[name] = {"m": m, "k": k, "n": n, "tile": t, "devices": ndev, "capacity": cap, "coherence": coh,
                      "kind": kind, "stats": stats_dict(stats)}
    # session reuse (tests/test_scheduler.py:413-422) and transposed identity (425-438)
    rng = np.random.default_rng(17)
    a, b = int_matrix(rng, 16, 16), int_matrix(rng, 16, 16)
    rt = ref.Runtime(ref.homogeneous_machine(1), tile_size=4)
    _, s1 = rt.multiply(a, b, a_uid="X", b_uid="W")
    _, s2 = rt.multiply(a, b, a_uid="X", b_uid="W")
    meta["session_reuse"] = {"first": stats_dict(s1), "second": stats_dict(s2)}
    arrays["session_reuse_a"], arrays["session_reuse_b"] = a, b
    rng = np.random.default_rng(18)
    x, w, y = rng.standard_normal((12, 8)), rng.standard_normal((8, 8)), rng.standard_normal((12, 8))
    rt = ref.Runtime(ref.homogeneous_machine(1), tile_size=4)
    rt.multiply(x, w, a_uid="X", b_uid="W")
    before = rt.directory.stats()
    c, _ = rt.multiply(x, y, transpose_a=True, a_uid="X", b_uid="Y2")
    after = rt.directory.stats()
    arrays["transpose_x"], arrays["transpose_w"], arrays["transpose_y"], arrays["transpose_c"] = x, w, y, c
    meta["transpose"] = {"host_fetch_delta": after.host_fetches - before.host_fetches}
    np.savez_compressed(HERE / "runs.npz", **arrays)
    (HERE / "runs.json").write_text(json.dumps(meta, indent=1))


def key_of(t):
    return ref.TileKey(t[0], t[1], t[2])


def gen_directory():
    seqs = []
    rng = np.random.default_rng(99)
    for trial in range(16):
        n = int(rng.integers(1, 4))
        caps = [int(rng.integers(3, 7)) if rng.integers(0, 3) else None for _ in range(n)]
        hops = rng.integers(1, 4, size=(n, n))
        hops = np.triu(hops, 1)
        hops = hops + hops.T
        policy = "fifo" if trial % 5 == 4 else "lru"
        enabled = trial % 7 != 6
        devs = [ref.DeviceSpec(i, capacity_tiles=caps[i]) for i in range(n)]
        m = ref.Machine(devs, ref.ProximityMatrix(hops, np.full((n, n), 10.0)))
        d = ref.CacheDirectory(m, enabled=enabled, policy=policy, debug=False)
        universe = [("t", i, j) for i in range(3) for j in range(4)]
        ops = []
        for _ in range(250):
            op = ["lookup", "admit", "pin", "unpin", "acquire", "release", "admit_out", "release_out"][
                int(rng.integers(0, 8))]
            dev = int(rng.integers(0, n))
            k = universe[int(rng.integers(0, len(universe)))]
            key = key_of(k)
            rec = {"op": op, "dev": dev, "key": list(k)}
            try:
                if op == "lookup":
                    r = d.lookup(dev, key)
                    rec["out"] = [r.level.value, r.owner]
                elif op == "admit":
                    rec["out"] = [list(e) for e in d.admit(dev, key)]
                elif op == "pin":
                    d.pin(dev, key)
                elif op == "unpin":
                    d.unpin(dev, key)
                elif op == "acquire":
                    r = d.acquire_input(dev, key, 7 + k[1] * 4 + k[2])
                    rec["out"] = [r.level.value, r.source, r.nbytes_moved, [list(e) for e in r.evicted]]
                elif op == "release":
                    d.release_input(dev, key)
                elif op == "admit_out":
                    rec["out"] = [list(e) for e in d.admit_output(dev, key)]
                elif op == "release_out":
                    d.release_output(dev, key, 64)
                rec["err"] = None
            except ref.CapacityError:
                rec["err"] = "capacity"
            except ValueError:
                rec["err"] = "value"
            except KeyError:
                rec["err"] = "key"  # reference raises KeyError when releasing a non-resident output
            rec["residents"] = [[list(x) for x in d.residents(i)] for i in range(n)]
            rec["stats"] = d.stats().as_dict()
            ops.append(rec)
        seqs.append({"caps": caps, "hops": hops.tolist(), "policy": policy, "enabled": enabled, "ops": ops,
                     "per_device": {str(i): s.as_dict() for i, s in d.stats_per_device().items()}})
    (HERE / "directory.json").write_text(json.dumps(seqs))


def gen_ann():
    out = {}
    # xor trajectory, 50 steps (tests/test_ann.py:411-424)
    rng = np.random.default_rng(0)
    net = ref_ann.Network.from_sizes([2, 8, 1], rng, activation="sigmoid")
    out["xor_w0"] = [l.weights.copy() for l in net.layers][0]
    x, target = ref_ann.xor_dataset()
    losses = [ref_ann.train_step(net, x, target, 0.5, ref_ann.DenseBackend()) for _ in range(50)]
    out["xor_losses"] = np.array(losses)
    for i, l in enumerate(net.layers):
        out[f"xor_final_w{i}"], out[f"xor_final_b{i}"] = l.weights, l.bias
    # per-layer scaled net (scale = 1/sqrt(fan_in)), 10 steps, sigmoid and relu
    for act in ("sigmoid", "relu"):
        rng = np.random.default_rng(5)
        sizes = [24, 40, 40, 6]
        layers = [ref_ann.Layer.random(sizes[i], sizes[i + 1], rng, activation=act, scale=1 / np.sqrt(sizes[i]),
                                       tag=f"layer{i}") for i in range(3)]
        net = ref_ann.Network(layers)
        for i, l in enumerate(net.layers):
            out[f"{act}_init_w{i}"], out[f"{act}_init_b{i}"] = l.weights.copy(), l.bias.copy()
        x, target = ref_ann.random_regression(rng, 16, 24, 6)
        out[f"{act}_x"], out[f"{act}_t"] = x, target
        loss, grads = ref_ann.loss_gradients(net, x, target, ref_ann.DenseBackend())
        out[f"{act}_loss0"] = np.array([loss])
        for i, (gw, gb) in enumerate(grads):
            out[f"{act}_gw{i}"], out[f"{act}_gb{i}"] = gw, gb
        traj = [ref_ann.train_step(net, x, target, 0.1, ref_ann.DenseBackend()) for _ in range(10)]
        out[f"{act}_losses"] = np.array(traj)
        for i, l in enumerate(net.layers):
            out[f"{act}_final_w{i}"], out[f"{act}_final_b{i}"] = l.weights, l.bias
    np.savez_compressed(HERE / "ann.npz", **out)


def tile_checksums(c, t):
    g = -(-c.shape[0] // t)
    return np.array([[c[i * t:(i + 1) * t, j * t:(j + 1) * t].sum(dtype=np.float64) for j in range(g)]
                     for i in range(g)])


def _sim_record(stats, rt=None):
    rec = stats_dict(stats)
    rec["makespan"] = float(stats.makespan).hex()
    rec["steal_events"] = [[e.thief, e.victim, e.task_id, float(e.time).hex()] for e in stats.steal_events]
    if rt is not None:
        rec["sim_now"] = float(rt.sim_now()).hex()
    return rec


def _sim_machines():
    D = ref.DeviceSpec
    out = {}
    out["homog1"] = ref.homogeneous_machine(1)
    out["homog3"] = ref.homogeneous_machine(3)
    out["hetero_1234"] = ref.Machine([D(i, flops_per_unit=1000.0 * (i + 1), host_bandwidth=8192.0) for i in range(4)],
                                     ref.ProximityMatrix.uniform(4, bandwidth=32768.0))
    out["bounded_cap6"] = ref.homogeneous_machine(3, capacity_tiles=6)
    out["cap3_2dev"] = ref.homogeneous_machine(2, capacity_tiles=3)
    out["host_worker_mix"] = ref.Machine(
        [D(0, flops_per_unit=2000.0, host_bandwidth=4096.0), D(1, flops_per_unit=1500.0, host_bandwidth=8192.0, slots=2),
         D(2, kind="host-worker", flops_per_unit=300.0, host_bandwidth=1.0, subtile_factor=2)],
        ref.ProximityMatrix.uniform(3, bandwidth=16384.0))
    hops = np.array([[0, 1, 2, 2], [1, 0, 2, 2], [2, 2, 0, 1], [2, 2, 1, 0]])
    bw = np.array([[1.0, 50000.0, 9000.0, 9000.0], [50000.0, 1.0, 9000.0, 9000.0],
                   [9000.0, 9000.0, 1.0, 50000.0], [9000.0, 9000.0, 50000.0, 1.0]])
    out["fabric_latency"] = ref.Machine([D(i, flops_per_unit=1000.0 + 250.0 * i, host_bandwidth=6000.0 + 1000.0 * i,
                                           slots=3 + (i % 2)) for i in range(4)],
                                        ref.ProximityMatrix(hops, bw), transfer_latency=0.37)
    out["float32_homog2"] = ref.homogeneous_machine(2, dtype=np.float32)
    return out


SIM_CASES = [
    # name, machine, m, k, n, tile, coherence, steal
    ("homog1_12_t4", "homog1", 12, 12, 12, 4, True, True),
    ("homog3_24_t4", "homog3", 24, 24, 24, 4, True, True),
    ("hetero_64_t8", "hetero_1234", 64, 64, 64, 8, True, True),
    ("hetero_64_t8_nosteal", "hetero_1234", 64, 64, 64, 8, True, False),
    ("bounded_24_t4", "bounded_cap6", 24, 24, 24, 4, True, True),
    ("cap3_16_t4", "cap3_2dev", 16, 16, 16, 4, True, True),
    ("hostmix_30x18x25_t7", "host_worker_mix", 30, 18, 25, 7, True, True),
    ("fabric_40_t5", "fabric_latency", 40, 40, 40, 5, True, True),
    ("fabric_40_t5_bypass", "fabric_latency", 40, 40, 40, 5, False, True),
    ("ragged_37x53x29_t8", "homog3", 37, 53, 29, 8, True, True),
    ("t1_9x7x5", "float32_homog2", 9, 7, 5, 1, True, True),
]


def gen_sim():
    machines = _sim_machines()
    out = {"machines": {k: m.to_dict() for k, m in machines.items()}, "runs": {}, "sessions": {}}
    for name, mk, m, k, n, t, coh, steal in SIM_CASES:
        rng = np.random.default_rng(len(name))
        a, b = int_matrix(rng, m, k), int_matrix(rng, k, n)
        _, stats = ref.run(machines[mk], a, b, tile_size=t, mode="sim", coherence=coh, steal=steal)
        out["runs"][name] = {"machine": mk, "m": m, "k": k, "n": n, "tile": t, "coherence": coh, "steal": steal,
                             "stats": _sim_record(stats)}
    # sessions: clocks and residency persist across calls (an ANN-like sequence
    # with a transposed reuse of X and a re-multiply that hits L1 everywhere)
    for mk in ("homog3", "fabric_latency", "hetero_1234"):
        rng = np.random.default_rng(7)
        x, w, dy = int_matrix(rng, 20, 12), int_matrix(rng, 12, 16), int_matrix(rng, 20, 16)
        rt = ref.Runtime(machines[mk], tile_size=4)
        seq = []
        _, s = rt.multiply(x, w, a_uid="X", b_uid="W", c_uid="Y")
        seq.append(_sim_record(s, rt))
        _, s = rt.multiply(x, dy, transpose_a=True, a_uid="X", b_uid="DY", c_uid="DW")
        seq.append(_sim_record(s, rt))
        _, s = rt.multiply(dy, w, transpose_b=True, a_uid="DY", b_uid="W", c_uid="DX")
        seq.append(_sim_record(s, rt))
        _, s = rt.multiply(x, w, a_uid="X", b_uid="W", c_uid="Y2")
        seq.append(_sim_record(s, rt))
        out["sessions"][mk] = seq
    # the reference CLI's sweep table (cli.py:131-189, sim engine), byte for byte
    import tempfile

    from tilerun import cli as ref_cli

    sweeps = {}
    with tempfile.TemporaryDirectory() as td:
        dev = Path(td) / "devices.json"
        ref.save_machine(dev, machines["fabric_latency"])
        out["sweep_devices"] = machines["fabric_latency"].to_dict()
        for name, extra in (("plain", []), ("bypass", ["--no-coherence"]), ("template", ["--devices", str(dev)])):
            path = Path(td) / f"{name}.csv"
            ref_cli.main(["sweep", "--sizes", "8,16,20", "--device-counts", "2,3", "--tile-size", "4", "--seed", "3",
                          "--out", str(path), *extra])
            sweeps[name] = path.read_text()
    out["sweeps"] = sweeps
    (HERE / "sim_runs.json").write_text(json.dumps(out, indent=1))


def gen_cfg1():
    n, t = 2048, 512
    a = np.random.default_rng(1).standard_normal((n, n)).astype(np.float32)
    b = np.random.default_rng(2).standard_normal((n, n)).astype(np.float32)
    t0 = time.perf_counter()
    c32, stats = ref.run(ref.homogeneous_machine(4, dtype=np.float32), a, b, t, mode="threaded")
    wall = time.perf_counter() - t0
    rows = np.array([0, 1, 511, 512, 1023, 1500, 2046, 2047])
    cols = np.array([0, 7, 510, 513, 1024, 1777, 2040, 2047])
    c64 = ref.reference_gemm(a.astype(np.float64), b.astype(np.float64))
    np.savez_compressed(
        HERE / "cfg1.npz",
        a_sum=np.array([a.sum(dtype=np.float64), (a.astype(np.float64) ** 2).sum()]),
        b_sum=np.array([b.sum(dtype=np.float64), (b.astype(np.float64) ** 2).sum()]),
        rows=rows, cols=cols,
        c32_block=c32[np.ix_(rows, cols)], c64_block=c64[np.ix_(rows, cols)],
        c32_tiles=tile_checksums(c32.astype(np.float64), t), c64_tiles=tile_checksums(c64, t),
        c64_fro=np.array([np.linalg.norm(c64)]),
        stats=np.array([stats.cache.host_fetches, stats.cache.bytes_host, stats.cache.l1_hits + stats.cache.l2_hits,
                        stats.cache.writebacks, stats.cache.bytes_writeback, stats.total_tasks]),
        ref_wall=np.array([wall]),
    )


if __name__ == "__main__":
    which = sys.argv[1:] or ["tiles", "plans", "runs", "directory", "ann", "sim", "cfg1"]
    for w in which:
        t0 = time.perf_counter()
        globals()[f"gen_{w}"]()
        print(f"{w}: {time.perf_counter() - t0:.1f}s")
