"""The simulated engine (mode="sim", TR_FLAG_SIM; reference scheduler.py:432-464)
against the reference's own sim runs (tests/golden/sim_runs.json, made by
tests/golden/make_golden.py): makespans and steal times bit for bit, the same
steal events, per-device task counts and cache counters, and clocks that
persist across the calls of a session."""

import json
from pathlib import Path

import numpy as np
import pytest

from paper_1511_04348_b200 import Machine, Runtime, homogeneous_machine, run

G = json.loads((Path(__file__).resolve().parent / "golden" / "sim_runs.json").read_text())
MACHINES = {k: Machine.from_dict(v) for k, v in G["machines"].items()}


def check(stats, want, rt=None):
    assert stats.makespan.hex() == want["makespan"], (stats.makespan, float.fromhex(want["makespan"]))
    got_ev = [[e.thief, e.victim, e.task_id, e.time.hex()] for e in stats.steal_events]
    assert got_ev == want["steal_events"]
    assert {str(d): v for d, v in stats.tasks_by_device.items()} == want["tasks_by_device"]
    assert stats.cache.as_dict() == want["cache"]
    assert {str(d): s.as_dict() for d, s in stats.cache_per_device.items()} == want["per_device"]
    assert [stats.grid_rows, stats.grid_cols, stats.k_steps] == want["grid"]
    if rt is not None:
        assert rt.sim_now().hex() == want["sim_now"]


@pytest.mark.parametrize("name", sorted(G["runs"]))
def test_sim_run_matches_reference(name):
    case = G["runs"][name]
    a, b = np.zeros((case["m"], case["k"])), np.zeros((case["k"], case["n"]))
    c, stats = run(MACHINES[case["machine"]], a, b, case["tile"], mode="sim", coherence=case["coherence"],
                   steal=case["steal"], compute=False)
    assert c is None and stats.mode == "sim"
    check(stats, case["stats"])


@pytest.mark.parametrize("mk", sorted(G["sessions"]))
def test_sim_session_clocks_persist(mk):
    rt = Runtime(MACHINES[mk], 4, mode="sim", compute=False)
    x, w, dy = np.zeros((20, 12)), np.zeros((12, 16)), np.zeros((20, 16))
    calls = [dict(a=x, b=w, a_uid="X", b_uid="W", c_uid="Y"),
             dict(a=x, b=dy, transpose_a=True, a_uid="X", b_uid="DY", c_uid="DW"),
             dict(a=dy, b=w, transpose_b=True, a_uid="DY", b_uid="W", c_uid="DX"),
             dict(a=x, b=w, a_uid="X", b_uid="W", c_uid="Y2")]
    for kw, want in zip(calls, G["sessions"][mk]):
        _, s = rt.multiply(**kw)
        check(s, want, rt)
    rt.close()


def test_sim_rejects_batches_and_needs_positive_rates():
    rt = Runtime(homogeneous_machine(2), 4, mode="sim", compute=False)
    with pytest.raises(ValueError):
        rt.multiply_batch([])
    rt.close()
    from paper_1511_04348_b200 import DeviceSpec, ProximityMatrix

    from paper_1511_04348_b200.errors import ConfigError

    with pytest.raises((ConfigError, ValueError)):
        bad = Machine([DeviceSpec(0, flops_per_unit=0.0)], ProximityMatrix.uniform(1))
        Runtime(bad, 4, mode="sim", compute=False)


@pytest.mark.parametrize("name", ["plain", "bypass", "template"])
def test_cli_sweep_sim_is_byte_identical(tmp_path, name):
    """`sweep` (default --mode sim, like the reference's) reproduces the reference CLI's table byte for byte."""
    from paper_1511_04348_b200 import cli, save_machine

    extra = []
    if name == "bypass":
        extra = ["--no-coherence"]
    elif name == "template":
        dev = tmp_path / "devices.json"
        save_machine(dev, Machine.from_dict(G["sweep_devices"]))
        extra = ["--devices", str(dev)]
    out = tmp_path / "sweep.csv"
    assert cli.main(["sweep", "--sizes", "8,16,20", "--device-counts", "2,3", "--tile-size", "4", "--seed", "3",
                     "--out", str(out), *extra]) == 0
    assert out.read_text() == G["sweeps"][name]


def test_cli_sweep_speedup_curve_shape(tmp_path):
    """The reference's acceptance criterion 4 (test_acceptance.py:145-168): on the
    simulated sweep the 4-device speedup rises to its peak and stays within 5 %."""
    import csv

    from paper_1511_04348_b200 import cli

    dev = tmp_path / "template.json"
    dev.write_text('{"devices": [{"id": 0, "flops_per_unit": 1000.0, "host_bandwidth": 256.0}]}')
    out = tmp_path / "sweep.csv"
    assert cli.main(["sweep", "--sizes", "32,64,128,256,320", "--device-counts", "1,4", "--tile-size", "16",
                     "--devices", str(dev), "--out", str(out)]) == 0
    sp = [float(r["speedup"]) for r in csv.DictReader(out.read_text().splitlines()) if r["devices"] == "4"]
    assert len(sp) == 5
    peak = int(np.argmax(sp))
    assert all(sp[i] <= sp[i + 1] + 1e-12 for i in range(peak))
    assert all(s >= 0.95 * sp[peak] for s in sp[peak:])
