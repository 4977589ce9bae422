"""Host-side scheduling logic on CPU: tile geometry, the planner, reservation
stations and stealing, and whole products in the schedule-only ("dryrun")
session mode compared with the reference's exact counting identities and with
golden CacheStats recorded from the reference (tests/golden/runs.json)."""

import json
from pathlib import Path

import numpy as np
import pytest

from oracle import tilerun_oracle as O
from paper_1511_04348_b200 import (ConfigError, DeviceSpec, Machine, MichaelScottQueue, ProximityMatrix,
                                   ReservationStation, Runtime, TaskState, decode_task, encode_task,
                                   homogeneous_machine, partition, plan, reassemble, steal_task,
                                   write_report_csv, write_report_json)

G = Path(__file__).resolve().parent / "golden"


# ----------------------------------------------------------------- tiles (tiles.py)


def test_partition_and_census():
    tm = partition(np.arange(25, dtype=float).reshape(5, 5), 2)
    assert tm.grid_shape == (3, 3) and tm.full_tile_count == 4 and tm.ragged_tile_count == 5
    assert tm.tile_shape(0, 2) == (2, 1) and tm.tile_shape(2, 2) == (1, 1)
    for n in range(1, 20):
        for t in range(1, n + 2):
            tm = partition(np.zeros((n, n)), t)
            assert (tm.full_tile_count, tm.ragged_tile_count) == O.census(n, n, t)
    with pytest.raises(ValueError):
        partition(np.ones((2, 2)), 0)


def test_reassemble_roundtrip():
    rng = np.random.default_rng(123)
    for _ in range(40):
        m = rng.standard_normal((int(rng.integers(1, 30)), int(rng.integers(1, 30))))
        t = int(rng.integers(1, 12))
        tm = partition(m, t)
        assert np.array_equal(reassemble(tm), m)
        for i, j in tm.coords():
            blk = tm.tile(i, j)
            assert np.array_equal(blk, m[i * t:i * t + blk.shape[0], j * t:j * t + blk.shape[1]])


def test_task_codec():
    assert encode_task(1, 2, 3) == 5 and tuple(decode_task(5, 3, grid_rows=2)) == (1, 2)
    rng = np.random.default_rng(5)
    for _ in range(30):
        gr, gc = int(rng.integers(1, 12)), int(rng.integers(1, 12))
        ids = [encode_task(i, j, gc) for i in range(gr) for j in range(gc)]
        assert sorted(ids) == list(range(gr * gc))
        for tid in ids:
            assert encode_task(*decode_task(tid, gc, grid_rows=gr), gc) == tid
    for bad in [(6, 3, 2), (-1, 3, None), (0, 0, None)]:
        with pytest.raises(ValueError):
            decode_task(*bad)


# ----------------------------------------------------------------- plan (scheduler.py:165-197)


def test_plan_matches_reference_task_lists():
    for case in json.loads((G / "plans.json").read_text()):
        m, k, n, t = case["m"], case["k"], case["n"], case["tile"]
        if m * k > 1e7 or k * n > 1e7:
            continue
        p = plan(partition(np.zeros((m, k)), t), partition(np.zeros((k, n)), t))
        assert [[x.task_id, x.row, x.col, x.k_steps] for x in p.tasks] == case["tasks"]
        assert [p.grid_rows, p.grid_cols, p.k_steps] == case["grid"]
        assert p.queue.drain() == list(range(p.total_tasks))
        assert all(x.state is TaskState.QUEUED for x in p.tasks)
        assert not p.c.tiled.base.any()


def test_plan_rejects_mismatches():
    with pytest.raises(ValueError):
        plan(partition(np.zeros((4, 4)), 2), partition(np.zeros((5, 4)), 2))
    with pytest.raises(ValueError):
        plan(partition(np.zeros((4, 4)), 2), partition(np.zeros((4, 4)), 3))


# ----------------------------------------------------------------- stations (scheduler.py:200-249)


def fill_queue(ids):
    q = MichaelScottQueue()
    for i in ids:
        q.enqueue(i)
    return q


def test_station_refill_and_ends():
    st = ReservationStation(0, 4)
    q = fill_queue(range(10))
    assert st.refill(q) == [0, 1, 2, 3] and st.reserved_count() == 4
    assert q.drain() == [4, 5, 6, 7, 8, 9]
    st = ReservationStation(0, 4)
    st.refill(fill_queue([1, 2, 3]))
    assert st.try_steal() == 3 and st.pop_for_run() == 1 and st.pop_for_run() == 2 and st.pop_for_run() is None
    assert ReservationStation(0, 4).refill(MichaelScottQueue()) == []


def test_steal_victim_choice():
    stations = {i: ReservationStation(i, 4) for i in range(3)}
    stations[1].refill(fill_queue([10, 11, 12]))
    stations[2].refill(fill_queue([20]))
    assert steal_task(0, stations) == (12, 1)
    stations = {i: ReservationStation(i, 4) for i in range(3)}
    assert steal_task(0, stations) == (None, None)
    stations[1].refill(fill_queue([10, 11]))
    stations[2].refill(fill_queue([20, 21]))
    assert steal_task(0, stations)[1] == 1  # tie -> lowest id


# ----------------------------------------------------------------- dry-run products


def dry(machine, m, k, n, t, **kw):
    rt = Runtime(machine, t, mode="dryrun", **kw)
    try:
        return rt.multiply(np.zeros((m, k)), np.zeros((k, n)), a_uid="A", b_uid="B", c_uid="C")[1]
    finally:
        rt.close()


@pytest.mark.parametrize("ndev", [1, 2, 3, 4])
def test_first_touch_and_identities(ndev):
    g, t = 6, 4
    s = dry(homogeneous_machine(ndev), g * t, g * t, g * t, t, directory_debug=True)
    assert s.cache.host_fetches == 2 * g * g  # every distinct tile crosses the host link once
    assert s.cache.input_requests == 2 * g ** 3
    assert s.cache.bytes_host == 2 * g * g * t * t * 8
    assert s.cache.bytes_peer == s.cache.l2_hits * t * t * 8
    assert s.cache.writebacks == g * g and s.cache.evictions == 0
    assert sum(s.tasks_by_device.values()) == s.total_tasks == g * g
    if ndev == 1:
        assert s.cache.l2_hits == 0
    for ev in s.steal_events:
        assert ev.thief != ev.victim and ev.queue_empty_observed


def test_bypass_is_2g3():
    g, t = 6, 4
    s = dry(homogeneous_machine(2), g * t, g * t, g * t, t, coherence=False)
    assert s.cache.host_fetches == 2 * g ** 3 and s.cache.l1_hits == 0 and s.cache.l2_hits == 0


def test_c2_reuse_16x():
    g, t = 16, 4
    on = dry(homogeneous_machine(2), g * t, g * t, g * t, t)
    off = dry(homogeneous_machine(2), g * t, g * t, g * t, t, coherence=False)
    assert on.cache.host_fetches == 512 and off.cache.host_fetches == 8192 and on.cache.evictions == 0


def test_single_device_counters_equal_reference_exactly():
    """One device: the schedule is deterministic, so every counter must equal the
    reference's (golden), including capacity-3 eviction counts and bypass."""
    meta = json.loads((G / "runs.json").read_text())
    checked = 0
    for name, m in meta.items():
        if name in ("session_reuse", "transpose") or m["devices"] != 1:
            continue
        s = dry(homogeneous_machine(1, capacity_tiles=m["capacity"]), m["m"], m["k"], m["n"], m["tile"],
                coherence=m["coherence"], directory_debug=True)
        assert s.cache.as_dict() == m["stats"]["cache"], name
        checked += 1
    assert checked >= 3


def test_multi_device_schedule_independent_counters_equal_reference():
    meta = json.loads((G / "runs.json").read_text())
    for name, m in meta.items():
        if name in ("session_reuse", "transpose"):
            continue
        s = dry(homogeneous_machine(m["devices"], capacity_tiles=m["capacity"]), m["m"], m["k"], m["n"],
                m["tile"], coherence=m["coherence"], directory_debug=True)
        ref = m["stats"]["cache"]
        assert s.total_tasks == m["stats"]["total_tasks"]
        assert [s.grid_rows, s.grid_cols, s.k_steps] == m["stats"]["grid"]
        assert s.cache.input_requests == ref["l1_hits"] + ref["l2_hits"] + ref["host_fetches"]
        assert s.cache.writebacks == ref["writebacks"] and s.cache.bytes_writeback == ref["bytes_writeback"]
        if m["capacity"] is None:
            # first touch: host traffic is schedule-independent without evictions
            assert s.cache.host_fetches == ref["host_fetches"] and s.cache.bytes_host == ref["bytes_host"]
        else:
            assert s.cache.evictions > 0


def test_capacity_three_exact_with_evictions():
    s = dry(homogeneous_machine(2, capacity_tiles=3), 40, 40, 40, 5, directory_debug=True)
    assert s.cache.evictions > 0 and s.cache.input_requests == 2 * s.total_tasks * s.k_steps


def test_exactly_once_many_threaded_runs():
    rng = np.random.default_rng(6)
    for _ in range(60):
        t, g, ndev = int(rng.integers(3, 6)), int(rng.integers(2, 5)), int(rng.integers(2, 5))
        s = dry(homogeneous_machine(ndev), t * g, t * g, t * g, t, directory_debug=True)
        assert sum(s.tasks_by_device.values()) == s.total_tasks == g * g


def test_session_reuse_and_transposed_identity():
    rt = Runtime(homogeneous_machine(1), 4, mode="dryrun")
    a = np.zeros((16, 16))
    _, s1 = rt.multiply(a, a, a_uid="X", b_uid="W")
    _, s2 = rt.multiply(a, a, a_uid="X", b_uid="W")
    assert s1.cache.host_fetches == 32 and s2.cache.host_fetches == 0
    assert s2.cache.l1_hits == s2.cache.input_requests
    rt = Runtime(homogeneous_machine(1), 4, mode="dryrun")
    x, y = np.zeros((12, 8)), np.zeros((12, 8))
    rt.multiply(x, np.zeros((8, 8)), a_uid="X", b_uid="W")
    before = rt.directory.stats()
    rt.multiply(x, y, transpose_a=True, a_uid="X", b_uid="Y2")
    assert rt.directory.stats().host_fetches - before.host_fetches == partition(y, 4).total_tiles


def test_static_shards_cover_every_task_once():
    m = homogeneous_machine(1)
    rt = Runtime(m, 4, mode="dryrun")
    seen = []
    for off in range(3):
        _, s = rt.multiply(np.zeros((24, 8)), np.zeros((8, 20)), task_offset=off, task_stride=3)
        seen.append(s.total_tasks)
    assert sum(seen) == 6 * 5


def test_mode_and_config_errors():
    with pytest.raises(ValueError):
        Runtime(homogeneous_machine(1), 4, mode="simulated")
    with pytest.raises(ValueError):
        Runtime(homogeneous_machine(1), 0, mode="dryrun")
    with pytest.raises(ConfigError):
        Runtime(Machine([DeviceSpec(0), DeviceSpec(1, kind="host-worker")], ProximityMatrix.uniform(2)), 4,
                mode="dryrun")
    with pytest.raises(ValueError):
        Runtime(homogeneous_machine(1), 4, mode="dryrun").multiply(np.zeros((4, 4)), np.zeros((5, 4)))
    # host workers exist only in the simulated engine (no CPU compute path on hardware)
    Runtime(Machine([DeviceSpec(0), DeviceSpec(1, kind="host-worker")], ProximityMatrix.uniform(2)), 4,
            mode="sim", compute=False).close()


def test_reports(tmp_path):
    s = dry(homogeneous_machine(2), 12, 12, 12, 4)
    write_report_json(s, tmp_path / "r.json")
    doc = json.loads((tmp_path / "r.json").read_text())
    assert doc["schema_version"] == 1
    for k in ("mode", "tile_size", "grid", "total_tasks", "makespan", "wall_elapsed", "devices", "cache"):
        assert k in doc
    assert sum(d["tasks_completed"] for d in doc["devices"]) == doc["total_tasks"] == 9
    write_report_csv(s, tmp_path / "r.csv")
    rows = (tmp_path / "r.csv").read_text().strip().splitlines()
    assert rows[0].startswith("device_id,kind,tasks_completed") and rows[-1].startswith("total")


@pytest.mark.parametrize("order", ["row-major", "banded", "shells", "blocked"])
def test_every_order_plans_the_same_task_set(order):
    """Enqueue order is a scheduling choice only: the task set, exactly-once and
    the first-touch identity hold for every order (unbounded capacity)."""
    rt = Runtime(homogeneous_machine(3), 4, mode="dryrun")
    rt.set_order(order)
    _, s = rt.multiply(np.zeros((28, 20)), np.zeros((20, 36)), a_uid="A", b_uid="B")
    assert s.total_tasks == 7 * 9 and sum(s.tasks_by_device.values()) == 63
    assert s.cache.host_fetches == 7 * 5 + 5 * 9 and s.cache.input_requests == 2 * 63 * 5


def test_describe_strided_host_views():
    from paper_1511_04348_b200.matrix import describe

    m = np.zeros((10, 12))
    d = describe(m[2:7, 3:9])
    assert (d.rows, d.cols, d.ld) == (5, 6, 12)
    with pytest.raises(ValueError):
        describe(m.T)  # column-major: not readable in place
    with pytest.raises(ValueError):
        describe(m[:, ::2])


def test_completion_bitmap_contract_and_native_view():
    """Completion (scheduler.py:70-96): exactly once, all_done gate; every product's
    RunStats carries the native runtime's bitmap as one."""
    import numpy as np

    from paper_1511_04348_b200 import Runtime, homogeneous_machine
    from paper_1511_04348_b200.scheduler import Completion

    c = Completion(3)
    c.mark(0)
    c.mark(2)
    assert not c.all_done() and c.done_count == 2 and c.snapshot() == [True, False, True]
    with pytest.raises(RuntimeError, match="executed twice"):
        c.mark(2)
    c.mark(1)
    assert c.all_done()
    with Runtime(homogeneous_machine(2), 4, mode="dryrun") as rt:
        _, s = rt.multiply(np.zeros((12, 8)), np.zeros((8, 16)))
    assert s.completion.all_done() and s.completion.done_count == s.total_tasks == 12


def test_directory_lock_stats_dryrun():
    """Runtime.lock_stats (tr_session_lock_stats): every directory operation is one
    acquisition of the instrumented lock; reset=True zeroes the counters."""
    import numpy as np

    from paper_1511_04348_b200 import Runtime, homogeneous_machine

    with Runtime(homogeneous_machine(3), 4, mode="dryrun") as rt:
        rt.lock_stats(reset=True)
        rt.multiply(np.zeros((16, 12)), np.zeros((12, 20)))
        st = rt.lock_stats(reset=True)
        assert st["acquisitions"] >= 2 * 4 * 5 * 3  # >= one per input request (20 tasks x 3 k-steps x A, B)
        assert st["held_s"] >= 0 and st["waited_s"] >= 0 and st["max_hold_us"] >= 0
        assert rt.lock_stats()["acquisitions"] < st["acquisitions"]


def test_default_precision_resolution(monkeypatch):
    from paper_1511_04348_b200 import dense

    monkeypatch.delenv("TR_PRECISION", raising=False)
    assert dense.default_precision() == "fp32acc"
    monkeypatch.setenv("TR_PRECISION", "exact")
    assert dense.default_precision() == "exact" and dense.precision_code(None) == dense.PRECISIONS["exact"]
    dense.set_default_precision("bf16")
    try:
        assert dense.default_precision() == "bf16"
    finally:
        dense.set_default_precision(None)
    monkeypatch.setenv("TR_PRECISION", "fp16")
    with pytest.raises(ValueError):
        dense.default_precision()
    with pytest.raises(ValueError):
        dense.set_default_precision("tf32")
