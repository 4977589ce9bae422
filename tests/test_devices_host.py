"""Machine model and cost functions of the host mirror (devices.py), checked
against the behaviour the reference's device tests pin down
(reference pkg/tests/test_devices.py:24-193; pkg/src/tilerun/devices.py:30-305).

These functions price the simulated engine (mode="sim") and validate the
machine configs the GPU runtime is built from; no GPU is needed."""
import json

import numpy as np
import pytest

import paper_1511_04348_b200 as tr
from paper_1511_04348_b200.devices import (
    HOST, Clock, ConfigError, DeviceSpec, Machine, ProximityMatrix, closest_owner, compute_cost,
    homogeneous_machine, load_machine, save_machine, transfer_cost)


# ---- compute_cost: 2mkn / flops_per_unit (devices.py:255-261) ----------------

@pytest.mark.parametrize("flops,a,b,expected", [
    (1000.0, (10, 10), (10, 10), 2.0),
    (8.0, (1, 1), (1, 1), 0.25),
    (1.0, (3, 5), (5, 7), 210.0),
    (4096.0, (512, 2), (2, 1), 0.5),
])
def test_compute_cost_values(flops, a, b, expected):
    assert compute_cost(DeviceSpec(0, flops_per_unit=flops), a, b) == expected


def test_compute_cost_inverse_in_throughput_and_shape_checked():
    half, full = DeviceSpec(0, flops_per_unit=250.0), DeviceSpec(1, flops_per_unit=500.0)
    assert compute_cost(half, (6, 3), (3, 9)) == 2 * compute_cost(full, (6, 3), (3, 9))
    with pytest.raises(ValueError):
        compute_cost(full, (4, 3), (2, 4))


# ---- transfer_cost (devices.py:264-282) -------------------------------------

def test_transfer_cost_endpoints():
    m = homogeneous_machine(2, host_bandwidth=50.0, peer_bandwidth=200.0)
    assert transfer_cost(m, 1, 1, 999) == 0.0 and transfer_cost(m, HOST, HOST, 999) == 0.0
    assert transfer_cost(m, HOST, 1, 400) == 8.0 == transfer_cost(m, 1, HOST, 400)   # both directions of the host link
    assert transfer_cost(m, 0, 1, 400) == 2.0                                         # the faster peer link
    with pytest.raises(ConfigError):
        transfer_cost(m, HOST, 5, 1)
    with pytest.raises(ConfigError):
        transfer_cost(m, 5, 0, 1)


def test_transfer_latency_is_per_transfer():
    m = homogeneous_machine(2, host_bandwidth=10.0, peer_bandwidth=20.0, transfer_latency=0.25)
    assert transfer_cost(m, HOST, 0, 10) == 1.25
    assert transfer_cost(m, 0, 1, 10) == 0.75
    assert transfer_cost(m, 0, 0, 10) == 0.0


def test_host_worker_reads_host_memory_for_free():
    devs = [DeviceSpec(0, flops_per_unit=10.0, host_bandwidth=4.0),
            DeviceSpec(1, kind="host-worker", flops_per_unit=5.0, host_bandwidth=1.0)]
    m = Machine(devs, ProximityMatrix.uniform(2, bandwidth=100.0))
    assert transfer_cost(m, HOST, 1, 4000) == 0.0 == transfer_cost(m, 1, HOST, 4000)
    assert transfer_cost(m, HOST, 0, 4000) == 1000.0


def test_costs_are_homogeneous_in_rates():
    """Scaling every rate by c divides every cost by c."""
    rng = np.random.default_rng(7)
    for _ in range(12):
        bw, fl, c = float(rng.uniform(5, 900)), float(rng.uniform(5, 900)), float(rng.uniform(0.2, 40))
        nbytes = int(rng.integers(1, 1 << 20))
        slow = homogeneous_machine(2, host_bandwidth=bw, peer_bandwidth=3 * bw, flops_per_unit=fl)
        fast = homogeneous_machine(2, host_bandwidth=c * bw, peer_bandwidth=3 * c * bw, flops_per_unit=c * fl)
        for src, dst in ((HOST, 0), (1, HOST), (0, 1)):
            assert transfer_cost(slow, src, dst, nbytes) == pytest.approx(c * transfer_cost(fast, src, dst, nbytes))
        assert compute_cost(slow.device(1), (16, 4), (4, 8)) == pytest.approx(
            c * compute_cost(fast.device(1), (16, 4), (4, 8)))


# ---- closest_owner (devices.py:285-291) -------------------------------------

def test_closest_owner_rules():
    uni = ProximityMatrix.uniform(5)
    assert closest_owner(0, {3}, uni) == 3
    assert closest_owner(4, {3, 1, 2}, uni) == 1                                 # tie -> lowest id
    hops = np.array([[0, 3, 2, 1], [3, 0, 1, 2], [2, 1, 0, 1], [1, 2, 1, 0]])
    prox = ProximityMatrix(hops, np.full((4, 4), 5.0))
    assert closest_owner(0, {1, 2, 3}, prox) == 3                                # fewest hops wins over id
    assert closest_owner(1, {0, 3}, prox) == 3
    with pytest.raises(ValueError):
        closest_owner(0, [], uni)


# ---- validation (devices.py:30-216) -----------------------------------------

@pytest.mark.parametrize("kw", [
    dict(flops_per_unit=0.0), dict(flops_per_unit=-3.0), dict(host_bandwidth=-1.0), dict(host_bandwidth=0.0),
    dict(capacity_tiles=2), dict(capacity_tiles=0), dict(kind="host-worker", capacity_tiles=16),
    dict(kind="tpu"), dict(slots=0),
])
def test_device_spec_rejects(kw):
    with pytest.raises(ConfigError):
        DeviceSpec(0, **kw)


def test_device_spec_minimum_capacity_and_error_class():
    assert DeviceSpec(0, capacity_tiles=3).capacity_tiles == 3
    assert issubclass(ConfigError, ValueError)


@pytest.mark.parametrize("hops,bw", [
    ([[0, 1], [3, 0]], np.ones((2, 2))),          # asymmetric
    ([[2]], np.ones((1, 1))),                     # non-zero diagonal
    ([[0, 1], [1, 0]], np.zeros((2, 2))),         # peer bandwidth must be > 0
    ([[0, -1], [-1, 0]], np.ones((2, 2))),        # negative hops
    ([[0, 1, 1], [1, 0, 1]], np.ones((2, 3))),    # not square
])
def test_proximity_rejects(hops, bw):
    with pytest.raises(ConfigError):
        ProximityMatrix(np.array(hops), bw)


def test_machine_rejects():
    with pytest.raises(ConfigError):
        Machine([], ProximityMatrix.uniform(0))
    with pytest.raises(ConfigError):
        Machine([DeviceSpec(1)], ProximityMatrix.uniform(1))                      # ids start at 0
    with pytest.raises(ConfigError):
        Machine([DeviceSpec(0), DeviceSpec(2)], ProximityMatrix.uniform(2))       # ids contiguous
    with pytest.raises(ConfigError):
        Machine([DeviceSpec(0)], ProximityMatrix.uniform(3))                      # size mismatch
    with pytest.raises(ConfigError):
        homogeneous_machine(2).device(2)


# ---- config files (devices.py:187-252) --------------------------------------

@pytest.mark.parametrize("dtype,elem", [(np.float64, 8), (np.float32, 4)])
def test_config_roundtrip(tmp_path, dtype, elem):
    m = homogeneous_machine(3, flops_per_unit=11.0, host_bandwidth=22.0, peer_bandwidth=33.0,
                            capacity_tiles=7, slots=3, transfer_latency=0.5, dtype=dtype)
    p = tmp_path / "machine.json"
    save_machine(p, m)
    back = load_machine(p)
    assert back.devices == m.devices
    assert np.array_equal(back.proximity.hops, m.proximity.hops)
    assert np.array_equal(back.proximity.peer_bandwidth, m.proximity.peer_bandwidth)
    assert back.transfer_latency == 0.5 and back.element_bytes == elem
    assert Machine.from_dict(json.loads(p.read_text())).to_dict() == m.to_dict()


@pytest.mark.parametrize("text", [
    '{"devices": [{"kind": "accelerator"}]}',                 # no id
    '{"devices": [{"id": 0, "kind": "fpga"}]}',               # unknown kind
    '{"devices": [{"id": 0, "capacity_tiles": 1}]}',          # below A+B+C
    '{"nodes": []}',                                          # no devices key
])
def test_malformed_config(tmp_path, text):
    p = tmp_path / "bad.json"
    p.write_text(text)
    with pytest.raises(ConfigError):
        load_machine(p)


def test_package_exports_the_machine_api():
    for name in ("DeviceSpec", "Machine", "ProximityMatrix", "ConfigError", "homogeneous_machine", "load_machine",
                 "save_machine", "closest_owner", "compute_cost", "transfer_cost", "Clock", "HOST"):
        assert hasattr(tr, name), name


# ---- Clock (devices.py:294-305) ---------------------------------------------

def test_clock_monotone():
    c = Clock()
    for t in (0.0, 1.5, 1.5, 4.0):
        c.advance_to(t)
    with pytest.raises(ValueError):
        c.advance_to(3.9)
    assert c.now == 4.0
