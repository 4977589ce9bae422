"""MLP training through the GPU tiled runtime vs the reference's golden
trajectories (tests/golden/ann.npz, produced by the real reference with its
f64 DenseBackend).  Losses must match within the fp32-accurate tolerance."""

from pathlib import Path

import numpy as np
import pytest

from paper_1511_04348_b200 import DenseBackend, Layer, Network, TiledBackend, homogeneous_machine
from paper_1511_04348_b200.ann import loss_gradients, train_step, xor_dataset

pytestmark = pytest.mark.gpu
G = Path(__file__).resolve().parent / "golden"


@pytest.fixture(scope="module")
def g():
    return np.load(G / "ann.npz")


def net_from(g, act):
    return Network([Layer(g[f"{act}_init_w{i}"].copy(), g[f"{act}_init_b{i}"].copy(), act, tag=f"layer{i}")
                    for i in range(3)])


def relerr(x, ref):
    return float(np.linalg.norm(np.asarray(x) - ref) / max(np.linalg.norm(ref), 1e-300))


@pytest.mark.parametrize("act", ["sigmoid", "relu"])
@pytest.mark.parametrize("backend_kind", ["tiled", "dense"])
def test_gradients_and_trajectory(g, act, backend_kind):
    """The fp32-accurate tensor-core path through the reference's ANN API (the
    backends' own default is exact, tested bitwise below)."""
    backend = (TiledBackend(homogeneous_machine(2), tile_size=16, mode="gpu", precision="fp32acc")
               if backend_kind == "tiled" else DenseBackend(precision="fp32acc"))
    net = net_from(g, act)
    loss, grads = loss_gradients(net, g[f"{act}_x"], g[f"{act}_t"], backend)
    assert abs(loss - g[f"{act}_loss0"][0]) <= 1e-5 * abs(g[f"{act}_loss0"][0])
    for i, (gw, gb) in enumerate(grads):
        assert relerr(gw, g[f"{act}_gw{i}"]) <= 1e-4 and relerr(gb, g[f"{act}_gb{i}"]) <= 1e-4
    traj = [train_step(net, g[f"{act}_x"], g[f"{act}_t"], 0.1, backend) for _ in range(10)]
    ref = g[f"{act}_losses"]
    assert np.max(np.abs(np.array(traj) - ref) / np.abs(ref)) <= 1e-5
    for i, layer in enumerate(net.layers):
        assert relerr(layer.weights, g[f"{act}_final_w{i}"]) <= 1e-5


def test_xor_trajectory_tiled_t2(g):
    rng = np.random.default_rng(0)
    net = Network.from_sizes([2, 8, 1], rng, activation="sigmoid")
    assert np.array_equal(net.layers[0].weights, g["xor_w0"])
    x, t = xor_dataset()
    backend = TiledBackend(homogeneous_machine(2), tile_size=2, mode="gpu")
    losses = np.array([train_step(net, x, t, 0.5, backend) for _ in range(50)])
    assert np.max(np.abs(losses - g["xor_losses"]) / g["xor_losses"]) <= 1e-5


def test_backward_reuses_forward_tiles():
    rng = np.random.default_rng(5)
    net = Network.from_sizes([8, 8, 4], rng)
    x, t = rng.uniform(-1, 1, (8, 8)), rng.uniform(-1, 1, (8, 4))
    backend = TiledBackend(homogeneous_machine(1), tile_size=4, mode="gpu")
    train_step(net, x, t, 0.1, backend)
    assert backend.runtime.directory.stats().l1_hits > 0
    assert len(backend.call_stats) == 3 * 2


def test_default_sim_backend_times_improve_with_devices():
    """TiledBackend in the reference's default mode "sim" (ann.py:85): products from
    the GPU kernel, bench_pass in simulated time, which falls with more devices
    (test_ann.py:200-208)."""
    from paper_1511_04348_b200.ann import bench_pass, random_regression

    rng = np.random.default_rng(6)
    net = Network.from_sizes([48, 48, 48], rng)
    x, t = random_regression(rng, 48, 48, 48)
    times = {}
    for n in (1, 4):
        backend = TiledBackend(homogeneous_machine(n), tile_size=8, mode="sim")
        times[n] = bench_pass(net, x, t, backend, repeats=3)
        loss, _ = loss_gradients(net, x, t, backend)
        assert np.isfinite(loss)
    assert 0 < times[4] < times[1]


@pytest.mark.parametrize("act", ["sigmoid", "relu"])
@pytest.mark.parametrize("backend_kind", ["tiled", "dense"])
def test_exact_precision_reproduces_the_reference_bitwise(g, act, backend_kind):
    """Precision "exact": the reference's DenseBackend trajectories (ann.npz, made
    by the reference itself) bit for bit -- gradients, 10 losses, final weights --
    through the tiled runtime on 2 devices or the dense GPU path."""
    backend = (TiledBackend(homogeneous_machine(2), tile_size=16, mode="gpu", precision="exact")
               if backend_kind == "tiled" else DenseBackend(precision="exact"))
    net = net_from(g, act)
    loss, grads = loss_gradients(net, g[f"{act}_x"], g[f"{act}_t"], backend)
    assert loss == g[f"{act}_loss0"][0]
    for i, (gw, gb) in enumerate(grads):
        assert np.array_equal(gw, g[f"{act}_gw{i}"]) and np.array_equal(gb, g[f"{act}_gb{i}"])
    traj = [train_step(net, g[f"{act}_x"], g[f"{act}_t"], 0.1, backend) for _ in range(10)]
    assert np.array_equal(np.array(traj), g[f"{act}_losses"])
    for i, layer in enumerate(net.layers):
        assert np.array_equal(layer.weights, g[f"{act}_final_w{i}"])


def test_backends_default_to_exact_like_the_reference_float64_ann(monkeypatch):
    from paper_1511_04348_b200 import dense
    from paper_1511_04348_b200.ann import ann_default_precision

    monkeypatch.delenv("TR_PRECISION", raising=False)
    assert ann_default_precision() == "exact" and DenseBackend().precision == "exact"
    tb = TiledBackend(homogeneous_machine(1), tile_size=8)
    assert tb.runtime.precision == "exact" and tb.runtime.mode == "sim"  # the reference's default (ann.py:85)
    assert TiledBackend(homogeneous_machine(1), tile_size=8, mode="gpu").runtime.precision == "exact"
    monkeypatch.setenv("TR_PRECISION", "fp32acc")
    assert DenseBackend().precision == "fp32acc"
    monkeypatch.delenv("TR_PRECISION")
    dense.set_default_precision("bf16")
    try:
        assert DenseBackend().precision == "bf16"
    finally:
        dense.set_default_precision(None)
