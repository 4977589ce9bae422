"""Pin the oracle: the CPU restatement (oracle/) against golden vectors produced
by running the REAL reference (tests/golden/make_golden.py).  Bit-exact."""

import json
from pathlib import Path

import numpy as np
import pytest

from oracle import tilerun_oracle as O

G = Path(__file__).resolve().parent / "golden"


@pytest.fixture(scope="module")
def tiles():
    return np.load(G / "tiles.npz")


@pytest.fixture(scope="module")
def c_lib():
    O.build_c_oracle()
    lib = O.c_oracle()
    assert lib is not None
    return lib


def test_known_answers(tiles):
    c = np.zeros((2, 2))
    O.accumulate_product(tiles["hand_a"], tiles["hand_b"], c)
    assert np.array_equal(c, tiles["hand_c"])
    assert np.array_equal(c, [[19.0, 22.0], [43.0, 50.0]])
    acc = np.array([[10.0]])
    O.accumulate_product(np.array([[1.0, 1.0]]), np.array([[2.0], [3.0]]), acc)
    assert np.array_equal(acc, tiles["acc_c"])


@pytest.mark.parametrize("idx", range(7))
def test_reference_gemm_bitwise(tiles, c_lib, idx):
    a, b = tiles[f"rand{idx}_a"], tiles[f"rand{idx}_b"]
    assert np.array_equal(O.reference_gemm(a, b), tiles[f"rand{idx}_c"])
    assert np.array_equal(c_lib.gemm(a, b, threads=3), tiles[f"rand{idx}_c"])
    a32, b32 = tiles[f"rand{idx}_a32"], tiles[f"rand{idx}_b32"]
    assert np.array_equal(O.reference_gemm(a32, b32), tiles[f"rand{idx}_c32"])
    assert np.array_equal(c_lib.gemm(a32, b32), tiles[f"rand{idx}_c32"])
    acc = tiles[f"rand{idx}_acc0"].copy()
    O.accumulate_product(a, b, acc)
    assert np.array_equal(acc, tiles[f"rand{idx}_acc"])
    acc2 = tiles[f"rand{idx}_acc0"].copy()
    c_lib.rank1_updates(np.ascontiguousarray(a), np.ascontiguousarray(b), acc2, a.shape[1])
    assert np.array_equal(acc2, tiles[f"rand{idx}_acc"])


def test_census(tiles):
    for rows, cols, t, gr, gc, full, ragged in tiles["census"]:
        assert O.grid_shape(rows, cols, t) == (gr, gc)
        assert O.census(rows, cols, t) == (full, ragged)


def test_plans_match_reference():
    for case in json.loads((G / "plans.json").read_text()):
        tasks = O.plan_tasks(case["m"], case["k"], case["n"], case["tile"])
        assert [[t.task_id, t.row, t.col, t.k_steps] for t in tasks] == case["tasks"]


def test_runs_products_bitwise():
    meta = json.loads((G / "runs.json").read_text())
    arr = np.load(G / "runs.npz")
    for name, m in meta.items():
        if name in ("session_reuse", "transpose"):
            continue
        a, b, c = arr[name + "_a"], arr[name + "_b"], arr[name + "_c"]
        assert np.array_equal(O.reference_gemm(a, b), c), name  # tiled reference == dense, bitwise
        g = m["stats"]["grid"]
        assert g == [O.grid_shape(m["m"], m["n"], m["tile"])[0], O.grid_shape(m["m"], m["n"], m["tile"])[1],
                     O.grid_shape(m["m"], m["k"], m["tile"])[1]]
    x, y, c = arr["transpose_x"], arr["transpose_y"], arr["transpose_c"]
    assert np.array_equal(O.reference_gemm(x.T, y), c)


def test_single_device_counters_match_reference():
    """The sequential _execute_task restatement reproduces the reference's
    one-device CacheStats exactly (incl. capacity-3 evictions and bypass)."""
    meta = json.loads((G / "runs.json").read_text())
    checked = 0
    for name, m in meta.items():
        if name in ("session_reuse", "transpose") or m["devices"] != 1:
            continue
        st = O.run_schedule_single_device(m["m"], m["k"], m["n"], m["tile"], capacity=m["capacity"],
                                          enabled=m["coherence"])
        assert st == m["stats"]["cache"], name
        checked += 1
    assert checked >= 3


def _apply(model, rec):
    op, dev, key = rec["op"], rec["dev"], tuple(rec["key"])
    try:
        if op == "lookup":
            lv, owner = model.lookup(dev, key)
            out = [lv, owner]
        elif op == "admit":
            out = [list(e) for e in model.admit(dev, key)]
        elif op == "pin":
            model.pin(dev, key)
            out = None
        elif op == "unpin":
            model.unpin(dev, key)
            out = None
        elif op == "acquire":
            lv, src, nb, ev = model.acquire_input(dev, key, 7 + key[1] * 4 + key[2])
            out = [lv, src, nb, [list(e) for e in ev]]
        elif op == "release":
            model.release_input(dev, key)
            out = None
        elif op == "admit_out":
            out = [list(e) for e in model.admit_output(dev, key)]
        else:
            model.release_output(dev, key, 64)
            out = None
        return out, None
    except O.CapacityErrorModel:
        return None, "capacity"
    except ValueError:
        return None, "value"
    except KeyError:
        return None, "key"


def test_directory_model_matches_reference():
    for seq in json.loads((G / "directory.json").read_text()):
        model = O.DirectoryModel(seq["caps"], seq["hops"], enabled=seq["enabled"], policy=seq["policy"])
        for rec in seq["ops"]:
            out, err = _apply(model, rec)
            assert err == rec["err"], rec
            if "out" in rec and err is None:
                assert out == rec["out"], rec
            assert [[list(k) for k in model.residents(d)] for d in range(len(seq["caps"]))] == rec["residents"]
            assert model.stats == rec["stats"]


def test_ann_oracle_matches_reference():
    g = np.load(G / "ann.npz")
    rng = np.random.default_rng(0)
    layers = O.network_from_sizes([2, 8, 1], rng)
    assert np.array_equal(layers[0].weights, g["xor_w0"])
    x, t = O.xor_dataset()
    losses = [O.train_step(layers, x, t, 0.5) for _ in range(50)]
    assert np.array_equal(np.array(losses), g["xor_losses"])
    for act in ("sigmoid", "relu"):
        layers = [O.OracleLayer(g[f"{act}_init_w{i}"].copy(), g[f"{act}_init_b{i}"].copy(), act) for i in range(3)]
        loss, grads = O.loss_gradients(layers, g[f"{act}_x"], g[f"{act}_t"])
        assert loss == g[f"{act}_loss0"][0]
        for i, (gw, gb) in enumerate(grads):
            assert np.array_equal(gw, g[f"{act}_gw{i}"]) and np.array_equal(gb, g[f"{act}_gb{i}"])
        traj = [O.train_step(layers, g[f"{act}_x"], g[f"{act}_t"], 0.1) for _ in range(10)]
        assert np.array_equal(np.array(traj), g[f"{act}_losses"])


def test_ann_blas_oracle_close_to_exact():
    """The BLAS-f64 MLP oracle used at large sizes differs from the exact one by ~1e-15."""
    g = np.load(G / "ann.npz")
    layers = [O.OracleLayer(g[f"sigmoid_init_w{i}"].copy(), g[f"sigmoid_init_b{i}"].copy()) for i in range(3)]
    loss, _ = O.loss_gradients(layers, g["sigmoid_x"], g["sigmoid_t"], matmul=O.blas_matmul)
    assert abs(loss - g["sigmoid_loss0"][0]) <= 1e-13 * abs(loss)


def test_cfg1_sampled_slices_and_checksums(c_lib):
    """cfg1 (N=2048, T=512): the sampled-slice oracle reproduces the reference's
    own threaded run bit-for-bit on the sampled block (fp32 machine)."""
    g = np.load(G / "cfg1.npz")
    a = np.random.default_rng(1).standard_normal((2048, 2048)).astype(np.float32)
    b = np.random.default_rng(2).standard_normal((2048, 2048)).astype(np.float32)
    assert np.allclose([a.sum(dtype=np.float64), (a.astype(np.float64) ** 2).sum()], g["a_sum"], rtol=0, atol=0)
    assert np.allclose([b.sum(dtype=np.float64), (b.astype(np.float64) ** 2).sum()], g["b_sum"], rtol=0, atol=0)
    rows, cols = g["rows"], g["cols"]
    assert np.array_equal(O.gemm_slice(a, b, rows, cols, dtype=np.float32), g["c32_block"])
    assert np.array_equal(O.gemm_slice(a, b, rows, cols, dtype=np.float64), g["c64_block"])
    # the reference's first-touch accounting at cfg1: 2 g^2 tiles of 512x512 fp32
    host_fetches, bytes_host, hits, writebacks, bytes_wb, tasks = g["stats"]
    assert host_fetches == 2 * 4 * 4 and bytes_host == 32 * 512 * 512 * 4
    assert hits + host_fetches == 2 * 16 * 4 and writebacks == tasks == 16


def test_band_samples_cover_every_band():
    """Sampled-slice indices: >= 8 per tile band, band edges included (ragged last band too)."""
    idx = O.band_samples(10000, 4096, per_band=8, seed=3)
    for lo in range(0, 10000, 4096):
        band = idx[(idx >= lo) & (idx < min(lo + 4096, 10000))]
        assert len(band) >= 8 and band[0] == lo and band[-1] == min(lo + 4096, 10000) - 1
