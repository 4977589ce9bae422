"""Precision "exact" (KX): the reference's own arithmetic on the GPU, bit for bit.

The reference accumulates every output element as k-ascending rank-1 updates,
a rounded multiply then a rounded add in the output dtype (tiles.py:154-172,
197-212).  KX does the same per element, so the scheduled product must equal
the reference's result with np.array_equal -- whatever the tile size, device
count, stealing or capacity-forced k-chunking -- and so must the dense
(in-core) path.  The reference's golden runs (tests/golden/runs.npz, made by
the reference itself) are compared bitwise here, float cases included.
"""

import json
from pathlib import Path

import numpy as np
import pytest
import torch

from oracle import tilerun_oracle as O
from paper_1511_04348_b200 import Runtime, homogeneous_machine, run
from paper_1511_04348_b200 import dense
from paper_1511_04348_b200.dense import dense_gemm

pytestmark = pytest.mark.gpu
G = Path(__file__).resolve().parent / "golden"


def diff(c, ref):
    bad = np.argwhere(c != ref)
    return f"{len(bad)} differing elements, first {bad[:3].tolist()}"


def test_golden_runs_bitwise():
    meta = json.loads((G / "runs.json").read_text())
    arr = np.load(G / "runs.npz")
    for name, m in meta.items():
        if name in ("session_reuse", "transpose"):
            continue
        a, b, cref = arr[name + "_a"], arr[name + "_b"], arr[name + "_c"]
        c, s = run(homogeneous_machine(m["devices"], capacity_tiles=m["capacity"]), a, b, m["tile"],
                   coherence=m["coherence"], directory_debug=True, precision="exact")
        assert c.dtype == cref.dtype
        assert np.array_equal(c, cref), (name, diff(c, cref))
        assert s.precision == "exact" and s.gpu_launches > 0


@pytest.mark.parametrize("dtype", [np.float64, np.float32])
@pytest.mark.parametrize("tile,devices,cap", [(32, 1, None), (48, 2, None), (100, 3, None), (40, 2, 4)])
def test_scheduled_bitwise(dtype, tile, devices, cap):
    rng = np.random.default_rng(tile + devices)
    a = rng.standard_normal((173, 211)).astype(dtype)
    b = rng.standard_normal((211, 157)).astype(dtype)
    ref = O.reference_gemm(a, b)
    c, s = run(homogeneous_machine(devices, capacity_tiles=cap, dtype=dtype), a, b, tile, precision="exact")
    assert c.dtype == ref.dtype
    assert np.array_equal(c, ref), diff(c, ref)
    assert sum(s.tasks_by_device.values()) == s.total_tasks


def test_mixed_dtypes_follow_the_reference_scheduler():
    # the scheduled product keeps A's dtype (scheduler.py:182) and updates it in place,
    # out += outer(a[:, k], b[k, :]) (scheduler.py:400 -> tiles.py:170-171)
    rng = np.random.default_rng(5)
    a32 = rng.standard_normal((70, 90)).astype(np.float32)
    b64 = rng.standard_normal((90, 50))
    ref = O.accumulate_product(a32, b64, np.zeros((70, 50), np.float32))
    c, _ = run(homogeneous_machine(2), a32, b64, 32, precision="exact")
    assert c.dtype == np.float32 and np.array_equal(c, ref), diff(c, ref)
    a64, b32 = a32.astype(np.float64) * 1.1, b64.astype(np.float32)
    ref = O.accumulate_product(a64, b32, np.zeros((70, 50)))
    c, _ = run(homogeneous_machine(2), a64, b32, 32, precision="exact")
    assert c.dtype == np.float64 and np.array_equal(c, ref), diff(c, ref)


def test_transposed_operands_and_session_reuse():
    rng = np.random.default_rng(9)
    x = rng.standard_normal((120, 75))
    w = rng.standard_normal((120, 66))
    with Runtime(homogeneous_machine(2), 32, precision="exact") as rt:
        c1, _ = rt.multiply(x, w, transpose_a=True, a_uid="X", b_uid="W")
        c2, s2 = rt.multiply(x, w, transpose_a=True, a_uid="X", b_uid="W")  # warm: tiles resident
        c3, _ = rt.multiply(w.T.copy(), x, transpose_b=False, a_uid="WT", b_uid="X")
    ref = O.reference_gemm(np.ascontiguousarray(x.T), w)
    assert np.array_equal(c1, ref), diff(c1, ref)
    assert np.array_equal(c2, ref) and s2.cache.host_fetches == 0
    assert np.array_equal(c3, O.reference_gemm(np.ascontiguousarray(w.T), x))


@pytest.mark.parametrize("dtype", [torch.float64, torch.float32])
@pytest.mark.parametrize("ta,tb", [(False, False), (True, False), (False, True), (True, True)])
def test_dense_gemm_bitwise(dtype, ta, tb):
    g = torch.Generator().manual_seed(3)
    m, k, n = 150, 257, 93
    a = torch.randn((k, m) if ta else (m, k), generator=g, dtype=dtype)
    b = torch.randn((n, k) if tb else (k, n), generator=g, dtype=dtype)
    an = a.numpy().T if ta else a.numpy()
    bn = b.numpy().T if tb else b.numpy()
    ref = O.reference_gemm(np.ascontiguousarray(an), np.ascontiguousarray(bn))
    c = dense_gemm(a.cuda(), b.cuda(), ta, tb, precision="exact").cpu().numpy()
    assert np.array_equal(c, ref), diff(c, ref)
    # accumulate: gemm_tile's c + a @ b (tiles.py:183-194), rank-1 updates onto C
    c0 = torch.randn((m, n), generator=g, dtype=dtype)
    out = c0.cuda()
    dense_gemm(a.cuda(), b.cuda(), ta, tb, out=out, precision="exact", accumulate=True)
    ref2 = O.accumulate_product(np.ascontiguousarray(an), np.ascontiguousarray(bn), c0.numpy().copy())
    assert np.array_equal(out.cpu().numpy(), ref2), diff(out.cpu().numpy(), ref2)


def test_default_precision_switch(monkeypatch):
    rng = np.random.default_rng(4)
    a, b = rng.standard_normal((64, 96)), rng.standard_normal((96, 40))
    ref = O.reference_gemm(a, b)
    monkeypatch.setenv("TR_PRECISION", "exact")
    c, s = run(homogeneous_machine(1), a, b, 32)
    assert s.precision == "exact" and np.array_equal(c, ref)
    monkeypatch.delenv("TR_PRECISION")
    dense.set_default_precision("exact")
    try:
        c, s = run(homogeneous_machine(1), a, b, 32)
        assert s.precision == "exact" and np.array_equal(c, ref)
    finally:
        dense.set_default_precision(None)
    c, s = run(homogeneous_machine(1), a, b, 32)
    assert s.precision == "fp32acc" and np.linalg.norm(c - ref) <= 1e-5 * np.linalg.norm(ref)


def test_exact_rejects_fused_epilogues():
    from paper_1511_04348_b200.gpu_mlp import GpuMLP

    with pytest.raises(ValueError, match="exact"):
        GpuMLP([], tile_size=32, precision="exact")


def test_tiles_reference_entry_points_default_to_exact():
    """tiles.reference_gemm / accumulate_product / gemm_tile promise the reference's
    fixed k-ascending order (tiles.py:154-212): by default they return its bits;
    precision="fp32acc" gives the tensor-core product."""
    from paper_1511_04348_b200 import accumulate_product, gemm_tile, reference_gemm

    rng = np.random.default_rng(12)
    a, b = rng.standard_normal((90, 70)), rng.standard_normal((70, 50))
    c0 = rng.standard_normal((90, 50))
    assert np.array_equal(reference_gemm(a, b), O.reference_gemm(a, b))
    out = c0.copy()
    accumulate_product(a, b, out)
    assert np.array_equal(out, O.accumulate_product(a, b, c0.copy()))
    assert np.array_equal(gemm_tile(a, b, c0), O.accumulate_product(a, b, c0.copy()))
    fast = reference_gemm(a, b, precision="fp32acc")
    ref = a @ b
    assert np.linalg.norm(fast - ref) <= 1e-5 * np.linalg.norm(ref)
