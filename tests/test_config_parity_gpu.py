"""Config-level parity on the GPU: BASELINE cfg1 exactly as the reference ran it,
and band-sampled products with ragged edges.

cfg1 = run(homogeneous_machine(n, dtype=float32), A, B, 512) on N = 2048 fp32
(A, B: default_rng(1|2).standard_normal, float32).  tests/golden/cfg1.npz holds
the reference's own threaded run of exactly that call (make_golden.py): input
checksums, a sampled 8x8 block in f32 and f64, per-tile checksums, the f64
Frobenius norm of C and the reference's CacheStats.  The GPU result must match
the f64 product within the north-star tolerance (1e-5 fp32acc, 1e-2 bf16) and
the counters must be the reference's (scheduler.py:165-197, coherence.py:210-280).
"""

from pathlib import Path

import numpy as np
import pytest

from oracle import tilerun_oracle as O
from paper_1511_04348_b200 import homogeneous_machine, run

pytestmark = pytest.mark.gpu
G = Path(__file__).resolve().parent / "golden"
TOL = {"fp32acc": 1e-5, "bf16": 1e-2}


def rel(c, ref):
    ref = np.asarray(ref, np.float64)
    return float(np.linalg.norm(np.asarray(c, np.float64) - ref) / np.linalg.norm(ref))


@pytest.fixture(scope="module")
def cfg1():
    g = np.load(G / "cfg1.npz")
    a = np.random.default_rng(1).standard_normal((2048, 2048)).astype(np.float32)
    b = np.random.default_rng(2).standard_normal((2048, 2048)).astype(np.float32)
    # the same inputs the reference ran on (its checksums, bit for bit)
    assert np.array_equal([a.sum(dtype=np.float64), (a.astype(np.float64) ** 2).sum()], g["a_sum"])
    assert np.array_equal([b.sum(dtype=np.float64), (b.astype(np.float64) ** 2).sum()], g["b_sum"])
    c64 = a.astype(np.float64) @ b.astype(np.float64)
    return g, a, b, c64


@pytest.mark.parametrize("precision", ["fp32acc", "bf16"])
@pytest.mark.parametrize("n_dev", [1, 2])
def test_cfg1_against_reference_run(cfg1, n_dev, precision):
    g, a, b, c64 = cfg1
    c, s = run(homogeneous_machine(n_dev, dtype=np.float32, gpus=[0] * n_dev), a, b, 512, precision=precision)
    tol = TOL[precision]
    assert c.dtype == np.float32 and c.shape == (2048, 2048)
    # whole product vs float64, the reference's sampled block, its tile sums and norm
    assert rel(c, c64) <= tol
    rows, cols = g["rows"], g["cols"]
    assert rel(c[np.ix_(rows, cols)], g["c64_block"]) <= tol
    sums = c.astype(np.float64).reshape(4, 512, 4, 512).sum(axis=(1, 3))
    ref_sums_err = rel(g["c32_tiles"], g["c64_tiles"])  # the reference's own f32 run vs f64
    assert rel(sums, g["c64_tiles"]) <= max(tol, 4 * ref_sums_err)
    assert abs(np.linalg.norm(c.astype(np.float64)) / g["c64_fro"][0] - 1.0) <= tol
    # the reference's counters: 2 g^2 first-touch fetches of 512x512 fp32 tiles,
    # every other request a hit, one writeback per task
    host_fetches, bytes_host, hits, writebacks, bytes_wb, tasks = (int(x) for x in g["stats"])
    cs = s.cache
    assert s.total_tasks == tasks == sum(s.tasks_by_device.values())
    assert (cs.host_fetches, cs.bytes_host) == (host_fetches, bytes_host)
    assert cs.l1_hits + cs.l2_hits == hits
    assert (cs.writebacks, cs.bytes_writeback) == (writebacks, bytes_wb)
    assert cs.bytes_peer == cs.l2_hits * 512 * 512 * 4
    if n_dev == 1:
        assert cs.l2_hits == 0 and cs.l1_hits == hits


@pytest.mark.parametrize("precision", ["fp32acc", "bf16"])
def test_band_sampled_ragged_product(precision):
    """>= 8 sampled rows and columns in every tile band, ragged last bands in M,
    K and N, host operands through run()."""
    T = 2048
    m, k, n = 2 * T + 1000, T + 777, 3 * T + 333
    rng = np.random.default_rng(11)
    a = rng.standard_normal((m, k)).astype(np.float32)
    b = rng.standard_normal((k, n)).astype(np.float32)
    c, s = run(homogeneous_machine(1, dtype=np.float32), a, b, T, precision=precision)
    rows, cols = O.band_samples(m, T, seed=1), O.band_samples(n, T, seed=2)
    assert len(rows) >= 8 * 3 and len(cols) >= 8 * 4
    err = O.sampled_rel_error(a[rows].astype(np.float64), b[:, cols].astype(np.float64), c[np.ix_(rows, cols)])
    assert err <= TOL[precision], err
    assert s.cache.host_fetches == 3 * 2 + 2 * 4 and s.cache.writebacks == 3 * 4

