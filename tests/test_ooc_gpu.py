"""Out-of-core products: A and B larger than the device's HBM tile budget, so
tiles are evicted (LRU, never pinned) and re-fetched from pinned host memory
while tasks compute (north-star item 4, BASELINE cfg4 scaled to one GPU by
capping the HBM budget instead of growing the matrices past 180 GB)."""

import numpy as np
import pytest
import torch

from oracle import tilerun_oracle as O
from paper_1511_04348_b200 import Runtime, homogeneous_machine
from paper_1511_04348_b200.matrix import pinned_empty

pytestmark = pytest.mark.gpu


def _inputs(n, seed):
    g = torch.Generator(device="cuda").manual_seed(seed)
    a = pinned_empty((n, n), np.float32)
    b = pinned_empty((n, n), np.float32)
    a[...] = torch.randn((n, n), device="cuda", generator=g).cpu().numpy()
    b[...] = torch.randn((n, n), device="cuda", generator=g).cpu().numpy()
    return a, b


def _check_slices(a, b, c, n):
    rows = np.array([0, 1, n // 3, n // 2 + 7, n - 1])
    cols = np.array([0, 5, n // 4, n - 300, n - 1])
    ref = O.gemm_slice(a, b, rows, cols)
    got = c[np.ix_(rows, cols)].astype(np.float64)
    return float(np.linalg.norm(got - ref) / np.linalg.norm(ref))


@pytest.mark.parametrize("order", ["auto", "row-major"])
def test_hbm_budget_smaller_than_operands(order):
    n, T = 8192, 1024  # 64 + 64 input tiles of 4 MiB (split planes)
    a, b = _inputs(n, 5)
    slot = 2 * T * T * 2
    overhead = (4 + 2) * 2 * T * T * 8 + 4 * T * T * 8  # per-stream buffers + staging ring
    budget = overhead + (40 + 8) * slot  # ~40 tile slots for 128 distinct input tiles
    rt = Runtime(homogeneous_machine(1, dtype=np.float32), T, hbm_budget_bytes=budget)
    rt.set_order(order)
    c, s = rt.multiply(a, b, a_uid="A", b_uid="B")
    assert _check_slices(a, b, c, n) <= 1e-5
    assert s.cache.evictions > 0
    assert s.cache.host_fetches > 2 * 8 * 8  # tiles streamed in more than once
    assert s.cache.input_requests == 2 * 8 ** 3
    rt.close()


def test_bounded_capacity_keeps_reference_semantics():
    n, T = 4096, 512
    a, b = _inputs(n, 6)
    rt = Runtime(homogeneous_machine(2, capacity_tiles=24, dtype=np.float32), T, directory_debug=True)
    c, s = rt.multiply(a, b, a_uid="A", b_uid="B")
    assert _check_slices(a, b, c, n) <= 1e-5
    assert s.cache.evictions > 0 and s.cache.input_requests == 2 * 8 ** 3
    rt.close()


@pytest.mark.parametrize("precision", ["fp32acc", "bf16"])
def test_out_of_core_kpanel_blocks_integer_exact(precision):
    """Ragged out-of-core product (A and B planes ~5x the tile budget) on one
    device: the block-wise k-panel schedule with future-aware eviction is exact
    on integer inputs, computes every task once and writes every C tile once."""
    rng = np.random.default_rng(40)
    m, k, n, T = 1400, 1900, 1250, 128  # 11 x 10 tasks, 15 k-steps; 165 + 150 input tiles
    a = rng.integers(-4, 5, size=(m, k)).astype(np.float32)
    b = rng.integers(-4, 5, size=(k, n)).astype(np.float32)
    planes = 2 if precision == "fp32acc" else 1
    slot = planes * T * T * 2
    overhead = (4 + 2) * 2 * T * T * 8 + 4 * T * T * 8
    rt = Runtime(homogeneous_machine(1, dtype=np.float32), T, precision=precision,
                 hbm_budget_bytes=overhead + (60 + 8) * slot)
    c, s = rt.multiply(a, b, a_uid="A", b_uid="B")
    assert np.array_equal(c, a.astype(np.float64) @ b.astype(np.float64))
    assert s.total_tasks == 110 and s.cache.writebacks == 110 and s.tasks_by_device == {0: 110}
    assert s.cache.input_requests == 2 * 110 * 15 and s.cache.evictions > 0
    rt.close()
