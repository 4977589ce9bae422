"""The tile cache's coherence modes on the GPU at hardware scale (SURVEY §8f
row 4): the reference's acceptance criterion C2 (test_acceptance.py:95-113,
SPEC.md:574) with real H2D copies -- coherence on fetches every input tile once
(2 g^2 = 512 host fetches at g = 16), the --no-coherence bypass fetches every
request (2 g^3 = 8192) -- and the FIFO eviction policy (coherence.py:95-99)
against the oracle's directory model."""

import numpy as np
import pytest

from oracle import tilerun_oracle as O
from paper_1511_04348_b200 import Runtime, homogeneous_machine, run

pytestmark = pytest.mark.gpu


def int_matrix(rng, r, c):
    # integer-valued float32: exact in bf16 planes and in fp32 sums (|sum| < 2^24)
    return rng.integers(-4, 5, size=(r, c)).astype(np.float32)


def test_c2_coherence_vs_bypass_g16():
    g, T = 16, 1024
    rng = np.random.default_rng(2)
    a, b = int_matrix(rng, g * T, g * T), int_matrix(rng, g * T, g * T)
    rows = np.arange(0, g * T, 509)
    ref = a[rows].astype(np.float64) @ b.astype(np.float64)
    machine = homogeneous_machine(2, dtype=np.float32, gpus=[0, 0])
    c, s = run(machine, a, b, T, coherence=True)
    assert np.array_equal(c[rows], ref)
    assert s.cache.host_fetches == 2 * g * g == 512 and s.cache.evictions == 0
    assert s.cache.bytes_host == 512 * T * T * 4
    c, s = run(machine, a, b, T, coherence=False)
    assert np.array_equal(c[rows], ref)
    assert s.cache.host_fetches == 2 * g ** 3 == 8192 == 16 * 512
    assert s.cache.l1_hits == s.cache.l2_hits == 0 and s.cache.bytes_host == 8192 * T * T * 4


@pytest.mark.parametrize("policy", ["fifo", "lru"])
def test_bounded_cache_policy_counters_match_oracle(policy):
    """One device, capacity 3 (the reference's minimum: one A, one B, one C tile):
    every eviction decision follows the policy, so the counters are the oracle
    model's exactly; the product is exact on integer data."""
    T, m, k, n = 256, 5 * 256, 4 * 256 + 100, 3 * 256
    rng = np.random.default_rng(12)
    a, b = int_matrix(rng, m, k), int_matrix(rng, k, n)
    with Runtime(homogeneous_machine(1, capacity_tiles=3, dtype=np.float32), T, policy=policy,
                 directory_debug=True) as rt:
        c, s = rt.multiply(a, b, a_uid="A", b_uid="B", c_uid="C")
    assert np.array_equal(c, a.astype(np.float64) @ b.astype(np.float64))
    want = O.run_schedule_single_device(m, k, n, T, capacity=3, element_bytes=4, policy=policy)
    assert s.cache.as_dict() == want and want["evictions"] > 0


def test_fifo_and_lru_differ_where_the_model_says():
    """A 4-tile cache on a 4 x 2 task grid (k = 1): LRU refreshes the B tile each
    row reuses, FIFO evicts it -- 9 host fetches / 7 hits against 8 / 8; each
    run's counters equal its own oracle model exactly."""
    T = 128
    rng = np.random.default_rng(13)
    a, b = int_matrix(rng, 4 * T, T), int_matrix(rng, T, 2 * T)
    got = {}
    for policy in ("lru", "fifo"):
        with Runtime(homogeneous_machine(1, capacity_tiles=4, dtype=np.float32), T, policy=policy) as rt:
            c, s = rt.multiply(a, b, a_uid="A", b_uid="B", c_uid="C")
        assert np.array_equal(c, a.astype(np.float64) @ b.astype(np.float64))
        got[policy] = s.cache.as_dict()
        assert got[policy] == O.run_schedule_single_device(4 * T, T, 2 * T, T, capacity=4, element_bytes=4,
                                                          policy=policy)
    assert (got["lru"]["host_fetches"], got["fifo"]["host_fetches"]) == (9, 8)
