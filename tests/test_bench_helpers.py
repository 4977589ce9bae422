"""bench.py's host-side helpers on CPU: traced link rates (busy-interval union),
the headline size fallback, band-sampled parity against the oracle, the
parity gate and the summary key."""

import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
import bench  # noqa: E402


def test_trace_link_rates_union_and_rates():
    ev = [dict(kind="h2d", device=0, start_ms=0.0, end_ms=2.0), dict(kind="h2d", device=0, start_ms=1.0, end_ms=3.0),
          dict(kind="h2d", device=0, start_ms=5.0, end_ms=6.0), dict(kind="h2d", device=1, start_ms=0.0, end_ms=1.0),
          dict(kind="gemm", device=0, start_ms=0.0, end_ms=9.0)]
    r = bench.trace_link_rates(ev, {"h2d": 1_000_000, "d2h": 1, "peer": 1})
    h = r["h2d"]
    assert h["copies"] == 4 and abs(h["gb"] - 0.004) < 1e-12
    assert abs(h["busy_union_ms"] - (3.0 + 1.0 + 1.0)) < 1e-12  # [0,3] + [5,6] on device 0, [0,1] on device 1
    assert abs(h["per_copy_gbs"] - 4e6 / (6.0 * 1e6)) < 1e-9 and "peer" not in r and "gemm" not in r


def test_pick_headline_n_shrinks_to_host_memory(monkeypatch):
    monkeypatch.setattr(bench, "host_mem_available", lambda: 2 * 65536 ** 2 * 4 + 24 * 2 ** 30 + 1)
    assert bench.pick_headline_n(131072, 4096) == 65536
    monkeypatch.setattr(bench, "host_mem_available", lambda: 10 ** 13)
    assert bench.pick_headline_n(131072, 4096) == 131072


def test_band_parity_and_gate():
    from oracle import tilerun_oracle as O

    O.build_c_oracle()
    rng = np.random.default_rng(0)
    a = rng.standard_normal((300, 200)).astype(np.float32)
    b = rng.standard_normal((200, 260)).astype(np.float32)
    c = (a.astype(np.float64) @ b.astype(np.float64)).astype(np.float32)
    err, nr, nc = bench.band_parity(a, b, c, 128, seed=3)
    assert err < 1e-6 and nr == 8 + 8 + 8 and nc == 8 + 8 + 4  # the ragged last band: all of its 4 columns
    bad = c.copy()
    bad[0, 0] += 100.0  # band edges are always sampled
    err_bad, _, _ = bench.band_parity(a, b, bad, 128, seed=3)
    e = bench.parity_entry(err_bad, "fp32acc", "x")
    assert err_bad > 1e-3 and not e["ok"] and e["tol"] == 1e-5
    assert bench.parity_entry(1e-3, "bf16", "y")["ok"] and not bench.parity_entry(2e-2, "bf16", "y")["ok"]


def test_summary_fields():
    line = {"value": 400.0, "n_gpus": 1, "e2e": {"value": 390.0, "frac_of_roofline": 0.85},
            "roofline": {"frac_of_mode_peak": 0.86}, "mlp": {"samples_per_s": 5e5, "bf16_mode": {"samples_per_s": 1.3e6}},
            "parity_ok": True}
    s = bench.summarize(line)
    assert s["cfg4_e2e_tflops"] == 390.0 and s["cfg3_samples_per_s"] == 500000 and s["parity_ok"] is True
