"""The bench.py output contract, checked on the committed final line of the
round (profiles/r2_bench_final.json) and on the argument parser: every key
the driver and the judge read is present and typed, the timing rules hold
(W >= 3, device-timed, clocks sampled), every config's parity entry is within
its tolerance, and the reference arm's flags parse."""

import json
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent


@pytest.fixture(scope="module")
def line():
    return json.loads((ROOT / "profiles" / "r2_bench_final.json").read_text().strip().splitlines()[-1])


def test_top_level_keys(line):
    for k, t in [("metric", str), ("value", float), ("unit", str), ("n_gpus", int), ("steps", int),
                 ("warmup", int), ("ms_per_step", float), ("higher_is_better", bool), ("scaling", str),
                 ("dtype", str), ("data", str), ("config", dict), ("gpu_launches", int), ("clocks", dict)]:
        assert isinstance(line[k], t), k
    assert line["warmup"] >= 3 and line["steps"] >= 1 and line["gpu_launches"] > 0
    assert line["vs_baseline"] is None  # BASELINE.md publishes no number for this metric
    assert "workload" in line["config"] and "model" not in line["config"]
    assert line["metric"] == json.loads((ROOT / "BASELINE.json").read_text())["metric"]


def test_e2e_roofline_cpu_baseline(line):
    e = line["e2e"]
    assert e["value"] > 0 and e["unit"] == line["unit"]
    assert e["h2d_bytes_per_step"] > 0 and e["d2h_bytes_per_step"] > 0
    r = line["roofline"]
    assert r["bound"] in ("hbm", "tensor") and r["unit"] in ("GB/s", "TFLOP/s")
    assert abs(r["frac"] - r["achieved"] / r["peak"]) < 1e-9 and 0 < r["frac"] < 1
    assert r["traffic"] is None or r["traffic"] > 0
    c = line["cpu_baseline"]
    assert c["kind"] in ("port", "reference") and c["cores"] >= 1 and c["value"] > 0 and c["sample"]


def test_clocks_and_parity(line):
    clk = line["clocks"]
    assert clk["samples"] > 0 and clk["sm_mhz"] > 0
    assert not {"hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown"} & set(clk["reasons"])
    assert line["parity_ok"] is True

    def entries(d):
        if "rel_fro" in d:
            yield d
        else:
            for v in d.values():
                if isinstance(v, dict):
                    yield from entries(v)

    got = list(entries(line["parity"]))
    assert len(got) >= 10
    for e in got:
        assert e["rel_fro"] <= e["tol"] and e["ok"] and e["sample"]
    for cfg in ("cfg1", "cfg2", "cfg3", "cfg4", "cfg5"):
        assert cfg in line["parity"]
    assert "256 rows x 256 cols" in line["parity"]["cfg4"]["value"]["sample"]


def test_headline_is_cfg4_and_summary_last(line):
    assert line["config"]["n"] == 131072 and line["config"]["tile"] == 4096
    assert line["e2e"]["h2d_bytes_per_step"] == 2 * 32 * 32 * 4096 * 4096 * 4
    assert list(line)[-1] == "summary" and line["summary"]["parity_ok"] is True
    assert line["links"]["h2d_gbs"] > 1 and line["roofline"]["launches"] > 0
    for leg in ("cfg2", "mlp", "mlp_wide", "mlp_wide_hetero", "inhomogeneous", "coherence", "ooc"):
        assert leg in line, leg
    assert line["mlp_wide_hetero"]["max_rel_share_error"] <= 0.10
    assert line["inhomogeneous"]["max_rel_share_error"] <= 0.10


def test_parser_defaults():
    import sys

    sys.path.insert(0, str(ROOT))
    import bench

    old = sys.argv
    try:
        sys.argv = ["bench.py"]
        a = bench.parse()
        assert (a.gpus, a.impl, a.warmup) == (1, "ours", 3) and a.steps >= 1
        sys.argv = ["bench.py", "--impl", "reference", "--gpus", "2", "--steps", "2", "--warmup", "3"]
        a = bench.parse()
        assert (a.impl, a.gpus, a.steps) == ("reference", 2, 2)
    finally:
        sys.argv = old
