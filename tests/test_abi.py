"""The C-ABI boundary: the in-tree library loads on any host and exports every
function include/tilerun_b200.h declares; config objects round-trip."""

import ctypes
import json
import re
from pathlib import Path

import numpy as np
import pytest

import paper_1511_04348_b200 as tr
from paper_1511_04348_b200 import _native as N

ROOT = Path(__file__).resolve().parents[1]


def declared_functions():
    text = (ROOT / "include" / "tilerun_b200.h").read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"^\s*(?:const\s+)?\w+\**\s+\**(tr_\w+)\s*\(", text, flags=re.M)))


def test_header_declares_the_runtime_surface():
    names = declared_functions()
    for must in ("tr_gemm", "tr_session_create", "tr_queue_dequeue", "tr_dir_acquire_input", "tr_steal_task",
                 "tr_dense_gemm", "tr_last_error"):
        assert must in names
    assert len(names) >= 35


def test_library_exports_every_declared_symbol():
    lib = ctypes.CDLL(str(N._LIB_PATH))
    missing = [n for n in declared_functions() if not hasattr(lib, n)]
    assert not missing, missing


def test_every_declared_symbol_has_a_python_prototype():
    protos = set(N._PROTOS) | {"tr_last_error", "tr_abi_version"}
    assert set(declared_functions()) <= protos


def test_enum_constants_match_the_header():
    """Every TR_* enumerator of include/tilerun_b200.h that the Python mirror
    names has the header's value (precisions, dtypes, locations, ...)."""
    text = re.sub(r"/\*.*?\*/", "", (ROOT / "include" / "tilerun_b200.h").read_text(), flags=re.S)
    values = {}
    for body in re.findall(r"typedef\s+enum\s*\{(.*?)\}", text, flags=re.S):
        for name, val in re.findall(r"(TR_\w+)\s*=\s*(-?\w+)", body):
            values[name] = int(val, 0)
    assert values["TR_PREC_FP32HI"] == 3 and values["TR_PREC_EXACT"] == 2
    mirrored = {k: v for k, v in vars(N).items() if k in values}
    assert len(mirrored) >= 8
    assert {k: values[k] for k in mirrored} == mirrored


def test_abi_version_and_error_channel():
    assert N.ABI_VERSION == 1
    h = ctypes.c_void_p()
    st = N.lib.tr_station_create(0, 0, ctypes.byref(h))  # width 0 is a config error
    assert st == N.TR_ERR_CONFIG
    assert b"width" in N.lib.tr_last_error()


def test_no_gpu_means_loud_failure_not_fallback():
    if N.cuda_device_count() > 0:
        pytest.skip("a GPU is present")
    with pytest.raises(tr.NoDeviceError):
        tr.Runtime(tr.homogeneous_machine(1), 4)


def test_machine_config_roundtrip(tmp_path):
    m = tr.Machine([tr.DeviceSpec(0, capacity_tiles=5, slots=2, gpu=0), tr.DeviceSpec(1, flops_per_unit=3.0)],
                   tr.ProximityMatrix([[0, 2], [2, 0]], [[0, 5.0], [5.0, 0]]), dtype=np.float32)
    tr.save_machine(tmp_path / "m.json", m)
    m2 = tr.load_machine(tmp_path / "m.json")
    assert m2.to_dict() == m.to_dict() and m2.element_bytes == 4
    assert json.loads((tmp_path / "m.json").read_text())["devices"][0]["gpu"] == 0


@pytest.mark.parametrize("bad", [
    dict(device_id=-1), dict(device_id=0, kind="fpga"), dict(device_id=0, capacity_tiles=2),
    dict(device_id=0, slots=0), dict(device_id=0, kind="host-worker", capacity_tiles=4),
])
def test_device_spec_validation(bad):
    with pytest.raises(tr.ConfigError):
        tr.DeviceSpec(**bad)


def test_proximity_and_machine_validation():
    with pytest.raises(tr.ConfigError):
        tr.ProximityMatrix([[0, 1], [2, 0]], np.ones((2, 2)))
    with pytest.raises(tr.ConfigError):
        tr.Machine([tr.DeviceSpec(1)], tr.ProximityMatrix.uniform(1))
    with pytest.raises(tr.ConfigError):
        tr.Machine.from_dict({"nodevices": []})
    m = tr.homogeneous_machine(3)
    assert tr.closest_owner(0, {1, 2}, m.proximity) == 1
    assert tr.compute_cost(m.device(0), (2, 3), (3, 4)) == 2 * 2 * 3 * 4 / 1000.0
    assert tr.transfer_cost(m, tr.HOST, 0, 8192) == 1.0


def _build_c_client(tmp_path):
    import shutil
    import subprocess

    if shutil.which("gcc") is None:
        pytest.skip("needs gcc")
    exe = tmp_path / "c_client"
    lib_dir = Path(N._LIB_PATH).parent
    cmd = ["gcc", "-O2", "-std=c11", "-Wall", "-Werror", str(ROOT / "examples" / "c_client.c"),
           f"-I{ROOT / 'include'}", f"-L{lib_dir}", "-ltilerun_b200", "-lm", f"-Wl,-rpath,{lib_dir}", "-o", str(exe)]
    r = subprocess.run(cmd, capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    return exe


def test_pure_c_client_builds_against_the_header_and_library(tmp_path):
    """examples/c_client.c uses only include/tilerun_b200.h and libtilerun_b200.so
    (no Python, no torch): it compiles and links; without a GPU it exits 2."""
    import subprocess

    exe = _build_c_client(tmp_path)
    r = subprocess.run([str(exe)], capture_output=True, text=True, timeout=300)
    assert r.returncode in (0, 2), r.stdout + r.stderr


@pytest.mark.gpu
def test_pure_c_client_runs_on_the_gpu(tmp_path):
    """The C client multiplies host matrices through tr_gemm on two logical
    devices: fp32acc within 1e-5 with the reference's counters, exact bit for bit."""
    import subprocess

    exe = _build_c_client(tmp_path)
    r = subprocess.run([str(exe)], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0 and "c client ok" in r.stdout, r.stdout + r.stderr


def test_reference_module_namespaces_are_mirrored():
    """Every public name the reference's modules expose (tilerun/{scheduler,
    tiles,coherence,devices,ann,msqueue,matio}.py, including the names they
    import for their callers) resolves in the same module here."""
    import importlib

    expected = {
        "scheduler": ["Runtime", "run", "plan", "Plan", "Task", "TaskState", "Operand", "Completion", "RunStats",
                      "DeviceStats", "StealEvent", "ReservationStation", "steal_task", "write_report_json",
                      "write_report_csv", "AcquireResult", "DeviceSpec", "HOST", "accumulate_product", "compute_cost",
                      "reassemble", "transfer_cost"],
        "tiles": ["TileKey", "TiledMatrix", "partition", "reassemble", "accumulate_product", "gemm_tile",
                  "reference_gemm", "as_matrix", "encode_task", "decode_task"],
        "coherence": ["CacheDirectory", "CacheStats", "AcquireResult", "HitLevel", "closest_owner"],
        "devices": ["DeviceSpec", "Machine", "ProximityMatrix", "homogeneous_machine", "load_machine", "save_machine",
                    "compute_cost", "transfer_cost", "closest_owner", "HOST"],
        "ann": ["Layer", "Network", "DenseBackend", "TiledBackend", "train_step", "loss_gradients", "bench_pass",
                "finite_difference_gradients", "xor_dataset", "random_regression", "reference_gemm"],
        "msqueue": ["MichaelScottQueue"],
        "matio": ["save_matrix", "load_matrix", "as_matrix"],
    }
    missing = []
    for mod, names in expected.items():
        m = importlib.import_module(f"paper_1511_04348_b200.{mod}")
        missing += [f"{mod}.{n}" for n in names if not hasattr(m, n)]
    assert not missing, missing


def test_die_map_query_without_a_gpu_is_empty_not_an_error():
    import torch

    from paper_1511_04348_b200.dense import k1_die_map

    if torch.cuda.is_available():
        pytest.skip("CPU-only check")
    assert k1_die_map(0) == (0, 0)


def test_compat_tilerun_alias(monkeypatch):
    """compat/tilerun makes `import tilerun` (and its submodules) the B200 package."""
    import importlib
    import sys

    monkeypatch.syspath_prepend(str(ROOT / "compat"))
    for k in [k for k in sys.modules if k == "tilerun" or k.startswith("tilerun.")]:
        monkeypatch.delitem(sys.modules, k)
    t = importlib.import_module("tilerun")
    from tilerun.scheduler import Runtime as R2
    from tilerun.tiles import reference_gemm

    assert t.run is tr.run and R2 is tr.Runtime and reference_gemm is tr.reference_gemm
    assert t.cli.main is tr.cli.main and set(tr.__all__) <= set(dir(t))
