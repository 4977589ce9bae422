"""ThreadSanitizer run of the runtime's host-side concurrency (race
detection: TSAN on the C++ units): the lock-free MS queue, the reservation
stations with stealing and the tile-cache directory with its debug invariants,
stressed from 8 threads (tests/native/tsan_stress.cpp).  CPU only."""

import os
import shutil
import subprocess
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
CSRC = ROOT / "paper_1511_04348_b200" / "csrc"
CUDA = Path(os.environ.get("CUDA_HOME", "/usr/local/cuda"))


def test_host_concurrency_under_tsan(tmp_path):
    if shutil.which("g++") is None or not (CUDA / "include" / "cuda_runtime.h").exists():
        pytest.skip("needs g++ and the CUDA headers")
    exe = tmp_path / "tsan_stress"
    cmd = ["g++", "-std=c++17", "-O1", "-g", "-fsanitize=thread", f"-I{CUDA / 'include'}", f"-I{CSRC}",
           str(ROOT / "tests" / "native" / "tsan_stress.cpp"), str(CSRC / "msqueue.cpp"), str(CSRC / "directory.cpp"),
           f"-L{CUDA / 'lib64'}", "-lcudart", "-lpthread", "-o", str(exe)]
    build = subprocess.run(cmd, capture_output=True, text=True)
    if build.returncode != 0 and "tsan" in build.stderr.lower():
        pytest.skip("no ThreadSanitizer runtime: " + build.stderr[-200:])
    assert build.returncode == 0, build.stderr[-2000:]
    env = dict(os.environ, TSAN_OPTIONS="halt_on_error=1 exitcode=66",
               LD_LIBRARY_PATH=f"{CUDA / 'lib64'}:{os.environ.get('LD_LIBRARY_PATH', '')}")
    run = subprocess.run([str(exe)], capture_output=True, text=True, env=env, timeout=600)
    out = run.stdout + run.stderr
    assert "ThreadSanitizer" not in out, out[-4000:]
    assert run.returncode == 0 and "tsan stress ok" in out, out[-4000:]
