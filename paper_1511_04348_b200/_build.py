"""In-tree build of the native extension (libtilerun_b200.so) for sm_100a.

Every CUDA/C++ source under csrc/ is compiled with nvcc
(-gencode arch=compute_100a,code=sm_100a -lineinfo) and linked into ONE
shared library with a plain C ABI (include/tilerun_b200.h).  cudart is linked
statically, so the library loads on a host without a GPU or driver (the C-ABI
tests on CPU rely on that); calls that need a device then fail loudly with
TR_ERR_NODEVICE.
"""

from __future__ import annotations

import concurrent.futures as cf
import os
import shutil
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
BUILD = ROOT / "build" / "native"
LIB = PKG / "libtilerun_b200.so"

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
COMMON = ["-O3", "-std=c++17", "-lineinfo", "-Xcompiler", "-fPIC,-Wall,-Wno-unused-function",
          f"-I{ROOT / 'include'}"]


def _nvcc() -> str:
    for cand in (os.environ.get("NVCC"), shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and Path(cand).exists():
            return cand
    raise RuntimeError("nvcc not found: the B200 build needs the CUDA 12.9 toolkit")


def _sources():
    return sorted(list(CSRC.glob("*.cu")) + list(CSRC.glob("*.cpp")))


def _headers():
    return sorted(list(CSRC.glob("*.h")) + list(CSRC.glob("*.cuh")) + list((ROOT / "include").glob("*.h")))


def _compile(src: Path, nvcc: str, verbose: bool) -> Path:
    obj = BUILD / (src.name + ".o")
    cmd = [nvcc, *ARCH, *COMMON, "-c", str(src), "-o", str(obj)]
    if src.suffix == ".cu":
        cmd.insert(1, "-Xptxas=-v" if verbose else "-Xptxas=-O3")
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc failed on {src.name}:\n{r.stdout}\n{r.stderr}")
    if verbose and r.stderr:
        sys.stderr.write(r.stderr)
    return obj


def build(force: bool = False, verbose: bool = False) -> Path:
    """Compile (incrementally) and link libtilerun_b200.so; returns its path."""
    hdr_mtime = max((h.stat().st_mtime for h in _headers()), default=0.0)
    src_mtime = max((s.stat().st_mtime for s in _sources()), default=0.0)
    if not force and LIB.exists() and LIB.stat().st_mtime >= max(hdr_mtime, src_mtime):
        return LIB  # up to date (also the case on a GPU box that received the prebuilt .so)
    nvcc = _nvcc()
    BUILD.mkdir(parents=True, exist_ok=True)
    todo = []
    objs = []
    for src in _sources():
        obj = BUILD / (src.name + ".o")
        objs.append(obj)
        if force or not obj.exists() or obj.stat().st_mtime < max(src.stat().st_mtime, hdr_mtime):
            todo.append(src)
    if todo:
        with cf.ThreadPoolExecutor(max_workers=min(8, len(todo))) as ex:
            list(ex.map(lambda s: _compile(s, nvcc, verbose), todo))
    newest = max(o.stat().st_mtime for o in objs)
    if force or todo or not LIB.exists() or LIB.stat().st_mtime < newest:
        tmp = LIB.with_suffix(".so.tmp")
        cmd = [nvcc, *ARCH, "-shared", "-o", str(tmp), *map(str, objs), "-lpthread", "-ldl", "-lrt"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"link failed:\n{r.stdout}\n{r.stderr}")
        os.replace(tmp, LIB)
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
