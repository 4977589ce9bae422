"""Matrix files — the two on-disk formats of the reference (tilerun/matio.py).

* text (any suffix but ``.bin``): first line ``rows cols``, then the values in
  row-major order separated by arbitrary whitespace; written with 17
  significant digits so a float64 survives the round trip bit for bit
  (reference matio.py:26-46).
* binary (``.bin``): 16-byte header of two little-endian u64 (rows, cols),
  then the row-major little-endian float64 payload (matio.py:49-67).

B200 additions (same formats, same errors): ``load_matrix(..., pinned=True)``
reads a ``.bin`` payload straight into page-locked host memory with one
``readinto`` (no intermediate bytes object), which is what the runtime's H2D
fill path wants for host-resident operands; ``dtype=np.float32`` converts
once after the read (the files are always float64).
"""

from __future__ import annotations

import struct
from pathlib import Path

import numpy as np

from .tiles import as_matrix  # noqa: F401 (tilerun.matio name)

_HDR = struct.Struct("<QQ")  # rows, cols


def _as_2d(m) -> np.ndarray:
    a = np.asarray(m, dtype=np.float64)
    if a.ndim == 1:
        a = a.reshape(1, -1)
    if a.ndim != 2:
        raise ValueError(f"expected a 2-D matrix, got shape {a.shape}")
    return a


def _fmt_row(row) -> str:
    return " ".join(format(float(v), ".17g") for v in row)


def save_matrix_text(path, m) -> None:
    a = _as_2d(m)
    with open(path, "w") as f:
        f.write(f"{a.shape[0]} {a.shape[1]}\n")
        for row in a:
            f.write(_fmt_row(row))
            f.write("\n")


def load_matrix_text(path) -> np.ndarray:
    with open(path) as f:
        head = f.readline().split()
        if len(head) != 2:
            raise ValueError(f"{path}: first line must be 'rows cols'")
        rows, cols = int(head[0]), int(head[1])
        tokens = f.read().split()
    if len(tokens) != rows * cols:
        raise ValueError(f"{path}: {rows}x{cols} needs {rows * cols} values, file holds {len(tokens)}")
    out = np.empty(rows * cols, dtype=np.float64)
    for i, t in enumerate(tokens):
        out[i] = float(t)
    return out.reshape(rows, cols)


def save_matrix_binary(path, m) -> None:
    a = np.ascontiguousarray(_as_2d(m), dtype="<f8")
    with open(path, "wb") as f:
        f.write(_HDR.pack(a.shape[0], a.shape[1]))
        if a.size:
            f.write(memoryview(a).cast("B"))


def _host_buffer(rows: int, cols: int, pinned: bool) -> np.ndarray:
    if not pinned:
        return np.empty((rows, cols), dtype="<f8")
    from .matrix import pinned_empty

    return pinned_empty((rows, cols), np.float64)


def load_matrix_binary(path, pinned: bool = False) -> np.ndarray:
    with open(path, "rb") as f:
        head = f.read(_HDR.size)
        if len(head) < _HDR.size:
            raise ValueError(f"{path}: truncated header ({len(head)} of {_HDR.size} bytes)")
        rows, cols = _HDR.unpack(head)
        want = rows * cols * 8
        size = Path(path).stat().st_size - _HDR.size
        if size != want:
            raise ValueError(f"{path}: {rows}x{cols} needs {want} payload bytes, file holds {size}")
        out = _host_buffer(rows, cols, pinned)
        if want and f.readinto(memoryview(out).cast("B")) != want:
            raise ValueError(f"{path}: short read")
    return out


def save_matrix(path, m) -> None:
    """Format chosen by suffix: ``.bin`` binary, anything else text (matio.py:70-80)."""
    if Path(path).suffix == ".bin":
        save_matrix_binary(path, m)
    else:
        save_matrix_text(path, m)


def load_matrix(path, pinned: bool = False, dtype=np.float64) -> np.ndarray:
    if Path(path).suffix == ".bin":
        a = load_matrix_binary(path, pinned=pinned and np.dtype(dtype) == np.float64)
    else:
        a = load_matrix_text(path)
    if np.dtype(dtype) != np.float64:
        if pinned:
            from .matrix import pinned_empty

            out = pinned_empty(a.shape, np.dtype(dtype))
            out[...] = a
            return out
        return a.astype(dtype)
    if pinned and Path(path).suffix != ".bin":
        from .matrix import pinned_empty

        out = pinned_empty(a.shape, np.float64)
        out[...] = a
        return out
    return a
