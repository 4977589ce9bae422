"""Matrix descriptors for the C ABI and pinned host buffers.

Host matrices are numpy arrays (the reference's type, tiles.py:37-44); device
matrices are torch CUDA tensors.  torch is used here only as the allocator of
device memory and page-locked host memory.
"""

from __future__ import annotations

import numpy as np

from . import _native as N


def _torch():
    import torch

    return torch


class ShapeOnly:
    """A matrix known by shape and dtype only, with no data: an operand for
    ``mode="sim"`` / ``"dryrun"`` runs with ``compute=False``, which schedule,
    count and time a product without reading it.  A computing run rejects it
    (ValueError) instead of reading memory that does not exist."""

    ndim = 2

    def __init__(self, rows: int, cols: int, dtype=np.float32):
        if rows < 1 or cols < 1:
            raise ValueError(f"need a non-empty 2-D shape, got ({rows}, {cols})")
        self.shape = (int(rows), int(cols))
        self.dtype = np.dtype(dtype)
        dtype_code(self.dtype)


def is_device_tensor(x) -> bool:
    t = type(x)
    return t.__module__.startswith("torch") and getattr(x, "is_cuda", False)


def dtype_code(dt) -> int:
    s = str(dt)
    if s in ("float32", "torch.float32"):
        return N.TR_DTYPE_F32
    if s in ("float64", "torch.float64"):
        return N.TR_DTYPE_F64
    raise ValueError(f"unsupported element dtype {dt} (float32 / float64 only)")


def describe(x) -> N.MatrixC:
    """MatrixC for a 2-D row-major numpy array (host) or torch CUDA tensor (device)."""
    if is_device_tensor(x):
        if x.dim() != 2:
            raise ValueError(f"expected a 2-D matrix, got shape {tuple(x.shape)}")
        if x.stride(1) != 1 or x.stride(0) < max(1, x.shape[1]):
            raise ValueError("device matrix must be row-major with unit column stride")
        return N.MatrixC(x.data_ptr(), x.shape[0], x.shape[1], x.stride(0), dtype_code(x.dtype), N.TR_LOC_DEVICE)
    a = np.asarray(x)
    if a.ndim != 2:
        raise ValueError(f"expected a 2-D matrix, got shape {a.shape}")
    if not row_major_view(a):
        raise ValueError("host matrix must be row-major with unit column stride (a C-contiguous array or a "
                         "row/column slice of one)")
    ld = max(a.shape[1], 1) if a.shape[0] <= 1 else a.strides[0] // a.itemsize
    return N.MatrixC(a.ctypes.data, a.shape[0], a.shape[1], ld, dtype_code(a.dtype), N.TR_LOC_HOST)


def row_major_view(a: np.ndarray) -> bool:
    """True for a C-contiguous array or a sub-block view of one (unit column
    stride, row stride a positive multiple of the element size covering a row):
    the runtime reads such views in place with pitched copies (ld = row stride)."""
    if a.flags.c_contiguous:
        return True
    if a.shape[1] > 1 and a.strides[1] != a.itemsize:
        return False
    return a.shape[0] <= 1 or (a.strides[0] > 0 and a.strides[0] % a.itemsize == 0
                               and a.strides[0] // a.itemsize >= a.shape[1])


def pinned_empty(shape, dtype=np.float32) -> np.ndarray:
    """A numpy array backed by page-locked host memory (cudaHostAlloc via torch).

    The array keeps the owning tensor alive through its ``base``.
    """
    torch = _torch()
    tdt = {np.dtype(np.float32): torch.float32, np.dtype(np.float64): torch.float64}[np.dtype(dtype)]
    t = torch.empty(tuple(shape), dtype=tdt, pin_memory=True)
    return t.numpy()


def pinned_zeros(shape, dtype=np.float32) -> np.ndarray:
    a = pinned_empty(shape, dtype)
    a.fill(0)
    return a


def host_pinning_available() -> bool:
    try:
        return N.cuda_device_count() > 0
    except Exception:
        return False
