"""Dense in-core product on one GPU: one K1 launch over whole device matrices.

This is the B200 counterpart of the reference's ``DenseBackend`` product
(ann.py:62-75 -> tiles.py:197-212 ``reference_gemm``): no tiling, no
scheduler, no tile cache.  The paper's "in-core GPU" comparison point.
"""

from __future__ import annotations

from . import _native as N
from .matrix import describe, is_device_tensor

# "fp32acc": split-bf16x3 on the tensor cores (<= 1e-5); "fp32hi": split-bf16x6
# (three planes, ~10x more accurate, twice the tensor work); "bf16": one plane;
# "exact": the reference's own arithmetic (rounded multiply then rounded add per
# rank-1 update, k ascending, output dtype) on CUDA cores -- bit for bit its results
PRECISIONS = {"bf16": N.TR_PREC_BF16, "fp32acc": N.TR_PREC_FP32ACC, "fp32hi": N.TR_PREC_FP32HI,
              "exact": N.TR_PREC_EXACT}

_default_precision = None


def default_precision() -> str:
    """The precision used where a call does not name one: set_default_precision(),
    else the TR_PRECISION environment variable, else "fp32acc"."""
    import os

    p = _default_precision or os.environ.get("TR_PRECISION") or "fp32acc"
    if p not in PRECISIONS:
        raise ValueError(f"unknown precision {p!r} (TR_PRECISION); expected one of {sorted(PRECISIONS)}")
    return p


def reference_api_precision() -> str:
    """Default of the reference-semantics entry points -- tiles.accumulate_product /
    gemm_tile / reference_gemm (whose contract is the fixed k-ascending order,
    tiles.py:154-212) and the ANN backends (the reference's ANN is float64 end to
    end, ann.py:119-121): "exact", the reference's bits, unless TR_PRECISION or
    set_default_precision() names another precision."""
    import os

    if _default_precision or os.environ.get("TR_PRECISION"):
        return default_precision()
    return "exact"


def set_default_precision(p: str | None) -> None:
    """Process-wide default precision (a PRECISIONS key; None: back to the default)."""
    global _default_precision
    if p is not None and p not in PRECISIONS:
        raise ValueError(f"unknown precision {p!r}; expected one of {sorted(PRECISIONS)}")
    _default_precision = p


def precision_code(p) -> int:
    if p is None:
        p = default_precision()
    if isinstance(p, int):
        return p
    try:
        return PRECISIONS[p]
    except KeyError:
        raise ValueError(f"unknown precision {p!r}; expected one of {sorted(PRECISIONS)}") from None


def set_gemm_pairs(on: bool) -> None:
    """Select the CTA-pair (cta_group::2) kernel variant (opt-in) or single CTAs (default)."""
    N.call("tr_set_gemm_pairs", int(bool(on)))


def set_task_group(max_tasks: int) -> None:
    """Up to ``max_tasks`` (1..8) ready tasks per tile-GEMM launch for sessions created afterwards; 1 disables."""
    N.call("tr_set_task_group", int(max_tasks))


def set_splitk(max_splits: int) -> None:
    """At most ``max_splits`` (1..8) K-splits for tile GEMMs too small to fill the GPU; 1 disables."""
    N.call("tr_set_splitk", int(max_splits))


def set_small_gemm(on: bool) -> None:
    """CUDA-core kernel for tasks with output tiles <= 32 columns or contractions <= 32 (default on)."""
    N.call("tr_set_small_gemm", int(bool(on)))


def k1_die_map(gpu: int = 0) -> tuple[int, int]:
    """CTA-pair clusters of a persistent K1 launch expected on each die of GPU
    ``gpu`` (measured once per process); (0, 0) when unavailable or TR_K1_DIE=0."""
    import ctypes as C

    n0, n1 = C.c_int32(), C.c_int32()
    N.call("tr_k1_die_map", int(gpu), C.byref(n0), C.byref(n1))
    return n0.value, n1.value


def set_narrow_tc(on: bool) -> None:
    """Narrow output tiles (<= 32 columns) as the transposed product on the tensor cores (default on)."""
    N.call("tr_set_narrow_tc", int(bool(on)))


def dense_gemm(a, b, transpose_a=False, transpose_b=False, out=None, precision=None, accumulate=False,
               stream=None):
    """``out (+)= op(a) @ op(b)`` for torch CUDA tensors (float32/float64).

    Launches the sm_100a tile kernel directly on ``stream`` (default: torch's
    current stream).  Returns ``out``.
    """
    import torch

    if not (is_device_tensor(a) and is_device_tensor(b)):
        raise ValueError("dense_gemm takes CUDA tensors")
    m = a.shape[1] if transpose_a else a.shape[0]
    n = b.shape[0] if transpose_b else b.shape[1]
    if out is None:
        out = torch.zeros((m, n), dtype=a.dtype, device=a.device)
    if stream is None:
        stream = torch.cuda.current_stream(a.device)
    N.call("tr_dense_gemm", describe(a), int(transpose_a), describe(b), int(transpose_b), describe(out),
           precision_code(precision), int(accumulate), stream.cuda_stream)
    return out
