"""ctypes binding of libtilerun_b200.so (include/tilerun_b200.h).

The library is built in-tree by ``_build.build()``.  Importing this module
never falls back to anything: if the library is missing the import raises,
and every call that needs a GPU raises ``NoDeviceError`` on a host without
one.
"""

from __future__ import annotations

import ctypes as C
from pathlib import Path

from .errors import CapacityError, ConfigError, NoDeviceError

_LIB_PATH = Path(__file__).resolve().parent / "libtilerun_b200.so"

# ---- enums (mirror include/tilerun_b200.h)
TR_OK, TR_ERR_CONFIG, TR_ERR_SHAPE, TR_ERR_CAPACITY, TR_ERR_RUNTIME, TR_ERR_CUDA, TR_ERR_VALUE, \
    TR_ERR_INTERNAL, TR_ERR_NODEVICE = range(9)
TR_DTYPE_F32, TR_DTYPE_F64 = 0, 1
TR_LOC_HOST, TR_LOC_DEVICE = 0, 1
TR_PREC_BF16, TR_PREC_FP32ACC, TR_PREC_EXACT, TR_PREC_FP32HI = 0, 1, 2, 3
TR_POLICY_LRU, TR_POLICY_FIFO = 0, 1
TR_HIT_L1, TR_HIT_L2, TR_HIT_MISS = 0, 1, 2
TR_SOURCE_HOST = -1
TR_KIND_ACCELERATOR, TR_KIND_HOST_WORKER = 0, 1
TR_ACT_IDENTITY, TR_ACT_SIGMOID, TR_ACT_RELU = 0, 1, 2
TR_FLAG_STEAL, TR_FLAG_COHERENCE, TR_FLAG_DEBUG, TR_FLAG_DRYRUN, TR_FLAG_FIFO, TR_FLAG_NO_PREFETCH, TR_FLAG_TRACE = \
    1, 2, 4, 8, 16, 32, 64
TR_FLAG_SIM = 128

i32, i64, u64, u8, f64 = C.c_int32, C.c_int64, C.c_uint64, C.c_uint8, C.c_double
P = C.POINTER


class DeviceSpecC(C.Structure):
    _fields_ = [("device_id", i32), ("kind", i32), ("capacity_tiles", i64), ("slots", i32), ("gpu", i32),
                ("flops_per_unit", f64), ("host_bandwidth", f64), ("sm_count", i32)]


class MachineC(C.Structure):
    _fields_ = [("n_devices", i32), ("devices", P(DeviceSpecC)), ("hops", P(i64)), ("element_bytes", i32),
                ("peer_bandwidth", P(f64)), ("transfer_latency", f64)]


class TileKeyC(C.Structure):
    _fields_ = [("matrix", u64), ("row", i64), ("col", i64)]


class CacheStatsC(C.Structure):
    _fields_ = [(n, i64) for n in ("l1_hits", "l2_hits", "host_fetches", "bytes_host", "bytes_peer",
                                   "evictions", "writebacks", "bytes_writeback")]


class AcquireResultC(C.Structure):
    _fields_ = [("level", i32), ("source", i32), ("nbytes_moved", i64), ("n_evicted", i32)]


class MatrixC(C.Structure):
    _fields_ = [("ptr", C.c_void_p), ("rows", i64), ("cols", i64), ("ld", i64), ("dtype", i32),
                ("location", i32)]


class DeviceStatsC(C.Structure):
    _fields_ = [("tasks_completed", i64), ("steals_performed", i64), ("steals_suffered", i64),
                ("peer_copies_served", i64), ("macs", i64)]


class StealEventC(C.Structure):
    _fields_ = [("thief", i32), ("victim", i32), ("task_id", i64), ("time", f64)]


class ProductC(C.Structure):
    _fields_ = [("a", MatrixC), ("a_uid", u64), ("transpose_a", i32), ("b", MatrixC), ("b_uid", u64),
                ("transpose_b", i32), ("c", MatrixC), ("c_uid", u64), ("post", i32), ("act", i32),
                ("bias", C.c_void_p), ("aux", C.c_void_p), ("ldaux", i64), ("cache_as", u64),
                ("axpy", i32), ("alpha", C.c_float), ("colsum", C.c_void_p)]


TR_POST_NONE, TR_POST_BIAS_ACT, TR_POST_ACT_GRAD = 0, 1, 2


class TraceEventC(C.Structure):
    _fields_ = [("device", i32), ("kind", i32), ("stream", i32), ("task", i64), ("matrix", u64), ("row", i64),
                ("col", i64), ("start_ms", f64), ("end_ms", f64)]


TRACE_KINDS = ("h2d", "convert", "peer", "gemm", "d2h")


class GemmReportC(C.Structure):
    _fields_ = [("grid_rows", i64), ("grid_cols", i64), ("k_steps", i64), ("total_tasks", i64),
                ("wall_seconds", f64), ("cache", CacheStatsC), ("n_steals", i64), ("gpu_launches", i64),
                ("cache_per_device", P(CacheStatsC)), ("devices", P(DeviceStatsC)),
                ("steals", P(StealEventC)), ("steals_cap", i64), ("completion", P(u8)),
                ("completion_cap", i64), ("makespan", f64)]


vp = C.c_void_p
# name -> (argtypes); every function returns int status except the two noted
_PROTOS = {
    "tr_cuda_device_count": [P(i32)],
    "tr_queue_create": [P(vp)],
    "tr_queue_destroy": [vp],
    "tr_queue_enqueue": [vp, u64],
    "tr_queue_dequeue": [vp, P(u64), P(i32)],
    "tr_queue_is_empty": [vp, P(i32)],
    "tr_dir_create": [P(MachineC), i32, i32, i32, P(vp)],
    "tr_dir_destroy": [vp],
    "tr_dir_lookup": [vp, i32, P(TileKeyC), P(i32), P(i32)],
    "tr_dir_admit": [vp, i32, P(TileKeyC), P(TileKeyC), i32, P(i32)],
    "tr_dir_pin": [vp, i32, P(TileKeyC)],
    "tr_dir_unpin": [vp, i32, P(TileKeyC)],
    "tr_dir_is_pinned": [vp, i32, P(TileKeyC), P(i32)],
    "tr_dir_residents": [vp, i32, P(TileKeyC), i64, P(i64)],
    "tr_dir_used_tiles": [vp, i32, P(i64)],
    "tr_dir_acquire_input": [vp, i32, P(TileKeyC), i64, P(AcquireResultC), P(TileKeyC), i32],
    "tr_dir_release_input": [vp, i32, P(TileKeyC)],
    "tr_dir_admit_output": [vp, i32, P(TileKeyC), P(TileKeyC), i32, P(i32)],
    "tr_dir_release_output": [vp, i32, P(TileKeyC), i64],
    "tr_dir_stats": [vp, P(CacheStatsC), P(CacheStatsC)],
    "tr_dir_check_invariants": [vp],
    "tr_station_create": [i32, i32, P(vp)],
    "tr_station_destroy": [vp],
    "tr_station_refill": [vp, vp, P(u64), i32, P(i32)],
    "tr_station_pop_for_run": [vp, P(u64), P(i32)],
    "tr_station_try_steal": [vp, P(u64), P(i32)],
    "tr_station_reserved_count": [vp, P(i32)],
    "tr_steal_task": [i32, P(vp), i32, P(u64), P(i32), P(i32)],
    "tr_session_create": [P(MachineC), i32, i32, C.c_uint32, i64, P(vp)],
    "tr_session_destroy": [vp],
    "tr_session_directory": [vp, P(vp)],
    "tr_gemm": [vp, P(MatrixC), u64, i32, P(MatrixC), u64, i32, P(MatrixC), u64, P(GemmReportC)],
    "tr_gemm_shard": [vp, P(MatrixC), u64, i32, P(MatrixC), u64, i32, P(MatrixC), u64, i64, i64,
                      P(GemmReportC)],
    "tr_gemm_batch": [vp, i32, P(ProductC), P(GemmReportC)],
    "tr_session_kernel_ms": [vp, P(f64)],
    "tr_session_lock_stats": [vp, i32, P(i64)],
    "tr_session_span_ms": [vp, P(f64)],
    "tr_session_trace": [vp, vp, i64, P(i64)],
    "tr_session_set_inflight": [vp, i32],
    "tr_session_set_order": [vp, i32],
    "tr_release_cached_memory": [],
    "tr_dense_gemm": [P(MatrixC), i32, P(MatrixC), i32, P(MatrixC), i32, i32, vp],
    "tr_set_gemm_pairs": [i32],
    "tr_set_gemm_multicast": [i32],
    "tr_k1_die_map": [i32, C.POINTER(C.c_int32), C.POINTER(C.c_int32)],
    "tr_set_splitk": [i32],
    "tr_set_small_gemm": [i32],
    "tr_set_narrow_tc": [i32],
    "tr_set_task_group": [i32],
    "tr_mlp_bias_act": [vp, vp, vp, i64, i64, i32, vp],
    "tr_mlp_act_grad": [vp, vp, vp, vp, i64, i32, vp],
    "tr_mlp_mse_grad": [vp, vp, vp, i64, vp, vp],
    "tr_mlp_mse_grad_global": [vp, vp, vp, i64, i64, vp, vp],
    "tr_mlp_colsum": [vp, i64, i64, vp, vp],
    "tr_mlp_colsum_finish": [vp, i64, i64, vp, vp],
    "tr_mlp_sgd": [vp, vp, i64, C.c_float, vp],
    "tr_session_set_external_stream": [vp, vp, i32],
    "tr_session_set_async": [vp, i32],
    "tr_session_sim_now": [vp, P(f64)],
    "tr_session_forget": [vp, u64, P(i64)],
}


def _load():
    if not _LIB_PATH.exists():
        raise ImportError(
            f"{_LIB_PATH.name} is not built; run paper_1511_04348_b200._build.build() "
            "(there is no pure-Python fallback)")
    lib = C.CDLL(str(_LIB_PATH))
    lib.tr_last_error.restype = C.c_char_p
    lib.tr_last_error.argtypes = []
    lib.tr_abi_version.restype = C.c_int
    lib.tr_abi_version.argtypes = []
    for name, args in _PROTOS.items():
        fn = getattr(lib, name)
        fn.restype = C.c_int
        fn.argtypes = args
    return lib


lib = _load()
ABI_VERSION = lib.tr_abi_version()


class NativeError(RuntimeError):
    """CUDA / internal failure reported by the native runtime."""


def check(status: int) -> None:
    if status == TR_OK:
        return
    msg = (lib.tr_last_error() or b"").decode(errors="replace")
    if status == TR_ERR_CONFIG:
        raise ConfigError(msg)
    if status in (TR_ERR_SHAPE, TR_ERR_VALUE):
        raise ValueError(msg)
    if status == TR_ERR_CAPACITY:
        raise CapacityError(msg)
    if status == TR_ERR_RUNTIME:
        raise RuntimeError(msg)
    if status == TR_ERR_NODEVICE:
        raise NoDeviceError(msg)
    if status == TR_ERR_INTERNAL:
        raise AssertionError(msg)
    raise NativeError(msg)


def call(name: str, *args) -> None:
    check(getattr(lib, name)(*args))


def cuda_device_count() -> int:
    n = i32(0)
    call("tr_cuda_device_count", C.byref(n))
    return n.value
