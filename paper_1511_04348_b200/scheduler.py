"""Planning, reservation stations, the GPU session (Runtime) and run reports.

Python face of the native runtime (csrc/session.cpp), API-compatible with the
reference scheduler (pkg/src/tilerun/scheduler.py):

* ``plan`` builds one task per output tile with row-major ids and every task
  enqueued up front (scheduler.py:165-197).
* ``Runtime(machine, tile_size, ...)`` is a session whose tile cache and uid
  identities persist across ``multiply`` calls (scheduler.py:522-612).  Each
  product runs on one pinned C++ worker thread per logical device; a device's
  reservation-station entries feed its CUDA streams; each task is ONE
  tcgen05 GEMM launch over all its k-steps with inputs resolved L1 (own HBM)
  -> L2 (peer HBM over NVLink) -> host (pinned DRAM).
* ``mode``: "gpu" (default) and "threaded" (its alias: one real worker thread
  per device) run on B200s; "dryrun" runs the scheduler and directory only
  (no CUDA, result is None) for schedule-parity tests.  The reference's
  discrete-event "sim" engine is not part of the hardware build.
"""

from __future__ import annotations

import csv
import ctypes as C
import json
import threading
import time
from dataclasses import dataclass, field
from enum import Enum

import numpy as np

from . import _native as N
from .coherence import AcquireResult, CacheDirectory, CacheStats, UidTable  # noqa: F401 (tilerun.scheduler names)
from .dense import default_precision, precision_code, reference_api_precision
from .devices import HOST, DeviceSpec, Machine, compute_cost, transfer_cost  # noqa: F401 (tilerun.scheduler names)
from .errors import NoDeviceError
from .matrix import ShapeOnly, describe, is_device_tensor, pinned_empty, pinned_zeros
from .msqueue import MichaelScottQueue
from .tiles import TiledMatrix, TileKey, accumulate_product, decode_task, partition, reassemble  # noqa: F401

SCHEMA_VERSION = 1
MODES = ("gpu", "threaded", "dryrun", "sim")


class TaskState(Enum):
    QUEUED = "queued"
    RESERVED = "reserved"
    RUNNING = "running"
    DONE = "done"


@dataclass
class Task:
    task_id: int
    row: int
    col: int
    k_steps: int
    state: TaskState = TaskState.QUEUED


class Completion:
    """Exactly-once task bitmap with the contract of scheduler.py:70-96 (a second
    mark raises RuntimeError; ``all_done`` gates the result).  Stored as one byte
    per task -- the layout of the native runtime's bitmap
    (tr_gemm_report.completion, set by an atomic exchange per task), so
    ``Completion.of(bits)`` wraps a product's native snapshot without copying."""

    def __init__(self, n_tasks: int):
        self._bits = np.zeros(max(0, int(n_tasks)), dtype=np.uint8)
        self._guard = threading.Lock()

    @classmethod
    def of(cls, bits) -> "Completion":
        c = cls(0)
        c._bits = np.asarray(bits, dtype=np.uint8)
        return c

    def mark(self, task_id: int) -> None:
        with self._guard:
            if self._bits[task_id]:
                raise RuntimeError(f"task {task_id} executed twice")
            self._bits[task_id] = 1

    def all_done(self) -> bool:
        return bool(self._bits.all())

    @property
    def done_count(self) -> int:
        return int(np.count_nonzero(self._bits))

    def snapshot(self) -> list[bool]:
        return self._bits.astype(bool).tolist()


@dataclass
class Operand:
    """A tiled matrix as seen by the planner, optionally transposed (scheduler.py:99-138).

    Tile (i, k) of the transposed operand is stored tile (k, i); the cache key
    names STORED coordinates so both readings share tile identity.  On the
    GPU the transposition is a TMA/UMMA layout choice (MN-major operand), never
    a copy.
    """

    tiled: TiledMatrix
    uid: str
    transposed: bool = False

    @property
    def grid_rows(self) -> int:
        return self.tiled.grid_cols if self.transposed else self.tiled.grid_rows

    @property
    def grid_cols(self) -> int:
        return self.tiled.grid_rows if self.transposed else self.tiled.grid_cols

    @property
    def element_shape(self) -> tuple[int, int]:
        r, c = self.tiled.shape
        return (c, r) if self.transposed else (r, c)

    def tile_view(self, i: int, j: int):
        return self.tiled.tile(j, i).T if self.transposed else self.tiled.tile(i, j)

    def key(self, i: int, j: int) -> TileKey:
        return TileKey(self.uid, j, i) if self.transposed else TileKey(self.uid, i, j)

    def tile_nbytes(self, i: int, j: int, element_bytes: int) -> int:
        r, c = self.tiled.tile_shape(j, i) if self.transposed else self.tiled.tile_shape(i, j)
        return r * c * element_bytes


def _as_operand(x, uid: str) -> Operand:
    return x if isinstance(x, Operand) else Operand(x, uid)


@dataclass
class Plan:
    a: Operand
    b: Operand
    c: Operand
    tile_size: int
    grid_rows: int
    grid_cols: int
    k_steps: int
    tasks: list[Task]
    queue: MichaelScottQueue
    completion: Completion

    @property
    def total_tasks(self) -> int:
        return len(self.tasks)


def _zeros_like_output(a: Operand, rows: int, cols: int, pinned: bool, zero: bool = True):
    """Output storage where A lives.  The runtime overwrites every element
    (first k-chunk stores, later chunks accumulate), so it skips zeroing."""
    base = a.tiled.base
    if is_device_tensor(base):
        import torch

        alloc = torch.zeros if zero else torch.empty
        return alloc((rows, cols), dtype=base.dtype, device=base.device)
    dt = np.asarray(base).dtype
    if pinned and dt in (np.float32, np.float64):
        return pinned_zeros((rows, cols), dt) if zero else pinned_empty((rows, cols), dt)
    return np.zeros((rows, cols), dtype=dt)


def plan(a, b, a_uid: str = "A", b_uid: str = "B", c_uid: str = "C", *, _pinned_output: bool = False) -> Plan:
    """One task per output tile, all enqueued row-major (scheduler.py:165-197)."""
    a = _as_operand(a, a_uid)
    b = _as_operand(b, b_uid)
    if a.tiled.tile_size != b.tiled.tile_size:
        raise ValueError(f"tile sizes differ: {a.tiled.tile_size} vs {b.tiled.tile_size}")
    am, ak = a.element_shape
    bk, bn = b.element_shape
    if ak != bk:
        raise ValueError(f"inner dimensions differ: {a.element_shape} x {b.element_shape}")
    t = a.tiled.tile_size
    c = Operand(partition(_zeros_like_output(a, am, bn, _pinned_output), t), c_uid)
    gr, gc = c.grid_rows, c.grid_cols
    k_steps = a.grid_cols
    queue = MichaelScottQueue()
    tasks = []
    for tid in range(gr * gc):
        i, j = decode_task(tid, gc, gr)
        tasks.append(Task(tid, i, j, k_steps))
        queue.enqueue(tid)
    return Plan(a=a, b=b, c=c, tile_size=t, grid_rows=gr, grid_cols=gc, k_steps=k_steps, tasks=tasks, queue=queue,
                completion=Completion(len(tasks)))


def _execute_task(machine: Machine, plan_: Plan, directory: CacheDirectory, dev, task: Task):
    """One task by hand, outside a Runtime (the reference's internal helper,
    scheduler.py:371-410): the output tile is admitted and pinned for the task;
    per k-step A then B are acquired through ``directory``, ``c += a @ b`` runs
    as one GPU tile product (tiles.accumulate_product) and both inputs are
    released; then the output is written back and released, the completion
    bitmap marked (a second execution raises) and the task is DONE.  Returns
    ``(steps, writeback)`` in simulated time units, [(fetch, compute)] per
    k-step, from the machine's cost model (devices.py:255-283).  Runtime.multiply
    does all of this natively; this is for callers that drive the pieces."""
    from .devices import HOST, compute_cost, transfer_cost
    from .tiles import accumulate_product

    did, eb = dev.device_id, machine.element_bytes
    task.state = TaskState.RUNNING
    i, j = task.row, task.col
    c_key, c_view = plan_.c.key(i, j), plan_.c.tile_view(i, j)
    directory.admit_output(did, c_key)
    steps = []
    for k in range(task.k_steps):
        keys = (plan_.a.key(i, k), plan_.b.key(k, j))
        got = (directory.acquire_input(did, keys[0], plan_.a.tile_nbytes(i, k, eb)),
               directory.acquire_input(did, keys[1], plan_.b.tile_nbytes(k, j, eb)))
        fetch = sum(transfer_cost(machine, r.source, did, r.nbytes_moved) for r in got)
        a_view, b_view = plan_.a.tile_view(i, k), plan_.b.tile_view(k, j)
        accumulate_product(a_view, b_view, c_view)
        steps.append((fetch, compute_cost(dev, a_view.shape, b_view.shape)))
        for key in keys:
            directory.release_input(did, key)
    nbytes = int(np.prod(np.shape(c_view))) * eb
    writeback = transfer_cost(machine, did, HOST, nbytes)
    directory.release_output(did, c_key, nbytes)
    plan_.completion.mark(task.task_id)
    task.state = TaskState.DONE
    return steps, writeback


# ----------------------------------------------------------------- stations


class ReservationStation:
    """Fixed-width buffer of reserved task ids (scheduler.py:200-236), native.

    The owner pops the front, a thief the back; one lock per station.
    """

    def __init__(self, owner: int, width: int):
        self.owner = owner
        self.width = width
        h = C.c_void_p()
        N.call("tr_station_create", int(owner), int(width), C.byref(h))
        self._h = h
        self._buf = (N.u64 * max(1, width))()
        self._held: dict = {}  # native handle -> the reserved value

    def __del__(self):
        if getattr(self, "_h", None) is not None:
            N.lib.tr_station_destroy(self._h)
            self._h = None

    def refill(self, queue: MichaelScottQueue) -> list:
        """Pull from the global queue until full; returns the values taken."""
        # The native station stores queue handles; translate back to the objects.
        n = N.i32()
        N.call("tr_station_refill", self._h, queue.handle, self._buf, self.width, C.byref(n))
        pulled = []
        for i in range(n.value):
            hid = int(self._buf[i])
            val = queue._objs.pop(hid)
            self._held[hid] = val
            pulled.append(val)
        return pulled

    def _one(self, fn) -> object | None:
        v, got = N.u64(), N.i32()
        N.call(fn, self._h, C.byref(v), C.byref(got))
        return self._held.pop(int(v.value)) if got.value else None

    def pop_for_run(self):
        return self._one("tr_station_pop_for_run")

    def try_steal(self):
        return self._one("tr_station_try_steal")

    def reserved_count(self) -> int:
        n = N.i32()
        N.call("tr_station_reserved_count", self._h, C.byref(n))
        return n.value


def steal_task(thief: int, stations: dict) -> tuple:
    """Steal one reserved task from the most-loaded peer, ties to the lowest id
    (scheduler.py:239-249).  Returns (task_id, victim) or (None, None)."""
    ids = sorted(stations)
    arr = (C.c_void_p * len(ids))(*[stations[d]._h.value for d in ids])
    v, victim, got = N.u64(), N.i32(), N.i32()
    N.call("tr_steal_task", int(thief), arr, len(ids), C.byref(v), C.byref(victim), C.byref(got))
    if not got.value:
        return None, None
    return stations[victim.value]._held.pop(int(v.value)), victim.value


# ----------------------------------------------------------------- stats


@dataclass
class StealEvent:
    thief: int
    victim: int
    task_id: int
    queue_empty_observed: bool = True
    time: float | None = None


@dataclass
class DeviceStats:
    device_id: int
    kind: str
    tasks_completed: int = 0
    steals_performed: int = 0
    steals_suffered: int = 0
    peer_copies_served: int = 0  # B200: L2 fills sourced from this device (not in report schema v1)
    macs: int = 0  # B200: rows x cols x K summed over its tasks (work share of unequal tasks)


@dataclass
class RunStats:
    """Per-product report (scheduler.py:270-325) plus GPU measurements."""

    mode: str
    tile_size: int
    grid_rows: int
    grid_cols: int
    k_steps: int
    total_tasks: int
    steal_enabled: bool
    coherence_enabled: bool
    seed: int | None
    devices: dict[int, DeviceStats]
    cache: CacheStats
    cache_per_device: dict[int, CacheStats]
    makespan: float | None
    wall_elapsed: float
    steal_events: list[StealEvent] = field(default_factory=list)
    precision: str = "fp32acc"
    gpu_launches: int = 0
    kernel_ms: dict[int, float] = field(default_factory=dict)  # sum of tile-GEMM kernel durations
    span_ms: dict[int, float] = field(default_factory=dict)  # device-side span of the product
    trace: list = field(default_factory=list)  # Runtime(trace=True): device timeline of the product
    completion: Completion | None = None  # the native exactly-once bitmap of the product

    @property
    def tasks_by_device(self) -> dict[int, int]:
        return {d: s.tasks_completed for d, s in self.devices.items()}

    def to_report_dict(self) -> dict:
        return {
            "schema_version": SCHEMA_VERSION,
            "mode": self.mode,
            "tile_size": self.tile_size,
            "grid": {"rows": self.grid_rows, "cols": self.grid_cols, "k_steps": self.k_steps},
            "total_tasks": self.total_tasks,
            "steal": self.steal_enabled,
            "coherence": self.coherence_enabled,
            "seed": self.seed,
            "makespan": self.makespan,
            "wall_elapsed": self.wall_elapsed,
            "steals": len(self.steal_events),
            "devices": [
                {"device_id": s.device_id, "kind": s.kind, "tasks_completed": s.tasks_completed,
                 "steals_performed": s.steals_performed, "steals_suffered": s.steals_suffered}
                for s in self.devices.values()
            ],
            "cache": {**self.cache.as_dict(),
                      "per_device": {str(d): s.as_dict() for d, s in self.cache_per_device.items()}},
            "gpu": {"precision": self.precision, "launches": self.gpu_launches,
                    "kernel_ms": {str(d): v for d, v in self.kernel_ms.items()}},
        }


def write_report_json(stats: RunStats, path) -> None:
    with open(path, "w") as f:
        json.dump(stats.to_report_dict(), f, indent=2)
        f.write("\n")


_CSV_FIELDS = ["device_id", "kind", "tasks_completed", "steals_performed", "steals_suffered", "l1_hits", "l2_hits",
               "host_fetches", "bytes_host", "bytes_peer", "evictions", "writebacks", "bytes_writeback"]


def write_report_csv(stats: RunStats, path) -> None:
    """One row per device plus a total row (scheduler.py:341-361)."""
    with open(path, "w", newline="") as f:
        w = csv.DictWriter(f, fieldnames=_CSV_FIELDS)
        w.writeheader()
        for did, ds in sorted(stats.devices.items()):
            cs = stats.cache_per_device.get(did, CacheStats())
            w.writerow({"device_id": did, "kind": ds.kind, "tasks_completed": ds.tasks_completed,
                        "steals_performed": ds.steals_performed, "steals_suffered": ds.steals_suffered,
                        **{k: v for k, v in cs.as_dict().items() if k in _CSV_FIELDS}})
        w.writerow({"device_id": "total", "kind": "",
                    "tasks_completed": sum(d.tasks_completed for d in stats.devices.values()),
                    "steals_performed": sum(d.steals_performed for d in stats.devices.values()),
                    "steals_suffered": sum(d.steals_suffered for d in stats.devices.values()),
                    **{k: v for k, v in stats.cache.as_dict().items() if k in _CSV_FIELDS}})


# ----------------------------------------------------------------- the session


def _host_matrix(x):
    """Host operand as a row-major float32/float64 array (ints widen to f64); a
    row/column slice of a row-major array is read in place (no copy)."""
    from .matrix import row_major_view

    a = np.asarray(x)
    if a.dtype not in (np.float32, np.float64):
        a = a.astype(np.float64)
    return a if a.ndim == 2 and row_major_view(a) else np.ascontiguousarray(a)


class Runtime:
    """A session: one machine, one HBM tile cache, any number of products.

    Signature follows scheduler.py:531-533, plus ``precision`` ("fp32acc" |
    "fp32hi" | "bf16" | "exact"; None = ``dense.default_precision()``, or
    ``dense.reference_api_precision()`` ("exact") in mode "sim") and
    ``hbm_budget_bytes`` (per GPU; 0 = 80% of free HBM).
    """

    def __init__(self, machine: Machine, tile_size: int, mode: str = "gpu", steal: bool = True,
                 coherence: bool = True, seed: int | None = None, directory_debug: bool = False,
                 precision: str | None = None, hbm_budget_bytes: int = 0, policy: str = "lru",
                 fetch_ahead: bool = True, trace: bool = False, compute: bool = True):
        if mode not in MODES:
            raise ValueError(f"unknown mode {mode!r}")
        if tile_size < 1:
            raise ValueError(f"tile_size must be >= 1, got {tile_size}")
        self.machine = machine
        self.tile_size = tile_size
        self.mode = mode
        self.steal = steal
        self.coherence = coherence
        self.seed = seed
        # the simulated engine is the reference's (scheduler.py:432-464): its numbers
        # default to the reference's bits too; the hardware modes default to fp32acc
        precision = precision or (reference_api_precision() if mode == "sim" else default_precision())
        self.precision = precision
        flags = (N.TR_FLAG_STEAL if steal else 0) | (N.TR_FLAG_COHERENCE if coherence else 0)
        flags |= N.TR_FLAG_DEBUG if directory_debug else 0
        flags |= N.TR_FLAG_DRYRUN if mode == "dryrun" else 0
        flags |= N.TR_FLAG_SIM if mode == "sim" else 0
        self.compute = compute
        flags |= N.TR_FLAG_FIFO if policy == "fifo" else 0
        flags |= 0 if fetch_ahead else N.TR_FLAG_NO_PREFETCH
        flags |= N.TR_FLAG_TRACE if trace else 0
        self.tracing = trace
        mc, keep = machine._as_c()
        h = C.c_void_p()
        N.call("tr_session_create", C.byref(mc), int(tile_size), precision_code(precision), flags,
               int(hbm_budget_bytes), C.byref(h))
        self._h = h
        self._uids = UidTable()
        dh = C.c_void_p()
        N.call("tr_session_directory", h, C.byref(dh))
        self.directory = CacheDirectory(machine, enabled=coherence, policy=policy, debug=directory_debug,
                                        _native_handle=dh, _uids=self._uids, _owner=self)
        self._uid_n = 0
        self._lock = threading.Lock()  # one product at a time per session

    def close(self) -> None:
        h = getattr(self, "_h", None)
        if h is not None and h.value:
            N.lib.tr_session_destroy(h)
        self._h = None

    def __del__(self):
        self.close()

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    def set_inflight(self, max_inflight: int) -> None:
        """Tasks each device executes concurrently (default 2; 1 serialises)."""
        N.call("tr_session_set_inflight", self._h, int(max_inflight))

    def set_order(self, order: str) -> None:
        """Task order: "row-major" (reference), "banded", "shells", "blocked", "k-panels"
        (cold single-device products: the first half of the k-panels streamed
        k-major), or "auto" (k-panels for cold in-core single-device
        products, else shells / blocked / row-major)."""
        code = {"auto": -1, "row-major": 0, "banded": 1, "shells": 2, "blocked": 3, "k-panels": 4}[order]
        N.call("tr_session_set_order", self._h, code)

    def set_stream(self, stream=None, ordered: bool = False) -> None:
        """Order products after the work queued on ``stream`` (a ``torch.cuda.Stream``
        or raw cudaStream_t handle; None clears).  ``ordered=True`` makes products
        whose operands are all CUDA tensors stream-ordered: the call returns once
        the tasks are enqueued and ``stream`` waits for them (tr_session_set_async);
        per-launch kernel times and the device span are then not measured."""
        h = None if stream is None else int(getattr(stream, "cuda_stream", stream))  # 0: legacy default stream
        N.call("tr_session_set_external_stream", self._h, h or None, int(h is not None))
        N.call("tr_session_set_async", self._h, int(bool(ordered) and h is not None))

    def lock_stats(self, reset: bool = True) -> dict:
        """The directory lock's cost since the last reset: seconds held, seconds
        callers waited for it, acquisitions, longest hold (tr_session_lock_stats)."""
        out = (N.i64 * 4)()
        N.call("tr_session_lock_stats", self._h, int(reset), out)
        return {"held_s": out[0] / 1e9, "waited_s": out[1] / 1e9, "acquisitions": int(out[2]),
                "max_hold_us": out[3] / 1e3}

    def forget(self, uid) -> int:
        """Drop every cached tile of matrix ``uid`` (its content is dead); returns the count."""
        n = N.i64()
        N.call("tr_session_forget", self._h, self._uids.id(uid), C.byref(n))
        return n.value

    def fresh_uid(self, prefix: str = "m") -> str:
        self._uid_n += 1
        return f"{prefix}#{self._uid_n}"

    def sim_now(self) -> float:
        """Simulated time of the session (mode="sim"; scheduler.py:552-553), else 0.0."""
        out = N.f64()
        N.call("tr_session_sim_now", self._h, C.byref(out))
        return out.value

    def operand(self, m, uid: str | None = None, transposed: bool = False) -> Operand:
        tiled = m if isinstance(m, TiledMatrix) else partition(m, self.tile_size)
        return Operand(tiled, uid or self.fresh_uid(), transposed)

    def multiply(self, a, b, transpose_a: bool = False, transpose_b: bool = False, a_uid: str | None = None,
                 b_uid: str | None = None, c_uid: str | None = None, *, out=None, task_offset: int = 0,
                 task_stride: int = 1):
        """Full scheduled product; returns ``(result, RunStats)`` (scheduler.py:559-612).

        Host operands (numpy) are read tile by tile from (pinned) host memory;
        CUDA-tensor operands are read from HBM.  The result lives where A lives.
        ``task_offset``/``task_stride`` run only the tasks t with
        t % stride == offset (static multi-process sharding).
        """
        if (isinstance(a, Operand) and transpose_a) or (isinstance(b, Operand) and transpose_b):
            raise ValueError("transposition of an Operand is fixed at construction")
        a_op = a if isinstance(a, Operand) else self.operand(self._prep(a), a_uid, transpose_a)
        b_op = b if isinstance(b, Operand) else self.operand(self._prep(b), b_uid, transpose_b)
        if a_op.tiled.tile_size != b_op.tiled.tile_size or a_op.tiled.tile_size != self.tile_size:
            raise ValueError(f"tile sizes differ: {a_op.tiled.tile_size} vs {b_op.tiled.tile_size}")
        am, ak = a_op.element_shape
        bk, bn = b_op.element_shape
        if ak != bk:
            raise ValueError(f"inner dimensions differ: {a_op.element_shape} x {b_op.element_shape}")
        c_uid = c_uid or self.fresh_uid("c")
        dry = self.mode in ("dryrun", "sim")
        if out is None:
            out = None if dry else _zeros_like_output(a_op, am, bn, pinned=True, zero=False)
        ma = self._desc(a_op.tiled.base, dry)
        mb = self._desc(b_op.tiled.base, dry)
        mc = self._desc(out, dry, shape=(am, bn), dtype=a_op.tiled.base.dtype)
        total = -(-am // self.tile_size) * -(-bn // self.tile_size)
        ids = (self._uids.id(a_op.uid), self._uids.id(b_op.uid), self._uids.id(c_uid))

        def call(rep):
            N.call("tr_gemm_shard", self._h, C.byref(ma), ids[0], int(a_op.transposed), C.byref(mb), ids[1],
                   int(b_op.transposed), C.byref(mc), ids[2], int(task_offset), int(task_stride), C.byref(rep))

        stats = self._execute(call, total, lambda t: t % task_stride == task_offset)
        if self.mode == "sim" and self.compute:
            if isinstance(a_op.tiled.base, ShapeOnly) or isinstance(b_op.tiled.base, ShapeOnly):
                raise ValueError("ShapeOnly operands carry no data: use Runtime(..., compute=False)")
            out = self._sim_product(a_op, b_op, out)
        return out, stats

    def _sim_product(self, a_op: Operand, b_op: Operand, out):
        """The numbers of a simulated run: the reference's sim engine computes the
        product alongside its simulated clock; here the same sm_100a tile kernel
        computes it in one dense launch (dense_gemm) -- there is no CPU path."""
        if N.cuda_device_count() < 1:
            raise NoDeviceError("mode='sim' computes the product on the GPU; Runtime(..., compute=False) "
                                "simulates schedule, counters and time only")
        import torch

        from .dense import dense_gemm

        on_device = is_device_tensor(a_op.tiled.base)
        to_dev = lambda x: x if is_device_tensor(x) else torch.from_numpy(np.ascontiguousarray(x)).cuda()
        a, b = to_dev(a_op.tiled.base), to_dev(b_op.tiled.base)
        if b.dtype != a.dtype:
            b = b.to(a.dtype)
        c = dense_gemm(a, b, transpose_a=a_op.transposed, transpose_b=b_op.transposed, precision=self.precision)
        if out is not None:
            if is_device_tensor(out):
                out.copy_(c)
            else:
                out[...] = c.cpu().numpy()
            return out
        return c if on_device else c.cpu().numpy()

    def multiply_batch(self, products) -> RunStats:
        """Independent products scheduled as ONE round (tr_gemm_batch): their tasks
        interleave on the devices, so a small product overlaps a large one and the
        per-call overhead is paid once.  Each product is a dict with keys ``a``,
        ``b``, ``out`` (CUDA tensors), optional ``transpose_a``/``transpose_b``,
        ``a_uid``/``b_uid``/``c_uid``, and an optional fused epilogue
        ``post=("bias_act", bias, activation)`` or ``post=("act_grad", a_prev,
        activation)`` (float32 device outputs).  ``cache_as=uid`` marks an output that a
        later product reads as an input under ``uid``: the producing kernel writes
        its converted tiles straight into the tile cache (tr_product.cache_as).
        ``axpy=alpha`` accumulates instead: out += alpha * a.b (tr_product.axpy; the
        fused SGD update W += (-lr) X^T dY).  ``colsum=buf`` (a float32 CUDA tensor of
        ceil(rows/32) x cols) receives the 32-row block column sums of the final
        output, summed by ``tr_mlp_colsum_finish`` (the bias gradient without a pass
        over the output).  Returns the combined RunStats."""
        if self.mode == "sim":
            raise ValueError("multiply_batch runs on the GPU; the simulated engine takes one product per call")
        acts = {"identity": N.TR_ACT_IDENTITY, "sigmoid": N.TR_ACT_SIGMOID, "relu": N.TR_ACT_RELU}
        arr = (N.ProductC * len(products))()
        keep = []
        total = 0
        for k, pr in enumerate(products):
            a, b, out = pr["a"], pr["b"], pr["out"]
            ta, tb = bool(pr.get("transpose_a", False)), bool(pr.get("transpose_b", False))
            q = arr[k]
            q.a, q.b, q.c = describe(a), describe(b), describe(out)
            q.transpose_a, q.transpose_b = int(ta), int(tb)
            q.a_uid = self._uids.id(pr.get("a_uid") or self.fresh_uid())
            q.b_uid = self._uids.id(pr.get("b_uid") or self.fresh_uid())
            q.c_uid = self._uids.id(pr.get("c_uid") or self.fresh_uid("c"))
            if pr.get("cache_as"):  # the output is read later as an input under this uid
                q.cache_as = self._uids.id(pr["cache_as"])
            if pr.get("axpy") is not None:  # out += alpha * a.b (float32 device out, no post-op)
                q.axpy, q.alpha = 1, float(pr["axpy"])
            if pr.get("colsum") is not None:  # 32-row block column sums of the final output (tr_product.colsum)
                q.colsum = pr["colsum"].data_ptr()
                keep.append(pr["colsum"])
            post = pr.get("post")
            if post is not None:
                kind, ref, act = post
                q.act = acts[act]
                if kind == "bias_act":
                    q.post = N.TR_POST_BIAS_ACT
                    q.bias = None if ref is None else ref.data_ptr()
                elif kind == "act_grad":
                    q.post = N.TR_POST_ACT_GRAD
                    q.aux, q.ldaux = ref.data_ptr(), ref.stride(0)
                else:
                    raise ValueError(f"unknown post-op {kind!r}")
                keep.append(ref)
            m = a.shape[1] if ta else a.shape[0]
            nn = b.shape[0] if tb else b.shape[1]
            total += -(-m // self.tile_size) * -(-nn // self.tile_size)

        def call(rep):
            N.call("tr_gemm_batch", self._h, len(products), arr, C.byref(rep))

        return self._execute(call, total, lambda t: True)

    def _execute(self, call, total: int, planned) -> RunStats:
        n = self.machine.n_devices
        rep = N.GemmReportC()
        per_cache = (N.CacheStatsC * n)()
        per_dev = (N.DeviceStatsC * n)()
        steals = (N.StealEventC * max(1, total))()
        completion = (N.u8 * max(1, total))()
        rep.cache_per_device, rep.devices = per_cache, per_dev
        rep.steals, rep.steals_cap = steals, total
        rep.completion, rep.completion_cap = completion, total
        with self._lock:
            call(rep)
            kms = (N.f64 * n)()
            N.call("tr_session_kernel_ms", self._h, kms)
            span = (N.f64 * n)()
            N.call("tr_session_span_ms", self._h, span)
            trace = self._read_trace() if self.tracing else []
        done = Completion.of(np.frombuffer(completion, dtype=np.uint8, count=total).copy())
        want = np.array([planned(t) for t in range(total)], dtype=bool)
        if not np.array_equal(done._bits.astype(bool), want):
            raise RuntimeError(f"run incomplete: {done.done_count}/{int(want.sum())} tasks")
        return RunStats(
            mode=self.mode, tile_size=self.tile_size, grid_rows=int(rep.grid_rows), grid_cols=int(rep.grid_cols),
            k_steps=int(rep.k_steps), total_tasks=int(rep.total_tasks), steal_enabled=self.steal,
            coherence_enabled=self.coherence, seed=self.seed,
            devices={d: DeviceStats(d, self.machine.devices[d].kind, int(per_dev[d].tasks_completed),
                                    int(per_dev[d].steals_performed), int(per_dev[d].steals_suffered),
                                    int(per_dev[d].peer_copies_served), int(per_dev[d].macs))
                     for d in range(n)},
            cache=CacheStats.from_c(rep.cache),
            cache_per_device={d: CacheStats.from_c(per_cache[d]) for d in range(n)},
            makespan=float(rep.makespan) if self.mode == "sim" else None, wall_elapsed=float(rep.wall_seconds),
            steal_events=[StealEvent(int(steals[i].thief), int(steals[i].victim), int(steals[i].task_id), True,
                                     float(steals[i].time) if self.mode == "sim" else None)
                          for i in range(min(int(rep.n_steals), total))],
            precision=self.precision, gpu_launches=int(rep.gpu_launches),
            kernel_ms={d: float(kms[d]) for d in range(n)},
            span_ms={d: float(span[d]) for d in range(n)},
            trace=trace, completion=done,
        )

    def _read_trace(self) -> list[dict]:
        n = N.i64()
        N.call("tr_session_trace", self._h, None, 0, C.byref(n))
        buf = (N.TraceEventC * max(1, n.value))()
        N.call("tr_session_trace", self._h, buf, n.value, C.byref(n))
        out = []
        for k in range(n.value):
            e = buf[k]
            out.append({"device": e.device, "kind": N.TRACE_KINDS[e.kind], "stream": e.stream, "task": e.task,
                        "tile": (self._uids.uid(e.matrix) if e.matrix else None, e.row, e.col),
                        "start_ms": e.start_ms, "end_ms": e.end_ms})
        return out

    @staticmethod
    def _prep(x):
        return x if is_device_tensor(x) or isinstance(x, ShapeOnly) else _host_matrix(x)

    @staticmethod
    def _desc(x, dry, shape=None, dtype=None) -> N.MatrixC:
        if isinstance(x, ShapeOnly):
            if not dry:
                raise ValueError("ShapeOnly operands carry no data: only mode='sim'/'dryrun' runs take them")
            shape, dtype, x = x.shape, x.dtype, None
        if x is None:  # dry run: shape-only descriptor
            from .matrix import dtype_code

            r, c = shape
            return N.MatrixC(None, r, c, c, dtype_code(dtype), N.TR_LOC_HOST)
        return describe(x)


def run(machine: Machine, a, b, tile_size: int, mode: str = "gpu", steal: bool = True, coherence: bool = True,
        seed: int | None = None, directory_debug: bool = False, precision: str | None = None, compute: bool = True):
    """One-shot product through a fresh session with uids "A","B","C" (scheduler.py:615-621)."""
    rt = Runtime(machine, tile_size, mode=mode, steal=steal, coherence=coherence, seed=seed,
                 directory_debug=directory_debug, precision=precision, compute=compute)
    try:
        return rt.multiply(a, b, a_uid="A", b_uid="B", c_uid="C")
    finally:
        rt.close()


def standalone_rates(machine: Machine, tile_size: int, a, b, *, out=None, precision: str | None = None,
                     reps: int = 2) -> list[float]:
    """Throughput (flop/s) of every logical device of ``machine`` running the
    product ``a @ b`` ALONE: a one-device machine with the device's GPU, green-
    context SM count and slots, warm (the operands' tiles already cached), best
    device-side span of ``reps`` products.  Devices with the same (gpu, sms,
    slots) are measured once.  This is the yardstick work shares are judged
    against on inhomogeneous machines -- the reference's acceptance test compares
    each device's share with its throughput share (test_acceptance.py:130-141)."""
    from .devices import DeviceSpec, ProximityMatrix

    flops = 2.0 * np.shape(a)[0] * np.shape(a)[1] * np.shape(b)[1]
    cache: dict = {}
    rates = []
    for spec in machine.devices:
        key = (spec.gpu, spec.sms, spec.slots)
        if key not in cache:
            one = Machine([DeviceSpec(0, gpu=spec.gpu, sms=spec.sms, slots=spec.slots)], ProximityMatrix.uniform(1),
                          dtype=machine.dtype)
            with Runtime(one, tile_size, precision=precision) as rt:
                rt.multiply(a, b, a_uid="A", b_uid="B", out=out)
                best = min(rt.multiply(a, b, a_uid="A", b_uid="B", out=out)[1].span_ms[0] for _ in range(reps))
            cache[key] = flops / (best / 1e3)
        rates.append(cache[key])
    return rates


def release_cached_memory() -> None:
    """Hand every HBM block cached by closed sessions back to CUDA (devpool.h):
    one-shot ``run()`` calls reuse those blocks, a workload switching to very
    different buffer sizes wants them freed first."""
    N.call("tr_release_cached_memory")
