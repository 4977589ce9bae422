"""Numpy / pure-Python restatement of the reference hot path (TEST INFRASTRUCTURE ONLY).

Each function cites the reference file:line (under /root/reference/pkg/src/tilerun/)
whose behaviour it restates.  Arithmetic is kept in the reference's exact
operation order (k ascending, one rank-1 update per contraction index), so on
float64 inputs it is bit-identical to the reference.
"""

from __future__ import annotations

import ctypes
import math
import os
from collections import Counter, OrderedDict, defaultdict
from dataclasses import dataclass, field
from pathlib import Path

import numpy as np

# ----------------------------------------------------------------- tiles.py


def grid_shape(rows: int, cols: int, tile: int) -> tuple[int, int]:
    """tiles.py:63-64: ceil(rows/T) x ceil(cols/T)."""
    if tile < 1:
        raise ValueError(f"tile_size must be >= 1, got {tile}")
    return math.ceil(rows / tile), math.ceil(cols / tile)


def tile_extent(n: int, tile: int, idx: int) -> int:
    """Size of tile `idx` along a dimension of length n (ragged last tile, tiles.py:66-69)."""
    return min(tile, n - idx * tile)


def census(rows: int, cols: int, tile: int) -> tuple[int, int]:
    """(full, ragged) tile counts, tiles.py:84-90."""
    gr, gc = grid_shape(rows, cols, tile)
    full = (rows // tile) * (cols // tile)
    return full, gr * gc - full


def encode_task(row: int, col: int, grid_cols: int) -> int:
    """tiles.py:125-131."""
    if grid_cols < 1:
        raise ValueError(f"grid_cols must be >= 1, got {grid_cols}")
    if row < 0 or col < 0 or col >= grid_cols:
        raise ValueError(f"tile coord ({row},{col}) invalid for grid_cols={grid_cols}")
    return row * grid_cols + col


def decode_task(task_id: int, grid_cols: int, grid_rows: int | None = None) -> tuple[int, int]:
    """tiles.py:134-145."""
    if grid_cols < 1:
        raise ValueError(f"grid_cols must be >= 1, got {grid_cols}")
    if task_id < 0:
        raise ValueError(f"task id must be >= 0, got {task_id}")
    if grid_rows is not None and task_id >= grid_rows * grid_cols:
        raise ValueError(f"task id {task_id} out of range for a {grid_rows}x{grid_cols} grid")
    return divmod(task_id, grid_cols)


def accumulate_product(a, b, out):
    """tiles.py:154-172: out += a @ b as k-ascending rank-1 updates (literal form)."""
    m, k = a.shape
    kb, n = b.shape
    if k != kb:
        raise ValueError(f"inner dimensions differ: {a.shape} x {b.shape}")
    if out.shape != (m, n):
        raise ValueError(f"accumulator shape {out.shape}, expected {(m, n)}")
    for kk in range(k):
        out += np.multiply.outer(a[:, kk], b[kk, :])
    return out


def reference_gemm(a, b):
    """tiles.py:197-212: dense product, zeros then one rank-1 update per k ascending."""
    a = np.asarray(a)
    b = np.asarray(b)
    if a.shape[1] != b.shape[0]:
        raise ValueError(f"inner dimensions differ: {a.shape} x {b.shape}")
    out = np.zeros((a.shape[0], b.shape[1]), dtype=np.result_type(a, b))
    for k in range(a.shape[1]):
        out += a[:, k : k + 1] * b[k : k + 1, :]
    return out


def gemm_slice(a, b, rows, cols, dtype=np.float64):
    """Sampled-slice oracle: reference_gemm(A[rows,:], B[:,cols]) in `dtype`.

    Each output element depends only on its row of A and column of B with the
    same k order, so this equals the same block of a full reference run
    (SURVEY.md §0 finding 3).  Uses the C restatement when built (bit-identical,
    checked by tests/test_oracle_golden.py), else the numpy form.
    """
    sa = np.ascontiguousarray(np.asarray(a)[np.asarray(rows), :], dtype=dtype)
    sb = np.ascontiguousarray(np.asarray(b)[:, np.asarray(cols)], dtype=dtype)
    lib = c_oracle()
    if lib is not None:
        return lib.gemm(sa, sb)
    return reference_gemm(sa, sb)


def band_samples(n: int, tile: int, per_band: int = 8, seed: int = 0) -> np.ndarray:
    """Sample indices for a sampled-slice check: at least
    ``per_band`` distinct indices in EVERY tile band [b*T, min((b+1)*T, n)) --
    both band edges plus seeded interior picks -- so every tile row/column of
    the task grid, the ragged last band included, is checked.  Sorted, unique."""
    rng = np.random.default_rng(seed)
    out = []
    for lo in range(0, n, tile):
        hi = min(lo + tile, n)
        width = hi - lo
        if width <= per_band:
            out.extend(range(lo, hi))
            continue
        pick = {lo, hi - 1}
        while len(pick) < per_band:
            pick.add(lo + int(rng.integers(0, width)))
        out.extend(sorted(pick))
    return np.unique(np.asarray(out, dtype=np.int64))


def sampled_rel_error(a_rows, b_cols, got) -> float:
    """Relative Frobenius error of a sampled block ``got`` = C[rows][:, cols]
    against the k-ascending float64 product of A[rows, :] and B[:, cols]
    (the C restatement; bit-identical to reference_gemm on float64)."""
    ref = gemm_slice(np.asarray(a_rows, np.float64), np.asarray(b_cols, np.float64),
                     np.arange(np.shape(a_rows)[0]), np.arange(np.shape(b_cols)[1]))
    den = np.linalg.norm(ref)
    return float(np.linalg.norm(np.asarray(got, np.float64) - ref) / (den if den else 1.0))


# ----------------------------------------------------------------- scheduler.py: plan


@dataclass
class PlannedTask:
    task_id: int
    row: int
    col: int
    k_steps: int


def plan_tasks(m: int, k: int, n: int, tile: int) -> list[PlannedTask]:
    """scheduler.py:165-197: one task per C tile, row-major ids, k_steps = A.grid_cols."""
    gr, _ = grid_shape(m, n, tile)
    _, gc = grid_shape(m, n, tile)
    _, k_steps = grid_shape(m, k, tile)
    out = []
    for tid in range(gr * gc):
        i, j = decode_task(tid, gc, gr)
        out.append(PlannedTask(tid, i, j, k_steps))
    return out


def operand_key(uid: str, i: int, j: int, transposed: bool) -> tuple[str, int, int]:
    """scheduler.py:132-134: cache key in STORED coordinates."""
    return (uid, j, i) if transposed else (uid, i, j)


# ----------------------------------------------------------------- msqueue.py


class FifoModel:
    """Sequential model of MichaelScottQueue's contract (msqueue.py:9-12, 36-67)."""

    def __init__(self):
        self.items: list = []

    def enqueue(self, v):
        if v is None:
            raise ValueError("None is the empty sentinel and cannot be enqueued")
        self.items.append(v)

    def dequeue(self):
        return self.items.pop(0) if self.items else None

    def is_empty(self):
        return not self.items


# ----------------------------------------------------------------- stations


class StationModel:
    """scheduler.py:200-236."""

    def __init__(self, owner: int, width: int):
        self.owner, self.width, self.slots = owner, width, []

    def refill(self, queue) -> list:
        pulled = []
        while len(self.slots) < self.width:
            v = queue.dequeue()
            if v is None:
                break
            self.slots.append(v)
            pulled.append(v)
        return pulled

    def pop_for_run(self):
        return self.slots.pop(0) if self.slots else None

    def try_steal(self):
        return self.slots.pop() if self.slots else None

    def reserved_count(self):
        return len(self.slots)


def steal_task_model(thief: int, stations: dict) -> tuple:
    """scheduler.py:239-249: most reserved victim, ties to the lowest id."""
    counts = [(s.reserved_count(), d) for d, s in stations.items() if d != thief]
    for count, victim in sorted(counts, key=lambda cv: (-cv[0], cv[1])):
        if count == 0:
            break
        tid = stations[victim].try_steal()
        if tid is not None:
            return tid, victim
    return None, None


# ----------------------------------------------------------------- coherence.py


class CapacityErrorModel(RuntimeError):
    pass


STAT_FIELDS = ("l1_hits", "l2_hits", "host_fetches", "bytes_host", "bytes_peer", "evictions", "writebacks",
               "bytes_writeback")


class DirectoryModel:
    """coherence.py:86-313 restated: residency map, per-device LRU/FIFO, pins, stats.

    ``capacity`` is a list (None = unbounded); ``hops`` an n x n list;
    ``host_worker`` a list of bools.
    """

    def __init__(self, capacity, hops, host_worker=None, enabled=True, policy="lru"):
        n = len(capacity)
        self.n, self.capacity, self.hops = n, list(capacity), hops
        self.host_worker = list(host_worker or [False] * n)
        self.enabled, self.policy = enabled, policy
        self.residency = defaultdict(set)
        self.order = {d: OrderedDict() for d in range(n)}
        self.pins = {d: Counter() for d in range(n)}
        self.stats = dict.fromkeys(STAT_FIELDS, 0)
        self.dev_stats = {d: dict.fromkeys(STAT_FIELDS, 0) for d in range(n)}

    def _bump(self, d, name, v=1):
        self.stats[name] += v
        self.dev_stats[d][name] += v

    def closest_owner(self, req, owners):  # devices.py:285-291
        return min(owners, key=lambda o: (self.hops[req][o], o))

    def lookup(self, req, key):  # coherence.py:124-134
        owners = self.residency.get(key)
        if owners and req in owners:
            if self.policy == "lru":
                self.order[req].move_to_end(key)
            return ("l1", None)
        if owners:
            return ("l2", self.closest_owner(req, owners))
        return ("miss", None)

    def admit(self, dev, key):  # coherence.py:147-174
        order = self.order[dev]
        if key in order:
            raise ValueError(f"{key} already resident on device {dev}")
        cap = self.capacity[dev]
        evicted = []
        if cap is not None and len(order) >= cap:
            need = len(order) + 1 - cap
            victims = [k for k in order if self.pins[dev][k] == 0][:need]
            if len(victims) < need:
                raise CapacityErrorModel(f"device {dev}: capacity exhausted")
            for v in victims:
                del order[v]
                self.residency[v].discard(dev)
                if not self.residency[v]:
                    del self.residency[v]
                evicted.append(v)
            self._bump(dev, "evictions", len(victims))
        order[key] = None
        self.residency[key].add(dev)
        return evicted

    def pin(self, dev, key):
        if key not in self.order[dev]:
            raise ValueError("cannot pin: not resident")
        self.pins[dev][key] += 1

    def unpin(self, dev, key):
        if self.pins[dev][key] < 1:
            raise ValueError("unpin below zero")
        self.pins[dev][key] -= 1
        if self.pins[dev][key] == 0:
            del self.pins[dev][key]

    def acquire_input(self, req, key, nbytes):  # coherence.py:210-246
        if self.host_worker[req]:
            self._bump(req, "host_fetches")
            return ("miss", "host", 0, [])
        if not self.enabled:
            self._bump(req, "host_fetches")
            self._bump(req, "bytes_host", nbytes)
            return ("miss", "host", nbytes, [])
        level, owner = self.lookup(req, key)
        if level == "l1":
            self._bump(req, "l1_hits")
            self.pins[req][key] += 1
            return ("l1", req, 0, [])
        if level == "l2":
            self._bump(req, "l2_hits")
            self._bump(req, "bytes_peer", nbytes)
            ev = self.admit(req, key)
            self.pins[req][key] += 1
            return ("l2", owner, nbytes, ev)
        self._bump(req, "host_fetches")
        self._bump(req, "bytes_host", nbytes)
        ev = self.admit(req, key)
        self.pins[req][key] += 1
        return ("miss", "host", nbytes, ev)

    def release_input(self, dev, key):  # 248-252
        if not self.enabled or self.host_worker[dev]:
            return
        self.unpin(dev, key)

    def admit_output(self, dev, key):  # 254-261
        if not self.enabled or self.host_worker[dev]:
            return []
        ev = self.admit(dev, key)
        self.pins[dev][key] += 1
        return ev

    def release_output(self, dev, key, nbytes):  # 263-280
        if not self.enabled or self.host_worker[dev]:
            return
        self.unpin(dev, key)
        del self.order[dev][key]
        self.residency[key].discard(dev)
        if not self.residency[key]:
            del self.residency[key]
        self._bump(dev, "writebacks")
        self._bump(dev, "bytes_writeback", nbytes)

    def residents(self, dev):
        return list(self.order[dev])


def run_schedule_single_device(m, k, n, tile, capacity=None, element_bytes=8, enabled=True, ta=False, tb=False,
                               policy="lru"):
    """Sequential _execute_task loop on ONE device (scheduler.py:371-410) over the
    directory model: the exact counters a one-device run must produce."""
    d = DirectoryModel([capacity], [[0]], enabled=enabled, policy=policy)
    gr, gc = grid_shape(m, n, tile)
    ks = math.ceil(k / tile)
    for t in plan_tasks(m, k, n, tile):
        i, j = t.row, t.col
        ckey = ("C", i, j)
        d.admit_output(0, ckey)
        for kk in range(ks):
            ak = operand_key("A", i, kk, ta)
            bk = operand_key("B", kk, j, tb)
            a_bytes = tile_extent(m, tile, i) * tile_extent(k, tile, kk) * element_bytes
            b_bytes = tile_extent(k, tile, kk) * tile_extent(n, tile, j) * element_bytes
            d.acquire_input(0, ak, a_bytes)
            d.acquire_input(0, bk, b_bytes)
            d.release_input(0, ak)
            d.release_input(0, bk)
        d.release_output(0, ckey, tile_extent(m, tile, i) * tile_extent(n, tile, j) * element_bytes)
    return d.stats


# ----------------------------------------------------------------- ann.py


def activate(name, y):  # ann.py:30-37
    if name == "identity":
        return y
    if name == "sigmoid":
        return 1.0 / (1.0 + np.exp(-y))
    if name == "relu":
        return np.maximum(y, 0.0)
    raise ValueError(f"unknown activation {name!r}")


def activation_grad(name, y, a):  # ann.py:40-48
    if name == "identity":
        return np.ones_like(y)
    if name == "sigmoid":
        return a * (1.0 - a)
    if name == "relu":
        return (y > 0.0).astype(y.dtype)
    raise ValueError(f"unknown activation {name!r}")


def mse(pred, target):  # ann.py:51-52
    return float(((pred - target) ** 2).mean())


def mse_grad(pred, target):  # ann.py:55-56
    return 2.0 * (pred - target) / pred.size


@dataclass
class OracleLayer:
    weights: np.ndarray
    bias: np.ndarray | None
    activation: str = "sigmoid"


def random_layer(fan_in, fan_out, rng, activation="sigmoid", scale=1.0, bias=True):
    """ann.py:142-148 (same rng draw order: weights then bias)."""
    w = rng.uniform(-scale, scale, size=(fan_in, fan_out))
    b = rng.uniform(-scale, scale, size=fan_out) if bias else None
    return OracleLayer(np.asarray(w, dtype=np.float64), None if b is None else np.asarray(b, np.float64),
                       activation)


def network_from_sizes(sizes, rng, activation="sigmoid", scale=1.0, bias=True):
    """ann.py:181-193."""
    return [random_layer(sizes[i], sizes[i + 1], rng, activation, scale, bias) for i in range(len(sizes) - 1)]


def dense_matmul(a, b, transpose_a=False, transpose_b=False):
    """DenseBackend.multiply (ann.py:65-69)."""
    a = a.T if transpose_a else a
    b = b.T if transpose_b else b
    return reference_gemm(a, b)


def blas_matmul(a, b, transpose_a=False, transpose_b=False):
    """Same algebra in float64 BLAS: the large-size MLP oracle."""
    a = a.T if transpose_a else a
    b = b.T if transpose_b else b
    return np.asarray(a, np.float64) @ np.asarray(b, np.float64)


def loss_gradients(layers, x, target, matmul=dense_matmul):
    """ann.py:151-236: forward, MSE, backward (dW = X^T dY, dX = dY W^T, db = colsum dY)."""
    xs, ys, acts = [], [], []
    cur = x
    for L in layers:
        xs.append(cur)
        y = matmul(cur, L.weights)
        if L.bias is not None:
            y = y + L.bias
        a = activate(L.activation, y)
        ys.append(y)
        acts.append(a)
        cur = a
    pred = acts[-1] if acts else x
    grads = [None] * len(layers)
    d_out = mse_grad(pred, target)
    for li in reversed(range(len(layers))):
        L = layers[li]
        d_y = d_out * activation_grad(L.activation, ys[li], acts[li])
        d_w = matmul(xs[li], d_y, transpose_a=True)
        d_x = matmul(d_y, L.weights, transpose_b=True)
        d_b = d_y.sum(axis=0) if L.bias is not None else None
        grads[li] = (d_w, d_b)
        d_out = d_x
    return mse(pred, target), grads


def train_step(layers, x, target, lr, matmul=dense_matmul):
    """ann.py:239-248: SGD after one forward/backward."""
    loss, grads = loss_gradients(layers, x, target, matmul)
    for L, (d_w, d_b) in zip(layers, grads):
        L.weights = L.weights - lr * d_w
        if L.bias is not None and d_b is not None:
            L.bias = L.bias - lr * d_b
    return loss


def random_regression(rng, batch, n_in, n_out):  # ann.py:319-322
    x = rng.uniform(-1.0, 1.0, size=(batch, n_in))
    target = rng.uniform(-1.0, 1.0, size=(batch, n_out))
    return x, target


def xor_dataset():  # ann.py:313-316
    x = np.array([[0.0, 0.0], [0.0, 1.0], [1.0, 0.0], [1.0, 1.0]])
    target = np.array([[0.0], [1.0], [1.0], [0.0]])
    return x, target


# ----------------------------------------------------------------- C restatement loader

_LIB_DIR = Path(__file__).resolve().parent
_C_LIB = None


class _COracle:
    def __init__(self, path):
        self.lib = ctypes.CDLL(str(path))
        dp = ctypes.POINTER(ctypes.c_double)
        fp = ctypes.POINTER(ctypes.c_float)
        i64 = ctypes.c_int64
        self.lib.oracle_gemm_f64.argtypes = [dp, dp, dp, i64, i64, i64, ctypes.c_int]
        self.lib.oracle_gemm_f32.argtypes = [fp, fp, fp, i64, i64, i64, ctypes.c_int]
        self.lib.oracle_rank1_f32.argtypes = [fp, fp, fp, i64, i64, i64, i64]
        self.lib.oracle_rank1_f64.argtypes = [dp, dp, dp, i64, i64, i64, i64]
        for f in ("oracle_gemm_f64", "oracle_gemm_f32", "oracle_rank1_f32", "oracle_rank1_f64"):
            getattr(self.lib, f).restype = None
        self.lib.oracle_max_threads.restype = ctypes.c_int

    def gemm(self, a, b, threads=0):
        """reference_gemm in C (k ascending, no FMA contraction), any thread count."""
        a = np.ascontiguousarray(a)
        b = np.ascontiguousarray(b)
        if a.dtype != b.dtype or a.dtype not in (np.float32, np.float64):
            raise ValueError("oracle gemm: a and b must share float32/float64 dtype")
        m, k = a.shape
        n = b.shape[1]
        out = np.zeros((m, n), dtype=a.dtype)
        if a.dtype == np.float64:
            P = ctypes.POINTER(ctypes.c_double)
            fn = self.lib.oracle_gemm_f64
        else:
            P = ctypes.POINTER(ctypes.c_float)
            fn = self.lib.oracle_gemm_f32
        fn(a.ctypes.data_as(P), b.ctypes.data_as(P), out.ctypes.data_as(P), m, k, n, int(threads))
        return out

    def rank1_updates(self, a, b, out, kk_count):
        """The reference's literal per-k update (tiles.py:170-171) for `kk_count` k values."""
        m, k = a.shape
        n = b.shape[1]
        if out.dtype == np.float64:
            P = ctypes.POINTER(ctypes.c_double)
            fn = self.lib.oracle_rank1_f64
        else:
            P = ctypes.POINTER(ctypes.c_float)
            fn = self.lib.oracle_rank1_f32
        fn(a.ctypes.data_as(P), b.ctypes.data_as(P), out.ctypes.data_as(P), m, k, n, int(kk_count))
        return out

    def max_threads(self):
        return self.lib.oracle_max_threads()


def c_oracle():
    """The compiled C restatement (oracle/liboracle.so), or None when not built."""
    global _C_LIB
    if _C_LIB is None:
        path = _LIB_DIR / "liboracle.so"
        if not path.exists():
            return None
        _C_LIB = _COracle(path)
    return _C_LIB


def build_c_oracle(force=False):
    """Compile oracle/gemm_ref.c -> oracle/liboracle.so (gcc, -ffp-contract=off)."""
    import subprocess

    src = _LIB_DIR / "gemm_ref.c"
    out = _LIB_DIR / "liboracle.so"
    if not force and out.exists() and out.stat().st_mtime >= src.stat().st_mtime:
        return out
    cmd = ["gcc", "-O3", "-march=x86-64-v2", "-ffp-contract=off", "-fno-fast-math", "-fopenmp", "-fPIC",
           "-shared", "-o", str(out), str(src)]
    subprocess.run(cmd, check=True, env={**os.environ})
    return out
