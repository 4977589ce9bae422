"""The two-level tile cache directory (L1 own HBM / L2 peer HBM / host).

Python face of the native directory (csrc/directory.cpp), API-compatible with
the reference CacheDirectory (coherence.py:86-313): same hit taxonomy, LRU or
FIFO eviction of unpinned tiles only, CapacityError leaving the directory
unchanged, exact counters, one lock making every composite operation
linearizable.  A session's directory (``Runtime.directory``) is the very
structure the GPU workers use; its resident tiles occupy HBM slab slots.
"""

from __future__ import annotations

import ctypes as C
import threading
from dataclasses import dataclass, fields
from enum import Enum

from . import _native as N
from .devices import HOST, Machine, closest_owner  # noqa: F401 (tilerun.coherence names)
from .errors import CapacityError
from .tiles import TileKey

__all__ = ["CacheDirectory", "CacheStats", "CapacityError", "HitLevel", "LookupResult", "AcquireResult",
           "UidTable"]


class HitLevel(Enum):
    L1 = "l1"
    L2 = "l2"
    MISS = "miss"


_LEVELS = {N.TR_HIT_L1: HitLevel.L1, N.TR_HIT_L2: HitLevel.L2, N.TR_HIT_MISS: HitLevel.MISS}


@dataclass(frozen=True)
class LookupResult:
    level: HitLevel
    owner: int | None = None  # L2 hits only


@dataclass(frozen=True)
class AcquireResult:
    level: HitLevel
    source: object  # device id or HOST
    nbytes_moved: int
    evicted: tuple = ()


@dataclass
class CacheStats:
    """coherence.py:59-83, field for field."""

    l1_hits: int = 0
    l2_hits: int = 0
    host_fetches: int = 0
    bytes_host: int = 0
    bytes_peer: int = 0
    evictions: int = 0
    writebacks: int = 0
    bytes_writeback: int = 0

    @classmethod
    def from_c(cls, s: N.CacheStatsC) -> "CacheStats":
        return cls(**{f.name: int(getattr(s, f.name)) for f in fields(cls)})

    def copy(self) -> "CacheStats":
        return CacheStats(**self.as_dict())

    def as_dict(self) -> dict:
        return {f.name: getattr(self, f.name) for f in fields(self)}

    def __sub__(self, other: "CacheStats") -> "CacheStats":
        return CacheStats(**{f.name: getattr(self, f.name) - getattr(other, f.name) for f in fields(self)})

    @property
    def input_requests(self) -> int:
        return self.l1_hits + self.l2_hits + self.host_fetches


class UidTable:
    """Interns matrix uids (any hashable, usually str) to the native 64-bit ids."""

    def __init__(self):
        self._to_id: dict = {}
        self._from_id: dict = {}
        self._lock = threading.Lock()

    def id(self, uid) -> int:
        with self._lock:
            i = self._to_id.get(uid)
            if i is None:
                i = len(self._to_id) + 1
                self._to_id[uid] = i
                self._from_id[i] = uid
            return i

    def uid(self, i: int):
        return self._from_id[i]


_EVICT_CAP = 4096


class CacheDirectory:
    """Directory over a ``Machine`` (coherence.py:95-114 signature)."""

    def __init__(self, machine: Machine, enabled: bool = True, policy: str = "lru", debug: bool = False,
                 *, _native_handle=None, _uids: UidTable | None = None, _owner=None):
        if policy not in ("lru", "fifo"):
            raise ValueError(f"unknown eviction policy {policy!r}")
        self.machine = machine
        self.enabled = enabled
        self.policy = policy
        self.debug = debug
        self._uids = _uids or UidTable()
        self._owner = _owner  # keeps a borrowing session alive
        self._owned = _native_handle is None
        if _native_handle is None:
            mc, keep = machine._as_c()
            h = C.c_void_p()
            N.call("tr_dir_create", C.byref(mc), int(enabled), N.TR_POLICY_FIFO if policy == "fifo" else
                   N.TR_POLICY_LRU, int(debug), C.byref(h))
            self._h = h
        else:
            self._h = _native_handle
        self._evicted = (N.TileKeyC * _EVICT_CAP)()

    def __del__(self):
        if getattr(self, "_owned", False) and getattr(self, "_h", None) is not None:
            N.lib.tr_dir_destroy(self._h)
            self._h = None

    # -- key plumbing
    def _k(self, key) -> N.TileKeyC:
        m, r, c = key
        return N.TileKeyC(self._uids.id(m), int(r), int(c))

    def _key(self, kc: N.TileKeyC) -> TileKey:
        return TileKey(self._uids.uid(kc.matrix), int(kc.row), int(kc.col))

    def _evicted_list(self, n: int) -> list[TileKey]:
        return [self._key(self._evicted[i]) for i in range(min(n, _EVICT_CAP))]

    # -- primitives (coherence.py:118-200)
    def lookup(self, requester: int, key) -> LookupResult:
        level, owner = N.i32(), N.i32()
        N.call("tr_dir_lookup", self._h, int(requester), C.byref(self._k(key)), C.byref(level), C.byref(owner))
        lv = _LEVELS[level.value]
        return LookupResult(lv, owner.value if lv is HitLevel.L2 else None)

    def admit(self, device: int, key) -> list[TileKey]:
        n = N.i32()
        N.call("tr_dir_admit", self._h, int(device), C.byref(self._k(key)), self._evicted, _EVICT_CAP, C.byref(n))
        return self._evicted_list(n.value)

    def pin(self, device: int, key) -> None:
        N.call("tr_dir_pin", self._h, int(device), C.byref(self._k(key)))

    def unpin(self, device: int, key) -> None:
        N.call("tr_dir_unpin", self._h, int(device), C.byref(self._k(key)))

    def is_pinned(self, device: int, key) -> bool:
        p = N.i32()
        N.call("tr_dir_is_pinned", self._h, int(device), C.byref(self._k(key)), C.byref(p))
        return bool(p.value)

    def residents(self, device: int) -> list[TileKey]:
        n = N.i64()
        N.call("tr_dir_residents", self._h, int(device), None, 0, C.byref(n))
        buf = (N.TileKeyC * max(1, n.value))()
        N.call("tr_dir_residents", self._h, int(device), buf, n.value, C.byref(n))
        return [self._key(buf[i]) for i in range(n.value)]

    def used_tiles(self, device: int) -> int:
        n = N.i64()
        N.call("tr_dir_used_tiles", self._h, int(device), C.byref(n))
        return n.value

    # -- composite operations (coherence.py:210-280)
    def acquire_input(self, requester: int, key, nbytes: int) -> AcquireResult:
        res = N.AcquireResultC()
        N.call("tr_dir_acquire_input", self._h, int(requester), C.byref(self._k(key)), int(nbytes), C.byref(res),
               self._evicted, _EVICT_CAP)
        src = HOST if res.source == N.TR_SOURCE_HOST else int(res.source)
        return AcquireResult(_LEVELS[res.level], src, int(res.nbytes_moved), tuple(self._evicted_list(res.n_evicted)))

    def release_input(self, device: int, key) -> None:
        N.call("tr_dir_release_input", self._h, int(device), C.byref(self._k(key)))

    def admit_output(self, device: int, key) -> list[TileKey]:
        n = N.i32()
        N.call("tr_dir_admit_output", self._h, int(device), C.byref(self._k(key)), self._evicted, _EVICT_CAP,
               C.byref(n))
        return self._evicted_list(n.value)

    def release_output(self, device: int, key, nbytes: int) -> None:
        N.call("tr_dir_release_output", self._h, int(device), C.byref(self._k(key)), int(nbytes))

    # -- observability (coherence.py:284-313)
    def stats(self) -> CacheStats:
        g = N.CacheStatsC()
        N.call("tr_dir_stats", self._h, C.byref(g), None)
        return CacheStats.from_c(g)

    def stats_per_device(self) -> dict[int, CacheStats]:
        n = self.machine.n_devices
        arr = (N.CacheStatsC * n)()
        N.call("tr_dir_stats", self._h, None, arr)
        return {i: CacheStats.from_c(arr[i]) for i in range(n)}

    def check_invariants(self) -> None:
        N.call("tr_dir_check_invariants", self._h)
