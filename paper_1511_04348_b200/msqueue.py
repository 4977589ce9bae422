"""The global task queue: a lock-free Michael-Scott MPMC FIFO in C++.

Same contract as the reference queue (msqueue.py:9-12, 28-67): every enqueued
value is dequeued exactly once or is still queued, one producer's values come
out in order, ``None`` is the empty sentinel, and ``is_empty`` is exact once
producers have quiesced.  The reference is two-lock; this one is the
counted-pointer CAS algorithm the paper names, see
csrc/msqueue.cpp.  Python objects ride through the native queue as integer
handles.
"""

from __future__ import annotations

import ctypes as C
import itertools
import threading

from . import _native as N

_tls = threading.local()


class MichaelScottQueue:
    def __init__(self):
        h = C.c_void_p()
        N.call("tr_queue_create", C.byref(h))
        self._h = h
        self._objs: dict[int, object] = {}
        self._ids = itertools.count(1)
        self._enq = N.lib.tr_queue_enqueue
        self._deq = N.lib.tr_queue_dequeue

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value:
            N.lib.tr_queue_destroy(h)
            self._h = None

    def enqueue(self, value) -> None:
        if value is None:
            raise ValueError("None is the empty sentinel and cannot be enqueued")
        hid = next(self._ids)
        self._objs[hid] = value  # published before the handle becomes visible
        st = self._enq(self._h, hid)
        if st:
            N.check(st)

    def dequeue(self):
        """Pop the oldest value, or None when the queue is empty."""
        tl = _tls.__dict__
        bufs = tl.get("bufs")
        if bufs is None:  # per-thread out-parameters, created once
            v, got = N.u64(), N.i32()
            bufs = tl["bufs"] = (v, got, C.byref(v), C.byref(got))
        v, got, pv, pgot = bufs
        st = self._deq(self._h, pv, pgot)
        if st:
            N.check(st)
        if not got.value:
            return None
        return self._objs.pop(v.value)

    def is_empty(self) -> bool:
        e = N.i32()
        N.check(N.lib.tr_queue_is_empty(self._h, C.byref(e)))
        return bool(e.value)

    def drain(self) -> list:
        """Dequeue everything currently visible (single-threaded helper)."""
        out = []
        while (v := self.dequeue()) is not None:
            out.append(v)
        return out

    @property
    def handle(self):
        return self._h
