"""Per-worker host scratch arenas (reference iterator.py:193-266), kept for API
compatibility.

The reference's threaded CPU kernels take flux scratch from a grow-only arena
per worker.  On the device the flux scratch lives in registers and shared
memory, so ``heat_step`` never draws from an arena (``high_water_bytes`` stays
0); the classes remain usable as host scratch for caller code, with the same
one-owner-thread rule.
"""

from __future__ import annotations

import threading

import numpy as np


class Arena:
    """Grow-only float64 scratch: acquisitions stay valid until ``reset``."""

    def __init__(self):
        self._buf = np.empty(0)
        self._top = 0          # doubles handed out since the last reset
        self._peak = 0         # most doubles ever live at once
        self._owner = None     # thread id of the first user

    def _own(self) -> None:
        me = threading.get_ident()
        if self._owner is None:
            self._owner = me
        elif self._owner != me:
            raise RuntimeError("arena accessed from a thread other than its owner")

    def acquire_doubles(self, n: int) -> np.ndarray:
        self._own()
        end = self._top + n
        if end > self._buf.size:  # grow geometrically, keeping live contents
            grown = np.empty(max(end, 2 * self._buf.size))
            grown[: self._top] = self._buf[: self._top]
            self._buf = grown
        view = self._buf[self._top:end]
        self._top = end
        self._peak = max(self._peak, end)
        return view

    def acquire(self, nbytes: int) -> np.ndarray:
        return self.acquire_doubles(-(-nbytes // 8))

    def acquire_f64(self, shape) -> np.ndarray:
        return self.acquire_doubles(int(np.prod(shape, dtype=np.int64))).reshape(shape, order="F")

    def reset(self) -> None:
        self._own()
        self._top = 0

    def release_owner(self) -> None:
        self._owner = None

    @property
    def high_water_bytes(self) -> int:
        return 8 * self._peak


class ArenaPool:
    """One arena per worker."""

    def __init__(self, worker_count: int):
        self.arenas = [Arena() for _ in range(worker_count)]

    def acquire(self, worker_id: int, nbytes: int) -> np.ndarray:
        return self.arenas[worker_id].acquire(nbytes)

    def reset(self, worker_id: int) -> None:
        self.arenas[worker_id].reset()

    def high_water_bytes(self) -> int:
        return max((a.high_water_bytes for a in self.arenas), default=0)

    def release_owners(self) -> None:
        for a in self.arenas:
            a.release_owner()
