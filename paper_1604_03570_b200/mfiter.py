"""Tile schedules and the MFIter facade.

Host-side restatement of the reference's tiled iteration
(``/root/reference/pkg/src/tilemesh/iterator.py``): ``build_schedule``
(:69-90) flattens (unit, tile) pairs, ``partition`` (:93-103) hands out
contiguous ranges, ``TileCursor`` (:106-155) exposes
``tilebox/validbox/growntilebox/nodaltilebox``.

On the device a schedule becomes the CTA work list of the sweep kernels:
one CTA per tile, all tiles of all boxes in one launch (see
``multifab.DeviceTiles``).  ``MFIter`` is the paper's iterator
(``MFIter mfi(mf, tiling)``) built on the same schedule,
for user loops that want tile boxes on the host.
"""

from __future__ import annotations

from typing import Callable, NamedTuple

from .box import Box, check_tile_size, decompose, to_face
from .boxarray import partition

DEFAULT_TILE_SIZE = (1048576, 8, 8)  # reference iterator.py:20
OFF = "off"
DEFAULT = "default"


class TileEntry(NamedTuple):
    unit: int
    tile: Box


class TileSchedule:
    """Ordered (unit, tile) list: units ascending, tiles x-fastest within a unit."""

    def __init__(self, entries: list, unit_boxes: list, nghost: int, units: list | None = None):
        self.entries = entries
        self.unit_boxes = unit_boxes
        self.nghost = nghost
        # global unit ids covered (all units unless built for one rank)
        self.units = units if units is not None else list(range(len(unit_boxes)))
        self._device = {}

    def __len__(self) -> int:
        return len(self.entries)

    def max_tile_extents(self) -> tuple:
        ex = [1, 1, 1]
        for e in self.entries:
            t = e.tile.extents
            for d in range(3):
                if t[d] > ex[d]:
                    ex[d] = t[d]
        return tuple(ex)

    def worker_range(self, worker_count: int, worker_id: int) -> tuple:
        return partition(len(self.entries), worker_count, worker_id)

    def worker_runs(self, worker_count: int, worker_id: int) -> list:
        """Runs of same-unit entries in one worker's range as
        ``(unit, [tile boxes])`` (reference iterator.py:50-66 returns the
        tiles as an int64 (n, 6) array; see ``tiles_array``)."""
        lo, hi = partition(len(self.entries), worker_count, worker_id)
        runs = []
        pos = lo
        while pos < hi:
            u = self.entries[pos].unit
            end = pos
            while end < hi and self.entries[end].unit == u:
                end += 1
            runs.append((u, [e.tile for e in self.entries[pos:end]]))
            pos = end
        return runs


def tiles_array(boxes) -> "np.ndarray":
    import numpy as np

    arr = np.empty((len(boxes), 6), dtype=np.int64)
    for n, b in enumerate(boxes):
        arr[n, 0:3] = b.lo
        arr[n, 3:6] = b.hi
    return arr


def _resolve_tile_size(mode, default_tile_size):
    if isinstance(mode, str):
        if mode == OFF:
            return None
        if mode == DEFAULT:
            return check_tile_size(default_tile_size)
        raise ValueError(f"unknown tiling mode {mode!r}")
    if mode is True:
        return check_tile_size(default_tile_size)
    if mode is False or mode is None:
        return None
    return check_tile_size(mode)


def build_schedule(mf, mode=OFF, default_tile_size=DEFAULT_TILE_SIZE, units=None) -> TileSchedule:
    """(unit, tile) schedule of ``mf`` under a tiling mode.

    ``mode`` is ``"off"`` (one tile per unit), ``"default"`` (use
    ``default_tile_size``) or an explicit tile-size triple.  ``units``
    restricts the schedule to a subset of global unit ids (the units one
    rank owns); default: the units ``mf`` stores locally.
    """
    ts = _resolve_tile_size(mode, default_tile_size)
    all_valid = [u.valid for u in mf.units]
    if units is None:
        units = getattr(mf, "local_units", None)
        if units is None:
            units = list(range(len(all_valid)))
    entries = []
    for u in units:
        v = all_valid[u]
        if ts is None:
            entries.append(TileEntry(u, v))
        else:
            entries.extend(TileEntry(u, t) for t in decompose(v, ts))
    return TileSchedule(entries, all_valid, mf.nghost, list(units))


class TileCursor:
    """One schedule position (reference iterator.py:106-155)."""

    __slots__ = ("schedule", "pos", "worker_id", "worker_count")

    def __init__(self, schedule: TileSchedule, pos: int, worker_id: int = 0, worker_count: int = 1):
        self.schedule = schedule
        self.pos = pos
        self.worker_id = worker_id
        self.worker_count = worker_count

    def _entry(self) -> TileEntry:
        if not 0 <= self.pos < len(self.schedule):
            raise IndexError("cursor exhausted")
        return self.schedule.entries[self.pos]

    def index(self) -> int:
        """Global unit id of the current tile (``MFIter::index``)."""
        return self._entry().unit

    def tilebox(self) -> Box:
        return self._entry().tile

    def validbox(self) -> Box:
        return self.schedule.unit_boxes[self._entry().unit]

    def growntilebox(self, ng: int) -> Box:
        """Tile grown by ``ng`` only on faces shared with its unit's valid
        box, so grown tiles of one unit tile ``grow(valid, ng)`` exactly."""
        if ng > self.schedule.nghost:
            raise ValueError(f"ng={ng} exceeds nghost={self.schedule.nghost}")
        t = self.tilebox()
        v = self.validbox()
        lo = [t.lo[d] - (ng if t.lo[d] == v.lo[d] else 0) for d in range(3)]
        hi = [t.hi[d] + (ng if t.hi[d] == v.hi[d] else 0) for d in range(3)]
        return Box(lo, hi)

    def nodaltilebox(self, direction: int) -> Box:
        """Face box of the tile in ``direction``; the high face is kept only
        on the unit's high boundary so per-unit face boxes are disjoint."""
        t = self.tilebox()
        fb = to_face(t, direction)
        if t.hi[direction] != self.validbox().hi[direction]:
            hi = list(fb.hi)
            hi[direction] -= 1
            fb = Box(fb.lo, hi, fb.itype)
        return fb


def parallel_for_tiles(schedule: TileSchedule, worker_count: int, body: Callable) -> None:
    """Run ``body(cursor)`` for every schedule entry, statically partitioned
    over ``worker_count`` host workers (reference iterator.py:158-190).

    Host-side convenience for user code; device sweeps never go through it.
    The first exception raised by ``body`` is re-raised after all workers
    stop.
    """
    import threading

    if worker_count < 1:
        raise ValueError("worker_count must be >= 1")
    n = len(schedule)
    errors: list = []

    def work(w):
        a, b = partition(n, worker_count, w)
        try:
            for p in range(a, b):
                body(TileCursor(schedule, p, w, worker_count))
        except BaseException as exc:  # noqa: BLE001 - re-raised below
            errors.append(exc)

    if worker_count == 1:
        work(0)
    else:
        ths = [threading.Thread(target=work, args=(w,)) for w in range(worker_count)]
        for th in ths:
            th.start()
        for th in ths:
            th.join()
    if errors:
        raise errors[0]


class MFIter:
    """``for mfi in MFIter(mf, tiling=True): mfi.tilebox() ...``

    ``tiling`` is ``True`` (default tile size ``(1048576, 8, 8)``),
    ``False`` (one tile per box) or an explicit tile-size triple.  Iterates
    the tiles of the boxes this rank owns; each step yields a ``TileCursor``
    whose ``index()`` addresses the FAB (``mf.fab(mfi.index())``).
    """

    def __init__(self, mf, tiling=False, tile_size=None):
        if tile_size is not None:
            mode = tile_size
        else:
            mode = DEFAULT if tiling is True else (OFF if tiling is False else tiling)
        self.mf = mf
        self.schedule = build_schedule(mf, mode)

    def __len__(self) -> int:
        return len(self.schedule)

    def __iter__(self):
        for p in range(len(self.schedule)):
            yield TileCursor(self.schedule, p)
