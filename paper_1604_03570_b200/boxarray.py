"""BoxArray, Geometry and DistributionMapping (host metadata).

Reference counterparts: ``BoxArray`` (level.py:41-71), ``Geometry``
(level.py:74-93).  ``DistributionMapping`` has no reference class
("single process owns all grids"); it is restated from the
reference's static ``partition`` rule (iterator.py:93-103) applied to the
x-fastest box order, which yields contiguous z-slabs of boxes per rank
(SURVEY.md §8a row a14).

The reference checks disjointness pairwise (O(n^2), level.py:49-54); here a
uniform bucket index makes the check O(n) so that 32,768-box arrays
(BASELINE config 5) construct in well under a second.
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import Iterable, Sequence

from .box import CELL, Box, decompose, intersect


class BoxIndex:
    """Uniform-bucket spatial index over a list of disjoint boxes.

    The bucket edge per dimension is the largest box extent, so each box
    lands in at most 2x2x2 buckets and a query touches O(1) buckets.
    ``query`` returns the ids of boxes intersecting a region, ascending.
    """

    def __init__(self, boxes: Sequence[Box]):
        self.boxes = list(boxes)
        nonempty = [b for b in self.boxes if not b.is_empty]
        if nonempty:
            self.edge = tuple(max(b.extents[d] for b in nonempty) for d in range(3))
            self.origin = tuple(min(b.lo[d] for b in nonempty) for d in range(3))
        else:
            self.edge, self.origin = (1, 1, 1), (0, 0, 0)
        self.buckets: dict = {}
        for n, b in enumerate(self.boxes):
            if b.is_empty:
                continue
            for key in self._keys(b.lo, b.hi):
                self.buckets.setdefault(key, []).append(n)

    def _keys(self, lo, hi):
        o, e = self.origin, self.edge
        r = [range((lo[d] - o[d]) // e[d], (hi[d] - o[d]) // e[d] + 1) for d in range(3)]
        return [(a, b, c) for c in r[2] for b in r[1] for a in r[0]]

    def query(self, region: Box) -> list:
        if region.is_empty:
            return []
        found = set()
        get = self.buckets.get
        for key in self._keys(region.lo, region.hi):
            ids = get(key)
            if ids:
                found.update(ids)
        rlo, rhi = region.lo, region.hi
        out = []
        for n in sorted(found):
            b = self.boxes[n]
            if (b.lo[0] <= rhi[0] and rlo[0] <= b.hi[0] and b.lo[1] <= rhi[1]
                    and rlo[1] <= b.hi[1] and b.lo[2] <= rhi[2] and rlo[2] <= b.hi[2]):
                out.append(n)
        return out


class BoxArray:
    """Ordered list of pairwise-disjoint, non-empty, cell-centred grids."""

    def __init__(self, boxes: Iterable[Box], _trusted: bool = False):
        boxes = list(boxes)
        for b in boxes:
            if b.is_empty or b.itype != CELL:
                raise ValueError(f"grids must be non-empty and cell-centered: {b}")
        if not _trusted:
            self._check_disjoint(boxes)
        self.boxes = boxes

    @staticmethod
    def _check_disjoint(boxes: list) -> None:
        index = BoxIndex(boxes)
        for key, ids in index.buckets.items():
            if len(ids) < 2:
                continue
            for a in range(len(ids)):
                for b in range(a + 1, len(ids)):
                    i, j = ids[a], ids[b]
                    if not intersect(boxes[i], boxes[j]).is_empty:
                        i, j = min(i, j), max(i, j)
                        raise ValueError(f"grids {i} and {j} overlap: {boxes[i]} vs {boxes[j]}")

    @staticmethod
    def chop(domain: Box, max_grid_size) -> "BoxArray":
        """Chop ``domain`` into grids of at most ``max_grid_size`` cells per
        dimension, x-fastest order (reference level.py:57-62)."""
        if isinstance(max_grid_size, int):
            max_grid_size = (max_grid_size,) * 3
        # decompose() tiles are disjoint by construction.
        return BoxArray(decompose(domain, max_grid_size), _trusted=True)

    def __len__(self) -> int:
        return len(self.boxes)

    def __getitem__(self, i: int) -> Box:
        return self.boxes[i]

    def __iter__(self):
        return iter(self.boxes)

    def __eq__(self, other) -> bool:
        return isinstance(other, BoxArray) and self.boxes == other.boxes

    __hash__ = None


@dataclass(frozen=True)
class Geometry:
    """Problem domain, per-dimension periodicity and mesh spacing."""

    domain: Box
    periodic: tuple = (True, True, True)
    dx: tuple = (1.0, 1.0, 1.0)

    def __post_init__(self):
        if self.domain.is_empty:
            raise ValueError("geometry domain must be non-empty")
        if any(d <= 0 for d in self.dx):
            raise ValueError(f"mesh spacings must be positive: {self.dx}")
        object.__setattr__(self, "periodic", tuple(bool(p) for p in self.periodic))
        object.__setattr__(self, "dx", tuple(float(d) for d in self.dx))

    @property
    def dxinv(self) -> tuple:
        return tuple(1.0 / d for d in self.dx)

    def lengths(self) -> tuple:
        return self.domain.extents


def partition(n_items: int, parts: int, part: int) -> tuple:
    """Static contiguous ``[start, stop)`` share of ``n_items`` for ``part``;
    the first ``n_items % parts`` parts get one extra item
    (reference iterator.py:93-103)."""
    if parts < 1 or not 0 <= part < parts:
        raise ValueError(f"bad worker {part}/{parts}")
    q, r = divmod(n_items, parts)
    start = part * q + min(part, r)
    return start, start + q + (1 if part < r else 0)


class DistributionMapping:
    """Box -> rank ownership.

    Default construction applies ``partition`` to the x-fastest box ids, so
    each rank owns a contiguous run of boxes: whole z-layers of a chopped
    domain when the box count divides evenly, else partial layers.  This
    minimises the number of remote neighbours per rank for slab-shaped
    decompositions (halo bytes ~ two faces per rank).
    """

    def __init__(self, ba_or_n, nranks: int = 1, owners: Sequence[int] | None = None):
        n = len(ba_or_n) if not isinstance(ba_or_n, int) else ba_or_n
        if nranks < 1:
            raise ValueError("nranks must be >= 1")
        if owners is not None:
            owners = [int(o) for o in owners]
            if len(owners) != n or any(not 0 <= o < nranks for o in owners):
                raise ValueError("owners must give a rank in [0, nranks) for every box")
        else:
            owners = [0] * n
            for r in range(nranks):
                a, b = partition(n, nranks, r)
                for i in range(a, b):
                    owners[i] = r
        self.nranks = nranks
        self.owners = owners

    def __len__(self) -> int:
        return len(self.owners)

    def __getitem__(self, i: int) -> int:
        return self.owners[i]

    def boxes_of(self, rank: int) -> list:
        return [i for i, o in enumerate(self.owners) if o == rank]

    def __eq__(self, other) -> bool:
        return (isinstance(other, DistributionMapping) and self.nranks == other.nranks
                and self.owners == other.owners)

    __hash__ = None
