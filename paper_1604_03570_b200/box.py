"""Index-space algebra for the host-side planner.

Mirrors the public surface of the reference's ``tilemesh.box``
(``/root/reference/pkg/src/tilemesh/box.py``): ``Box`` (:36-90),
``intersect`` (:93-103), ``grow`` (:106-116), ``to_face`` (:119-125),
``shift`` (:134-139), ``decompose`` (:155-173) and ``box_diff`` (:176-196),
with the same argument meaning, ordering guarantees and ``ValueError``
behaviour.  Boxes are small immutable value objects; they only ever live on
the host, where they describe FAB slots, copy tags and sweep tiles that are
then flattened into int tables for the device.
"""

from __future__ import annotations

from typing import Iterable, Sequence

IntVect = tuple  # (i, j, k)
IndexType = tuple  # (bool, bool, bool): True = node-centred in that dim
TileSize = tuple

CELL: IndexType = (False, False, False)


def face_type(direction: int) -> IndexType:
    """Node-centred in ``direction``, cell-centred in the other two."""
    return tuple(d == direction for d in range(3))


def check_tile_size(ts) -> TileSize:
    """Normalise a tile-size triple; every extent must be >= 1."""
    try:
        t = tuple(int(v) for v in ts)
    except TypeError as exc:  # not iterable
        raise ValueError(f"tile size must be a triple, got {ts!r}") from exc
    if len(t) != 3 or min(t) < 1:
        raise ValueError(f"tile size extents must be >= 1, got {t}")
    return t


class Box:
    """Inclusive ``[lo, hi]`` index box with a per-dimension centring.

    The canonical empty box is ``lo=(0,0,0), hi=(-1,-1,-1)``; a box that is
    inverted in some but not all dimensions is rejected, as in the reference
    (box.py:46-54).
    """

    __slots__ = ("lo", "hi", "itype", "_hash")

    def __init__(self, lo: Sequence[int], hi: Sequence[int], itype: IndexType = CELL):
        lo = (int(lo[0]), int(lo[1]), int(lo[2]))
        hi = (int(hi[0]), int(hi[1]), int(hi[2]))
        inv = (hi[0] < lo[0]) + (hi[1] < lo[1]) + (hi[2] < lo[2])
        if inv and inv != 3:
            raise ValueError(f"partially inverted box {lo}-{hi}; use Box.empty() for empties")
        object.__setattr__(self, "lo", lo)
        object.__setattr__(self, "hi", hi)
        object.__setattr__(self, "itype", tuple(bool(v) for v in itype))
        object.__setattr__(self, "_hash", None)

    def __setattr__(self, name, value):
        raise AttributeError("Box is immutable")

    # value semantics -----------------------------------------------------
    def __eq__(self, other) -> bool:
        if not isinstance(other, Box):
            return NotImplemented
        return self.lo == other.lo and self.hi == other.hi and self.itype == other.itype

    def __hash__(self) -> int:
        h = self._hash
        if h is None:
            h = hash((self.lo, self.hi, self.itype))
            object.__setattr__(self, "_hash", h)
        return h

    def __repr__(self) -> str:
        return f"Box({self.lo}, {self.hi}, {self.itype})"

    def __str__(self) -> str:
        t = "".join("n" if f else "c" for f in self.itype)
        return "({},{},{})-({},{},{})[{}]".format(*self.lo, *self.hi, t)

    def __reduce__(self):
        return (Box, (self.lo, self.hi, self.itype))

    # queries ---------------------------------------------------------------
    @staticmethod
    def empty(itype: IndexType = CELL) -> "Box":
        return Box((0, 0, 0), (-1, -1, -1), itype)

    @property
    def is_empty(self) -> bool:
        return self.hi[0] < self.lo[0]

    @property
    def extents(self) -> IntVect:
        if self.is_empty:
            return (0, 0, 0)
        lo, hi = self.lo, self.hi
        return (hi[0] - lo[0] + 1, hi[1] - lo[1] + 1, hi[2] - lo[2] + 1)

    @property
    def ncells(self) -> int:
        e = self.extents
        return e[0] * e[1] * e[2]

    def contains_point(self, p: Sequence[int]) -> bool:
        lo, hi = self.lo, self.hi
        return (lo[0] <= p[0] <= hi[0]) and (lo[1] <= p[1] <= hi[1]) and (lo[2] <= p[2] <= hi[2])

    def contains(self, other: "Box") -> bool:
        if other.is_empty:
            return True
        return self.contains_point(other.lo) and self.contains_point(other.hi)


def intersect(a: Box, b: Box) -> Box:
    """Largest box inside both ``a`` and ``b``; empty when they are disjoint."""
    if a.itype != b.itype:
        raise ValueError(f"cannot intersect boxes of types {a.itype} and {b.itype}")
    if a.is_empty or b.is_empty:
        return Box.empty(a.itype)
    alo, ahi, blo, bhi = a.lo, a.hi, b.lo, b.hi
    lo = (max(alo[0], blo[0]), max(alo[1], blo[1]), max(alo[2], blo[2]))
    hi = (min(ahi[0], bhi[0]), min(ahi[1], bhi[1]), min(ahi[2], bhi[2]))
    if hi[0] < lo[0] or hi[1] < lo[1] or hi[2] < lo[2]:
        return Box.empty(a.itype)
    return Box(lo, hi, a.itype)


def grow(b: Box, ng) -> Box:
    """``b`` widened by ``ng`` cells on every face (scalar or per-dim triple)."""
    if b.is_empty:
        raise ValueError("cannot grow an empty box")
    g = (ng, ng, ng) if isinstance(ng, int) else tuple(int(v) for v in ng)
    if min(g) < 0:
        raise ValueError(f"negative grow width {g}")
    return Box(
        (b.lo[0] - g[0], b.lo[1] - g[1], b.lo[2] - g[2]),
        (b.hi[0] + g[0], b.hi[1] + g[1], b.hi[2] + g[2]),
        b.itype,
    )


def to_face(b: Box, direction: int) -> Box:
    """Convert direction ``direction`` of ``b`` from cell to node centring."""
    if b.itype[direction]:
        raise ValueError(f"box {b} is already node-centered in direction {direction}")
    hi = list(b.hi)
    hi[direction] += 1
    t = list(b.itype)
    t[direction] = True
    return Box(b.lo, hi, tuple(t))


def shift(b: Box, v: Sequence[int]) -> Box:
    """Translate ``b`` by the integer vector ``v`` (empties stay as they are)."""
    if b.is_empty:
        return b
    return Box(
        (b.lo[0] + v[0], b.lo[1] + v[1], b.lo[2] + v[2]),
        (b.hi[0] + v[0], b.hi[1] + v[1], b.hi[2] + v[2]),
        b.itype,
    )


def split_extent(lo: int, length: int, ts: int) -> list:
    """1-D tiling rule of the reference (box.py:142-152): ``ceil(length/ts)``
    pieces of near-equal size, the longer pieces first.  Returns (lo, hi)
    inclusive pairs."""
    n = -(-length // ts)
    q, r = divmod(length, n)
    out = []
    start = lo
    for p in range(n):
        size = q + (p < r)
        out.append((start, start + size - 1))
        start += size
    return out


def decompose(b: Box, ts) -> list:
    """Tiles of a cell-centred box in x-fastest, then y, then z order."""
    ts = check_tile_size(ts)
    if b.is_empty:
        raise ValueError("cannot decompose an empty box")
    if b.itype != CELL:
        raise ValueError("decompose requires a cell-centered box")
    ex = b.extents
    px, py, pz = (split_extent(b.lo[d], ex[d], ts[d]) for d in range(3))
    return [Box((x0, y0, z0), (x1, y1, z1)) for (z0, z1) in pz for (y0, y1) in py for (x0, x1) in px]


def box_diff(a: Box, b: Box) -> list:
    """Disjoint boxes covering ``a`` minus ``b``.

    Slabs are peeled dimension by dimension (x low, x high, y low, ...), each
    peel shrinking the remainder, so the output order and shapes match the
    reference (box.py:176-196): for a ghost shell that is two full x-slabs,
    two y-slabs trimmed in x, then two z-slabs trimmed in x and y.
    """
    core = intersect(a, b)
    if core.is_empty:
        return [] if a.is_empty else [a]
    lo = list(a.lo)
    hi = list(a.hi)
    pieces = []
    for d in range(3):
        if lo[d] < core.lo[d]:
            top = list(hi)
            top[d] = core.lo[d] - 1
            pieces.append(Box(lo, top, a.itype))
            lo[d] = core.lo[d]
        if hi[d] > core.hi[d]:
            bot = list(lo)
            bot[d] = core.hi[d] + 1
            pieces.append(Box(bot, hi, a.itype))
            hi[d] = core.hi[d]
    return pieces


def bounding_box(boxes: Iterable[Box]) -> Box:
    lo = [None] * 3
    hi = [None] * 3
    for b in boxes:
        if b.is_empty:
            continue
        for d in range(3):
            lo[d] = b.lo[d] if lo[d] is None else min(lo[d], b.lo[d])
            hi[d] = b.hi[d] if hi[d] is None else max(hi[d], b.hi[d])
    if lo[0] is None:
        return Box.empty()
    return Box(lo, hi)
