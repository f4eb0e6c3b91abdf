"""FillBoundary copy plan (host side).

Produces exactly the tag list of the reference's ``build_fill_plan``
(level.py:262-287): for every destination unit, for every ghost slab of
``box_diff(grow(valid, ng), valid)``, for every periodic shift (zero first,
``_shift_candidates`` level.py:240-259), for every source unit in ascending
order whose shifted valid box meets the slab, one
``CopyTag(dst_unit, isect, src_unit, isect - s, s)``.

The reference scans every source unit for every (slab, shift) pair, which
is O(units^2 * shifts) (~30 days at 32,768 boxes).  Here
the source scan is a ``BoxIndex`` lookup and shifts that cannot reach the
domain are skipped per dimension, so the build is O(units) while emitting
the same tags in the same order.

``FillPlan.exec_tags`` restates ``_split_tags`` (level.py:213-229) for API
parity; the device path does not need it (the copy kernel balances work by
chunking tags itself) and it is computed lazily.
"""

from __future__ import annotations

from math import ceil
from typing import NamedTuple

from .box import Box, box_diff, grow, intersect, shift
from .boxarray import BoxIndex

SPLIT_CELLS = 4096  # reference level.py:38 (_SPLIT_CELLS)


class CopyTag(NamedTuple):
    dst_unit: int
    dst_box: Box
    src_unit: int
    src_box: Box
    shift: tuple


def _neg(v):
    return (-v[0], -v[1], -v[2])


def split_tags(tags: list) -> list:
    """Halve tags above ``SPLIT_CELLS`` cells along the longer of y/z, in the
    reference's LIFO order (level.py:213-229)."""
    out = []
    stack = list(tags)
    while stack:
        t = stack.pop()
        b = t.dst_box
        ex = b.extents
        d = 1 if ex[1] >= ex[2] else 2
        if b.ncells <= SPLIT_CELLS or ex[d] < 2:
            out.append(t)
            continue
        mid = b.lo[d] + ex[d] // 2 - 1
        lo_hi = list(b.hi)
        lo_hi[d] = mid
        hi_lo = list(b.lo)
        hi_lo[d] = mid + 1
        for part in (Box(b.lo, lo_hi), Box(hi_lo, b.hi)):
            stack.append(CopyTag(t.dst_unit, part, t.src_unit, shift(part, _neg(t.shift)), t.shift))
    return out


class FillPlan:
    """Ghost-cell copy tags of one MultiFab layout (``FillPlan`` level.py:207-210)."""

    def __init__(self, tags: list):
        self.tags = list(tags)
        self._exec = None
        self._device = {}  # per-(storage layout) device tables, see multifab.py

    @property
    def exec_tags(self) -> list:
        if self._exec is None:
            self._exec = split_tags(self.tags)
        return self._exec

    def __len__(self) -> int:
        return len(self.tags)


def periodic_shift_values(geom, nghost: int) -> list:
    """Per-dimension shift values ``[0, L, -L, 2L, -2L, ...]`` with
    ``K = ceil(nghost / L)`` images, or ``[0]`` when not periodic."""
    per_dim = []
    for d in range(3):
        if geom.periodic[d]:
            L = geom.lengths()[d]
            vals = [0]
            for k in range(1, ceil(nghost / L) + 1):
                vals += [k * L, -k * L]
            per_dim.append(vals)
        else:
            per_dim.append([0])
    return per_dim


def shift_candidates(geom, nghost: int) -> list:
    """All periodic image shifts, z-major product order with the zero shift
    moved to the front (reference level.py:240-259)."""
    per_dim = periodic_shift_values(geom, nghost)
    out = [(sx, sy, sz) for sz in per_dim[2] for sy in per_dim[1] for sx in per_dim[0]]
    out.sort(key=lambda s: s != (0, 0, 0))
    return out


def build_fill_plan_units(valids: list, geom, nghost: int, grids=None) -> FillPlan:
    """Plan over an explicit list of unit valid boxes (ghost width ``nghost``)."""
    if grids is not None:
        for b in grids:
            if not geom.domain.contains(b):
                raise ValueError(f"grid {b} outside domain {geom.domain}")
    if nghost == 0:
        return FillPlan([])
    shifts = shift_candidates(geom, nghost)
    order = {s: n for n, s in enumerate(shifts)}
    per_dim = periodic_shift_values(geom, nghost)
    dom = geom.domain
    index = BoxIndex(valids)
    tags = []
    for du, dv in enumerate(valids):
        for gbox in box_diff(grow(dv, nghost), dv):
            # shift values per dim that bring part of the slab back over the domain
            feas = []
            for d in range(3):
                feas.append([s for s in per_dim[d]
                             if gbox.lo[d] - s <= dom.hi[d] and gbox.hi[d] - s >= dom.lo[d]])
            cand = [(sx, sy, sz) for sz in feas[2] for sy in feas[1] for sx in feas[0]]
            cand.sort(key=order.__getitem__)
            for s in cand:
                for su in index.query(shift(gbox, _neg(s))):
                    isect = intersect(gbox, shift(valids[su], s))
                    if isect.is_empty:
                        continue
                    tags.append(CopyTag(du, isect, su, shift(isect, _neg(s)), s))
    return FillPlan(tags)


def build_fill_plan(mf, geom) -> FillPlan:
    """Ghost-cell copy tags for every unit of ``mf`` (all ranks' units; each
    rank later selects the tags it sends, receives or copies locally)."""
    return build_fill_plan_units([u.valid for u in mf.units], geom, mf.nghost, grids=list(mf.ba))
