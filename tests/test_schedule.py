"""Tile schedule / MFIter facade (reference iterator.py:20-190 semantics) and
the tile -> CTA block mapping of the sweep kernels."""

import numpy as np
import pytest

from paper_1604_03570_b200 import Box, BoxArray, TileCursor, build_schedule, partition
from paper_1604_03570_b200.box import grow, to_face
from paper_1604_03570_b200.mfiter import parallel_for_tiles
from paper_1604_03570_b200.multifab import MAX_BLOCK_NX, MAX_BLOCK_SEGS, merge_z, split_tile


class FakeMF:
    """Metadata-only stand-in (schedules need units + nghost, no storage)."""

    class U:
        def __init__(self, v):
            self.valid = v

    def __init__(self, grids, nghost=0):
        self.units = [self.U(g) for g in grids]
        self.nghost = nghost
        self.ba = BoxArray(grids)


def worked():
    return FakeMF([Box((0, 0, 0), (7, 3, 3)), Box((0, 4, 0), (3, 7, 3)), Box((0, 8, 0), (3, 11, 3)),
                   Box((0, 12, 0), (7, 15, 3))])


def test_worked_example_assignment():
    s = build_schedule(worked(), (2, 4, 4))
    assert len(s) == 12
    got = []
    for w in range(4):
        a, b = partition(len(s), 4, w)
        got.append([s.entries[p].unit for p in range(a, b)])
    assert got == [[0, 0, 0], [0, 1, 1], [2, 2, 3], [3, 3, 3]]
    runs = s.worker_runs(4, 1)
    assert [(u, len(t)) for u, t in runs] == [(0, 1), (1, 2)]


def test_modes():
    mf = FakeMF([Box((0, 0, 0), (63, 63, 63))])
    assert len(build_schedule(mf, "default")) == 64
    assert len(build_schedule(mf, True)) == 64
    assert len(build_schedule(mf, "off")) == 1
    with pytest.raises(ValueError):
        build_schedule(mf, (0, 4, 4))


def test_partition_properties():
    rng = np.random.default_rng(0)
    for _ in range(100):
        n, t = int(rng.integers(0, 50)), int(rng.integers(1, 9))
        r = [partition(n, t, w) for w in range(t)]
        assert [i for a, b in r for i in range(a, b)] == list(range(n))
        sizes = [b - a for a, b in r]
        assert max(sizes) - min(sizes) <= 1 and sizes == sorted(sizes, reverse=True)
    with pytest.raises(ValueError):
        partition(4, 2, 2)


def test_growntilebox_spec_and_cover():
    mf = FakeMF([Box((0, 0, 0), (63, 63, 63))], nghost=2)
    s = build_schedule(mf, (64, 4, 4))
    pos = next(p for p, e in enumerate(s.entries) if e.tile.lo == (0, 0, 4))
    assert TileCursor(s, pos).growntilebox(2) == Box((-2, -2, 4), (65, 3, 7))
    with pytest.raises(ValueError):
        TileCursor(s, pos).growntilebox(3)
    rng = np.random.default_rng(5)
    for _ in range(40):
        hi = tuple(int(v) for v in rng.integers(0, 12, 3))
        g = Box((0, 0, 0), hi)
        ng = int(rng.integers(0, 3))
        s = build_schedule(FakeMF([g], ng), tuple(int(v) for v in rng.integers(1, 7, 3)))
        tgt = grow(g, ng) if ng else g
        marks = np.zeros(tgt.extents, dtype=int)
        for p in range(len(s)):
            b = TileCursor(s, p).growntilebox(ng)
            marks[tuple(slice(b.lo[d] - tgt.lo[d], b.hi[d] - tgt.lo[d] + 1) for d in range(3))] += 1
        assert np.all(marks == 1)


def test_nodaltilebox_cover():
    g = Box((0, 0, 0), (9, 6, 5))
    s = build_schedule(FakeMF([g]), (4, 3, 2))
    for d in range(3):
        f = to_face(g, d)
        marks = np.zeros(f.extents, dtype=int)
        for p in range(len(s)):
            b = TileCursor(s, p).nodaltilebox(d)
            marks[tuple(slice(b.lo[k] - f.lo[k], b.hi[k] - f.lo[k] + 1) for k in range(3))] += 1
        assert np.all(marks == 1)
    with pytest.raises(IndexError):
        TileCursor(s, len(s)).tilebox()


def test_parallel_for_tiles_visits_all_and_reraises():
    s = build_schedule(worked(), (2, 4, 4))
    seen = []
    parallel_for_tiles(s, 3, lambda c: seen.append(c.pos))
    assert sorted(seen) == list(range(12))

    def boom(c):
        if c.pos == 7:
            raise RuntimeError("x")

    with pytest.raises(RuntimeError):
        parallel_for_tiles(s, 4, boom)


def test_split_tile_limits_and_cover():
    for t in [Box((0, 0, 0), (511, 511, 3)), Box((3, 2, 1), (130, 40, 9)), Box((0, 0, 0), (63, 7, 7))]:
        parts = split_tile(t)
        assert sum(p.ncells for p in parts) == t.ncells
        for p in parts:
            e = p.extents
            assert e[0] <= MAX_BLOCK_NX and e[1] * -(-e[0] // 32) <= MAX_BLOCK_SEGS
            assert p.lo[2] == t.lo[2] and p.hi[2] == t.hi[2]
    assert split_tile(Box((0, 0, 0), (63, 7, 7))) == [Box((0, 0, 0), (63, 7, 7))]


def test_merge_z_fuses_columns():
    rows = np.array([[0, 16, 1, 1 + 8 * k, 64, 8, 8, k & 1] for k in range(8)] +
                    [[0, 16, 9, 1 + 8 * k, 64, 8, 8, (k + 1) & 1] for k in range(8)], dtype=np.int64)
    m = merge_z(rows)
    assert len(m) == 2 and all(r[6] == 64 and r[3] == 1 for r in m)
