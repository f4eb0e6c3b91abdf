"""Index algebra: the reference's box semantics (box.py:36-196), checked by
brute-force cell enumeration and hypothesis properties."""

import itertools

import numpy as np
import pytest
from hypothesis import given, settings
from hypothesis import strategies as st

from paper_1604_03570_b200.box import Box, box_diff, decompose, grow, intersect, shift, to_face


def cells(b):
    if b.is_empty:
        return set()
    return set(itertools.product(*[range(b.lo[d], b.hi[d] + 1) for d in range(3)]))


boxes = st.builds(
    lambda lo, ext: Box(lo, tuple(l + e - 1 for l, e in zip(lo, ext))),
    st.tuples(*[st.integers(-6, 6)] * 3),
    st.tuples(*[st.integers(1, 6)] * 3),
)


def test_empty_and_partial_inversion():
    e = Box.empty()
    assert e.is_empty and e.extents == (0, 0, 0) and e.ncells == 0
    with pytest.raises(ValueError):
        Box((0, 0, 0), (-1, 3, 3))


def test_value_semantics():
    a = Box((0, 1, 2), (3, 4, 5))
    assert a == Box([0, 1, 2], [3, 4, 5]) and hash(a) == hash(Box((0, 1, 2), (3, 4, 5)))
    assert str(a) == "(0,1,2)-(3,4,5)[ccc]"
    with pytest.raises(AttributeError):
        a.lo = (1, 1, 1)


@settings(max_examples=200, deadline=None)
@given(boxes, boxes)
def test_intersect_is_cell_intersection(a, b):
    assert cells(intersect(a, b)) == cells(a) & cells(b)


@settings(max_examples=200, deadline=None)
@given(boxes, boxes)
def test_box_diff_partitions(a, b):
    parts = box_diff(a, b)
    got = [cells(p) for p in parts]
    union = set().union(*got) if got else set()
    assert union == cells(a) - cells(b)
    assert sum(len(g) for g in got) == len(union)  # disjoint


@settings(max_examples=100, deadline=None)
@given(boxes, st.tuples(*[st.integers(1, 9)] * 3))
def test_decompose_exact_cover_x_fastest(b, ts):
    tiles = decompose(b, ts)
    marks = np.zeros(b.extents, dtype=int)
    for t in tiles:
        sl = tuple(slice(t.lo[d] - b.lo[d], t.hi[d] - b.lo[d] + 1) for d in range(3))
        marks[sl] += 1
        assert all(t.extents[d] <= ts[d] for d in range(3))
    assert np.all(marks == 1)
    keys = [(t.lo[2], t.lo[1], t.lo[0]) for t in tiles]
    assert keys == sorted(keys)


def test_decompose_larger_first_even_split():
    tiles = decompose(Box((0, 0, 0), (9, 0, 0)), (4, 1, 1))  # 10 -> 3 tiles: 4,3,3
    assert [t.extents[0] for t in tiles] == [4, 3, 3]
    assert len(decompose(Box((0, 0, 0), (127, 127, 127)), (128, 4, 4))) == 1024


def test_grow_shift_to_face():
    b = Box((0, 0, 0), (3, 3, 3))
    assert grow(b, 1) == Box((-1, -1, -1), (4, 4, 4))
    assert grow(b, (1, 0, 2)) == Box((-1, 0, -2), (4, 3, 5))
    with pytest.raises(ValueError):
        grow(Box.empty(), 1)
    with pytest.raises(ValueError):
        grow(b, -1)
    assert shift(b, (1, -2, 3)) == Box((1, -2, 3), (4, 1, 6))
    f = to_face(b, 1)
    assert f.hi == (3, 4, 3) and f.itype == (False, True, False)
    with pytest.raises(ValueError):
        to_face(f, 1)
    with pytest.raises(ValueError):
        intersect(b, f)


def test_ghost_shell_slab_order():
    v = Box((0, 0, 0), (7, 7, 7))
    slabs = box_diff(grow(v, 2), v)
    # x slabs are full faces, y slabs trimmed in x, z slabs trimmed in x and y
    assert [s.extents for s in slabs] == [(2, 12, 12), (2, 12, 12), (8, 2, 12), (8, 2, 12), (8, 8, 2), (8, 8, 2)]
