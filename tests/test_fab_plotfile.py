"""Host FArrayBox and the plotfile-lite format (reference fab.py:19-122,
level.py:326-359) against the reference's own dumps
(tests/golden/plotfile.npz, made by tests/golden/make_golden.py)."""

import io
import json
import os
from types import SimpleNamespace

import numpy as np
import pytest

from paper_1604_03570_b200 import Box, BoxArray, FArrayBox, Geometry, copy_region, intersect_copy
from paper_1604_03570_b200.multifab import CONTIGUOUS, REGIONAL, unit_boxes
from paper_1604_03570_b200.plotfile import header_text

G = os.path.join(os.path.dirname(__file__), "golden")


def cases():
    z = np.load(os.path.join(G, "plotfile.npz"))
    return z, sorted({k.split("/")[0] for k in z.files})


def test_fab_dump_bytes_roundtrip_reference():
    z, names = cases()
    assert len(names) == 3
    for name in names:
        for f in z[name + "/files"]:
            raw = z[name + "/" + str(f)].tobytes()
            fab = FArrayBox.read(io.BytesIO(raw))
            out = io.BytesIO()
            fab.write(out)
            assert out.getvalue() == raw, (name, f)
            lo, hi = fab.abox.lo, fab.abox.hi
            assert fab.data.shape == (*fab.abox.extents, fab.ncomp)
            assert fab.at(*lo, c=0) == fab.flat[0] and fab.at(*hi, c=fab.ncomp - 1) == fab.flat[-1]


def test_header_text_matches_reference():
    z, names = cases()
    for name in names:
        m = json.loads(str(z[name + "/meta"]))
        dom = Box((0, 0, 0), tuple(m["hi"]))
        n = m["hi"][0] + 1
        geom = Geometry(dom, (True, True, True), (1.0 / n,) * 3)
        ba = BoxArray.chop(dom, m["mgs"]) if m["mgs"] else BoxArray([dom])
        layout = REGIONAL if m["region"] else CONTIGUOUS
        valids, grid_of = unit_boxes(ba, layout, m["region"])
        fake = SimpleNamespace(ncomp=m["nc"], nghost=m["ng"], layout_kind=layout,
                               units=[SimpleNamespace(grid=g, valid=v) for g, v in zip(grid_of, valids)])
        assert header_text(fake, geom) == str(z[name + "/HEADER"]), name


def test_farraybox_api():
    fab = FArrayBox(Box((1, 2, 3), (4, 4, 4)), 2)
    assert fab.flat.size == 4 * 3 * 2 * 2 and not fab.flat.any()
    fab.set_at(2, 3, 4, 7.5, c=1)
    assert fab.flat[fab.offset(2, 3, 4, 1)] == 7.5 and fab.at(2, 3, 4, 1) == 7.5
    with pytest.raises(IndexError):
        fab.at(0, 0, 0)
    with pytest.raises(ValueError):
        FArrayBox(Box.empty())
    other = FArrayBox(Box((3, 3, 3), (6, 6, 6)), 2)
    other.fill(2.0)
    intersect_copy(fab, other)
    assert fab.at(3, 3, 3) == 2.0 and fab.at(2, 3, 3) == 0.0
    with pytest.raises(ValueError):
        copy_region(fab, Box((1, 2, 3), (2, 2, 3)), other, Box((3, 3, 3), (3, 3, 3)))


