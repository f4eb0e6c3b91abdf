"""write_plotfile from device memory is byte-identical to the reference's
dumps of the same MultiFab (tests/golden/plotfile.npz); read_plotfile
returns the device data (reference test_level.py:262-273)."""

import json
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

G = os.path.join(os.path.dirname(__file__), "golden")


@pytest.fixture(scope="module")
def tm():
    import torch

    import paper_1604_03570_b200 as tm

    torch.cuda.set_device(0)
    return tm


def f_linear(i, j, k):
    return i + 10.0 * j + 100.0 * k


def test_plotfile_bytes_match_reference(tm, tmp_path):
    z = np.load(os.path.join(G, "plotfile.npz"))
    for name in sorted({k.split("/")[0] for k in z.files}):
        m = json.loads(str(z[name + "/meta"]))
        dom = tm.Box((0, 0, 0), tuple(m["hi"]))
        n = m["hi"][0] + 1
        geom = tm.Geometry(dom, (True, True, True), (1.0 / n,) * 3)
        ba = tm.BoxArray.chop(dom, m["mgs"]) if m["mgs"] else tm.BoxArray([dom])
        layout = tm.REGIONAL if m["region"] else tm.CONTIGUOUS
        mf = tm.MultiFab(ba, m["nc"], m["ng"], layout, tuple(m["region"]) if m["region"] else None)
        for c in range(m["nc"]):
            mf.set_from_function(lambda i, j, k, c=c: f_linear(i, j, k) + 1000.0 * c + 0.125, comp=c)
        if m["fill"]:
            tm.fill_boundary(mf, geom)
        path = str(tmp_path / name)
        tm.write_plotfile(mf, geom, path)
        assert open(os.path.join(path, "HEADER")).read() == str(z[name + "/HEADER"]), name
        files = sorted(f for f in os.listdir(path) if f.endswith(".fab"))
        assert files == [str(f) for f in z[name + "/files"]], name
        for f in files:
            assert open(os.path.join(path, f), "rb").read() == z[name + "/" + f].tobytes(), (name, f)
        header, fabs = tm.read_plotfile(path)
        assert f"ncomp {m['nc']}" in header and len(fabs) == len(mf.units)
        for u, fab in enumerate(fabs):
            assert fab.abox == mf.fab(u).abox
            assert np.array_equal(fab.flat, mf.fab(u).flat)
