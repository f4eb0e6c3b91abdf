"""REGIONAL layout (level.py:116-133) on the B200:
units, plans, FillBoundary, heat / wide4 runs and reduce_sum bit-identical
to the reference's own runs (tests/golden/regional.npz), and layout
transparency as the reference tests it (test_level.py:238-259,
test_kernels.py:270-284)."""

import hashlib
import json
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

G = os.path.join(os.path.dirname(__file__), "golden")
SENTINEL = -12345.6789


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a, dtype=np.float64).tobytes()).hexdigest()


@pytest.fixture(scope="module")
def tm():
    import torch

    import paper_1604_03570_b200 as tm

    torch.cuda.set_device(0)
    return tm


def f_linear(i, j, k):
    return i + 10.0 * j + 100.0 * k


def case(tm, z, name):
    m = json.loads(str(z[name + "/meta"]))
    dom = tm.Box((0, 0, 0), tuple(m["hi"]))
    ba = tm.BoxArray.chop(dom, m["mgs"]) if m["mgs"] else tm.BoxArray([dom])
    geom = tm.Geometry(dom, tuple(m["periodic"]), (1.0 / (m["hi"][0] + 1),) * 3)
    return m, ba, geom


def test_regional_matches_reference_runs(tm):
    z = np.load(os.path.join(G, "regional.npz"))
    for name in sorted({k.split("/")[0] for k in z.files}):
        m, ba, geom = case(tm, z, name)
        mf = tm.MultiFab(ba, 1, m["ng"], tm.REGIONAL, tuple(m["region"]))
        units = np.array([[u.grid, *u.valid.lo, *u.valid.hi] for u in mf.units], dtype=np.int64)
        assert np.array_equal(units, z[name + "/units"]), name
        plan = tm.build_fill_plan(mf, geom)
        rows = np.array([[t.dst_unit, *t.dst_box.lo, *t.dst_box.hi, t.src_unit, *t.src_box.lo, *t.src_box.hi,
                          *t.shift] for t in plan.tags], dtype=np.int64)
        assert np.array_equal(rows, z[name + "/tags"]), name
        if m["kernel"] == "fill":
            mf.fill(SENTINEL)
            mf.set_from_function(f_linear)
            tm.fill_boundary(mf, geom, plan)
            flat = np.concatenate([mf.fab(u).to_numpy().ravel(order="F") for u in range(len(mf.units))])
            assert np.array_equal(flat, z[name + "/fill"]), name
            continue
        n = m["hi"][0] + 1
        glob = tm.make_init(tm.CONFIGS["C1"].scaled(n, n, m["steps"]))
        mf.from_global(glob)
        new = mf.clone_empty()
        sched = tm.build_schedule(mf, (8, 8, 8))
        old, sums = mf, []
        for _ in range(m["steps"]):
            tm.fill_boundary(old, geom, plan)
            if m["kernel"] == "heat":
                tm.heat_step(new, old, geom, tm.HeatParams.stable(1.0, geom.dx), sched)
            else:
                tm.wide4_step(new, old, geom, 1.0, tm.wide4_stable_dt(1.0, geom.dx), sched)
            old, new = new, old
            sums.append(old.reduce_sum(0))
        assert sha(old.to_global().cpu().numpy()) == str(z[name + "/final_sha"]), name
        assert sums == list(z[name + "/sums"]), name


def test_regional_sum_and_fill_identical_to_contiguous(tm):
    ba = tm.BoxArray([tm.Box((0, 0, 0), (11, 11, 11))])
    vals = {}
    for layout, region in ((tm.CONTIGUOUS, None), (tm.REGIONAL, (4, 6, 5))):
        mf = tm.MultiFab(ba, 1, 1, layout, region)
        mf.set_from_function(lambda i, j, k: np.sin(i * 0.1 + j * 0.01 + k))
        vals[layout] = (mf.reduce_sum(0), mf.reduce_max(0), mf.reduce_min(0))
    assert vals[tm.CONTIGUOUS] == vals[tm.REGIONAL]
    ba2 = tm.BoxArray([tm.Box((0, 0, 0), (7, 7, 7)), tm.Box((8, 0, 0), (15, 7, 7))])
    geom = tm.Geometry(tm.Box((0, 0, 0), (15, 7, 7)), (True, False, True))
    arrays = {}
    for layout, region in ((tm.CONTIGUOUS, None), (tm.REGIONAL, (4, 4, 4))):
        mf = tm.MultiFab(ba2, 1, 2, layout, region)
        mf.set_from_function(f_linear)
        tm.fill_boundary(mf, geom)
        arrays[layout] = [mf.grid_valid_array(g) for g in range(len(ba2))]
    for a, b in zip(arrays[tm.CONTIGUOUS], arrays[tm.REGIONAL]):
        assert np.array_equal(a, b)


def test_heat_workers_and_layout_bitwise(tm):
    results = []
    for layout, region in ((tm.CONTIGUOUS, None), (tm.REGIONAL, (12, 12, 12)), (tm.REGIONAL, (5, 7, 24))):
        dom = tm.Box((0, 0, 0), (23, 23, 23))
        geom = tm.Geometry(dom, (True, True, True), (1.0 / 24,) * 3)
        mf = tm.MultiFab(tm.BoxArray([dom]), 1, 1, layout, region)
        tm.init_cosine(mf, geom)
        p = tm.HeatParams.stable(1.0, geom.dx[0])
        out = mf.clone_empty()
        for _ in range(5):
            tm.fill_boundary(mf, geom)
            tm.heat_step(out, mf, geom, p, (8, 8, 8))
            mf, out = out, mf
        results.append((mf.grid_valid_array(0), mf.reduce_sum()))
    for arr, s in results[1:]:
        assert np.array_equal(results[0][0], arr)
        assert s == results[0][1]


def test_regional_runner_and_gsrb(tm):
    """The step runner and the GSRB solve run on regional MultiFabs (unfused
    path: regions of a grid are not face-uniform in general) and agree with
    the contiguous layout bit for bit."""
    from paper_1604_03570_b200.runner import HeatRunner

    w = tm.CONFIGS["C1"].scaled(32, 16, 4)
    glob = tm.make_init(w)
    geom = tm.Geometry(w.domain, (True, True, True), (w.dx,) * 3)
    ba = tm.BoxArray.chop(w.domain, 16)
    outs = []
    for layout, region in ((tm.CONTIGUOUS, None), (tm.REGIONAL, (8, 16, 6))):
        mf = tm.MultiFab(ba, 1, 1, layout, region)
        mf.from_global(glob)
        r = HeatRunner(mf, geom, tm.HeatParams.stable(1.0, geom.dx), w.tile_size)
        out = r.advance(4)
        outs.append((out.to_global().cpu().numpy(), out.reduce_sum()))
    assert np.array_equal(outs[0][0], outs[1][0]) and outs[0][1] == outs[1][1]
    rhs_g = tm.make_init(tm.CONFIGS["C4"].scaled(32, 16, 3))
    res = []
    for layout, region in ((tm.CONTIGUOUS, None), (tm.REGIONAL, (16, 8, 8))):
        phi = tm.MultiFab(ba, 1, 1, layout, region)
        rhs = tm.MultiFab(ba, 1, 0, layout, region)
        rhs.from_global(rhs_g)
        tm.gsrb_solve(phi, rhs, geom, 3)
        res.append((phi.to_global().cpu().numpy(), tm.residual_maxnorm(phi, rhs, geom)))
    assert np.array_equal(res[0][0], res[1][0]) and res[0][1] == res[1][1]
