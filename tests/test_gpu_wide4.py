"""wide4 (9-point 8th-order Laplacian, nghost 4) on the
B200: bit-identical to the reference's own runs (tests/golden/wide4.npz,
made by tests/golden/make_golden.py from /root/reference) and to the oracle
on other layouts; plus the reference's own property tests
(test_kernels.py:330-427, test_acceptance.py:193-216)."""

import dataclasses
import hashlib
import json
import math
import os

import numpy as np
import pytest

from oracle import oracle as orc

pytestmark = pytest.mark.gpu

G = os.path.join(os.path.dirname(__file__), "golden")


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a, dtype=np.float64).tobytes()).hexdigest()


@pytest.fixture(scope="module")
def tm():
    import torch

    import paper_1604_03570_b200 as tm

    torch.cuda.set_device(0)
    return tm


def run_device(tm, w, glob, coeffs, dt, steps, max_rows=None, nctas=None):
    from paper_1604_03570_b200.wide4 import _launch

    geom = tm.Geometry(w.domain, (True, True, True), (w.dx,) * 3)
    ba = tm.BoxArray.chop(w.domain, w.max_grid_size)
    old = tm.MultiFab(ba, 1, 4)
    old.from_global(glob)
    new = old.clone_empty()
    plan = tm.build_fill_plan(old, geom)
    sums = []
    for _ in range(steps):
        tm.fill_boundary(old, geom, plan)
        if max_rows is None and nctas is None:
            tm.wide4_step(new, old, geom, 1.0, dt, None, 1, coeffs)
        else:
            _launch(new, old, geom, 1.0, dt, coeffs, max_rows, nctas)
        old, new = new, old
        sums.append(old.reduce_sum())
    return old, sums


def test_wide4_matches_reference_runs(tm):
    z = np.load(os.path.join(G, "wide4.npz"))
    coeffs = tm.StencilCoeffs8(*[float(v) for v in z["coeffs"]])
    names = sorted({k.split("/")[0] for k in z.files if "/" in k})
    for name in names:
        m = json.loads(str(z[name + "/meta"]))
        w = dataclasses.replace(tm.CONFIGS["C1"].scaled(m["n"], m["mgs"], m["steps"]), nghost=4)
        glob = tm.make_init(w)
        mf, sums = run_device(tm, w, glob, coeffs, float(z[name + "/dt"]), w.steps)
        fin = mf.to_global().cpu().numpy()
        assert sha(fin) == str(z[name + "/final_sha"]), name
        assert sums == list(z[name + "/sums"]), name


@pytest.mark.parametrize("n,mgs,steps,rows,nctas", [
    (40, 40, 2, None, None),   # 40-wide boxes: 2 cells per lane, partial lanes
    (37, 37, 2, None, 5),      # odd width, odd height
    (128, 128, 1, None, None),  # 128-wide: 4 cells per lane, 8-row columns
    (96, 48, 2, 5, 7),         # 5-row columns, segments crossing columns
    (24, 4, 2, None, None),    # 4^3 boxes: every ghost layer from a neighbour box
    (40, 16, 2, None, None),   # boxes 16 and 8 wide / high: Kernel W2 on non-uniform columns
    (24, 4, 2, None, 2),       # 216 four-plane columns on 2 CTAs: > 32 segments per CTA (W2's
                               # descriptor cache overflows to global memory)
    (64, 32, 2, None, 7),      # W2, segments crossing columns
])
def test_wide4_matches_oracle(tm, n, mgs, steps, rows, nctas):
    w = dataclasses.replace(tm.CONFIGS["C1"].scaled(n, mgs, steps), nghost=4)
    glob = tm.make_init(w)
    coeffs = tm.derive_coeffs8()
    dt = tm.wide4_stable_dt(1.0, (w.dx,) * 3)
    mf, _ = run_device(tm, w, glob, coeffs, dt, steps, rows, nctas)
    want = orc.wide4_periodic(glob[0], steps, coeffs.as_array(), (1.0 / w.dx ** 2,) * 3, dt)
    assert np.array_equal(mf.to_global().cpu().numpy()[0], want)


def test_wide4_constant_unchanged(tm):
    dom = tm.Box((0, 0, 0), (15, 15, 15))
    geom = tm.Geometry(dom, (True, True, True), (1.0 / 16,) * 3)
    mf = tm.MultiFab(tm.BoxArray([dom]), 1, 4)
    mf.fill(4.5)
    out = mf.clone_empty()
    dt = tm.wide4_stable_dt(1.0, geom.dx[0])
    for _ in range(3):
        tm.fill_boundary(mf, geom)
        tm.wide4_step(out, mf, geom, 1.0, dt, None)
        mf, out = out, mf
    assert np.all(mf.grid_valid_array(0) == 4.5)


def test_wide4_quadratic_laplacian_exact(tm):
    """u = i^2 + j^2 + k^2 (ghosts set analytically, no fill) has discrete
    Laplacian exactly 6 with dx = 1."""
    import torch

    dom = tm.Box((0, 0, 0), (11, 11, 11))
    geom = tm.Geometry(dom, (True, True, True), (1.0, 1.0, 1.0))
    mf = tm.MultiFab(tm.BoxArray([dom]), 1, 4)
    f = mf.fab(0)
    b = f.abox
    I, J, K = np.ogrid[b.lo[0]:b.hi[0] + 1, b.lo[1]:b.hi[1] + 1, b.lo[2]:b.hi[2] + 1]
    f.view(b, 0, 1)[..., 0].copy_(torch.from_numpy(np.ascontiguousarray((I ** 2 + J ** 2 + K ** 2).astype(float))))
    out = mf.clone_empty()
    dt, D = 1e-3, 2.0
    tm.wide4_step(out, mf, geom, D, dt, None)
    want = mf.grid_valid_array(0) + dt * D * 6.0
    assert np.max(np.abs(out.grid_valid_array(0) - want)) <= 1e-11


def test_wide4_symbol_amplification(tm):
    dom = tm.Box((0, 0, 0), (15, 15, 15))
    geom = tm.Geometry(dom, (True, True, True), (1.0 / 16,) * 3)
    mf = tm.MultiFab(tm.BoxArray([dom]), 1, 4)
    tm.init_cosine(mf, geom, modes=(1, 2, 3))
    u0 = mf.grid_valid_array(0).copy()
    dt = tm.wide4_stable_dt(1.0, geom.dx[0])
    out = mf.clone_empty()
    for _ in range(4):
        tm.fill_boundary(mf, geom)
        tm.wide4_step(out, mf, geom, 1.0, dt, None)
        mf, out = out, mf
    g4 = tm.wide4_amplification(1.0, dt, geom, modes=(1, 2, 3)) ** 4
    rel = np.max(np.abs(mf.grid_valid_array(0) - g4 * u0)) / np.max(np.abs(g4 * u0))
    assert rel <= 1e-12


def test_wide4_order_at_least_7_5(tm):
    def err(n):
        dom = tm.Box((0, 0, 0), (n - 1, n - 1, n - 1))
        geom = tm.Geometry(dom, (True, True, True), (1.0 / n,) * 3)
        mf = tm.MultiFab(tm.BoxArray([dom]), 1, 4)
        tm.init_cosine(mf, geom)
        out = mf.clone_empty()
        tm.fill_boundary(mf, geom)
        tm.wide4_step(out, mf, geom, 1.0, 1.0, None)
        lap_h = out.grid_valid_array(0) - mf.grid_valid_array(0)
        lap = -3.0 * (2.0 * math.pi) ** 2 * mf.grid_valid_array(0)
        return float(np.max(np.abs(lap_h - lap)))

    assert math.log2(err(16) / err(32)) >= 7.5


def test_wide4_tiling_and_workers_bitwise(tm):
    w = dataclasses.replace(tm.CONFIGS["C1"].scaled(32, 16, 2), nghost=4)
    glob = tm.make_init(w)
    geom = tm.Geometry(w.domain, (True, True, True), (w.dx,) * 3)
    dt = tm.wide4_stable_dt(1.0, geom.dx)
    outs = []
    for variant in ("tiled", "untiled"):
        mf = tm.MultiFab(tm.BoxArray.chop(w.domain, 16), 1, 4)
        mf.from_global(glob)
        out = mf.clone_empty()
        for _ in range(2):
            tm.fill_boundary(mf, geom)
            if variant == "tiled":
                tm.wide4_step(out, mf, geom, 1.0, dt, tm.build_schedule(mf, (8, 4, 4)), workers=3)
            else:
                tm.wide4_step(out, mf, geom, 1.0, dt, None, workers=2)
            mf, out = out, mf
        outs.append(mf.to_global().cpu().numpy())
    assert np.array_equal(outs[0], outs[1])


def test_wide4_needs_four_ghosts(tm):
    dom = tm.Box((0, 0, 0), (7, 7, 7))
    geom = tm.Geometry(dom, (True, True, True), (1.0 / 8,) * 3)
    mf = tm.MultiFab(tm.BoxArray([dom]), 1, 1)
    with pytest.raises(ValueError):
        tm.wide4_step(mf.clone_empty(), mf, geom, 1.0, 1e-5, None)
    mf2 = tm.MultiFab(tm.BoxArray([dom]), 2, 4)
    with pytest.raises(ValueError):
        tm.wide4_step(mf2.clone_empty(), mf2, geom, 1.0, 1e-5, None)


@pytest.mark.parametrize("n,mgs,steps,graph,nbr", [
    (64, 32, 5, True, None),     # 2^3 boxes of 32^3: Kernel W2, one 32-row column per box, odd step count
    (64, 32, 3, True, False),    # same boxes on Kernel W's scatter epilogue (16-row columns)
    (40, 40, 4, False, None),    # one 40^3 box: every face its own periodic image; W2 with 20-row columns
    (40, 40, 2, False, False),
    (48, 16, 3, True, None),     # 3^3 boxes of 16^3
    (24, 8, 6, True, None),      # 8^3 boxes: the 4-deep faces of a box cover it completely
    (24, 8, 3, True, False),
    (96, 96, 2, False, None),    # 96 wide: Kernel W (4 cells per lane, 8-row columns), scatter epilogue
])
def test_fused_wide4_runner_matches_oracle(tm, n, mgs, steps, graph, nbr):
    """One launch per step (neighbour-sourced halos, or FillBoundary fused into
    the epilogue) against the whole-domain oracle and against the
    reference-structured unfused loop."""
    w = dataclasses.replace(tm.CONFIGS["C1"].scaled(n, mgs, steps), nghost=4)
    glob = tm.make_init(w)
    geom = tm.Geometry(w.domain, (True, True, True), (w.dx,) * 3)
    ba = tm.BoxArray.chop(w.domain, w.max_grid_size)
    dt = tm.wide4_stable_dt(1.0, (w.dx,) * 3)
    coeffs = tm.derive_coeffs8()
    outs = []
    for fused in (True, False):
        mf = tm.MultiFab(ba, 1, 4)
        mf.from_global(glob)
        r = tm.Wide4Runner(mf, geom, 1.0, dt, coeffs, fused=fused, use_graph=graph,
                           nbr_halos=nbr if fused else None)
        assert r.fused == fused
        if fused:
            assert r.nbr_halos == (mgs <= 64 if nbr is None else nbr)
        res = r.advance(steps)
        outs.append(res.to_global().cpu().numpy()[0])
        if fused:  # the closing FillBoundary leaves the ghosts a fresh fill gives
            ref = tm.MultiFab(ba, 1, 4)
            ref.from_global(res.to_global())
            tm.fill_boundary(ref, geom)
            for u in res.local_units:  # whole grown boxes, ghosts included (not the row padding)
                fa, fb = res.fab(u), ref.fab(u)
                assert np.array_equal(fa.view(fa.abox, 0, 1).cpu().numpy(), fb.view(fb.abox, 0, 1).cpu().numpy())
        r.close()
    want = orc.wide4_periodic(glob[0], steps, coeffs.as_array(), (1.0 / w.dx ** 2,) * 3, dt)
    assert np.array_equal(outs[0], want)
    assert np.array_equal(outs[1], want)


def test_wide4_production_shape(tm):
    """The C2-shaped wide4 problem the bench times (256^3, 64 boxes of 64^3,
    4 ghosts): Kernel W2 with neighbour-sourced halos (fused runner, graph
    pairs), Kernel W2 on ghosts (reference loop) and the oracle, every cell."""
    w = dataclasses.replace(tm.CONFIGS["C2"].scaled(256, 64, 3), nghost=4)
    glob = tm.make_init(w)
    geom = tm.Geometry(w.domain, (True, True, True), (w.dx,) * 3)
    ba = tm.BoxArray.chop(w.domain, w.max_grid_size)
    dt = tm.wide4_stable_dt(1.0, (w.dx,) * 3)
    coeffs = tm.derive_coeffs8()
    want = orc.wide4_periodic(glob[0], 3, coeffs.as_array(), (1.0 / w.dx ** 2,) * 3, dt)
    mf = tm.MultiFab(ba, 1, 4)
    mf.from_global(glob)
    r = tm.Wide4Runner(mf, geom, 1.0, dt, coeffs)
    assert r.fused and r.nbr_halos
    assert np.array_equal(r.advance(3).to_global().cpu().numpy()[0], want)
    r.close()
    fin, _ = run_device(tm, w, glob, coeffs, dt, 3)
    assert np.array_equal(fin.to_global().cpu().numpy()[0], want)


def test_fused_wide4_eligibility(tm):
    dom = tm.Box((0, 0, 0), (23, 23, 23))
    geom = tm.Geometry(dom, (True, True, True), (1.0 / 24,) * 3)
    small = tm.MultiFab(tm.BoxArray.chop(dom, 6), 1, 4)  # 6^3 boxes: 4-deep faces would overlap
    assert not tm.Wide4Runner(small, geom, 1.0, 1e-6).fused
    with pytest.raises(ValueError):
        tm.Wide4Runner(small, geom, 1.0, 1e-6, fused=True)
    dom23 = tm.Box((0, 0, 0), (22, 22, 22))
    geom23 = tm.Geometry(dom23, (True, True, True), (1.0 / 23,) * 3)
    ragged = tm.MultiFab(tm.BoxArray.chop(dom23, 10), 1, 4)  # 8, 8, 7 cells: not uniform
    assert not tm.Wide4Runner(ragged, geom23, 1.0, 1e-6).fused


@pytest.mark.parametrize("n,mgs,steps", [(128, 64, 4), (96, 32, 5), (64, 16, 3)])
def test_wide4_reference_loop_fast_path(tm, n, mgs, steps):
    """fill_boundary (4 layers) + wide4_step on a W2-eligible layout: the fill is deferred and
    rides on the step's launch (tm_wide4_march_fill: face ghosts written as loaded, edge/corner
    cells by the producer warpgroup's idle warps).  Fields vs the oracle; the ghosts a caller
    observes between the calls equal a regular FillBoundary's."""
    w = dataclasses.replace(tm.CONFIGS["C1"].scaled(n, mgs, steps), nghost=4)
    glob = tm.make_init(w)
    geom = tm.Geometry(w.domain, (True, True, True), (w.dx,) * 3)
    ba = tm.BoxArray.chop(w.domain, w.max_grid_size)
    dt = tm.wide4_stable_dt(1.0, (w.dx,) * 3)
    coeffs = tm.derive_coeffs8()
    old = tm.MultiFab(ba, 1, 4)
    old.from_global(glob)
    new = old.clone_empty()
    plan = tm.build_fill_plan(old, geom)
    for s in range(steps):
        tm.fill_boundary(old, geom, plan)
        assert old._w4_deferred, "the wide4 fill fast path was not taken"
        if s == 1:  # observe the deferred ghosts: they must be a regular fill's
            ref = tm.MultiFab(ba, 1, 4)
            ref.from_global(old.to_global())
            ref.drop_deferred()
            copy, _ = __import__("paper_1604_03570_b200.multifab", fromlist=["_device_fill"])._device_fill(ref, plan)
            copy.run(ref.gptr, ref.layout.side(), ref.ptr, ref.layout.side(), ref.stream())
            for u in old.local_units:
                fa, fb = old.fab(u), ref.fab(u)  # .fab views settle the deferred ghosts first
                assert np.array_equal(fa.view(fa.abox, 0, 1).cpu().numpy(), fb.view(fb.abox, 0, 1).cpu().numpy())
            assert not old._w4_deferred
        settles = old.settles
        tm.wide4_step(new, old, geom, 1.0, dt, coeffs=coeffs)
        if s != 1:  # the fill rode on the step's launch: nothing was settled by a copy launch
            assert old.settles == settles and old._pending_faces is None
        if s == 2:  # the step wrote old's ghosts itself (nothing pending): they are a fill's
            assert old._pending_faces is None and not old._w4_deferred
            ref = tm.MultiFab(ba, 1, 4)
            ref.from_global(old.to_global())
            tm.fill_boundary(ref, geom, plan)
            for u in old.local_units:
                fa, fb = old.fab(u), ref.fab(u)
                assert np.array_equal(fa.view(fa.abox, 0, 1).cpu().numpy(), fb.view(fb.abox, 0, 1).cpu().numpy())
        old, new = new, old
    want = orc.wide4_periodic(glob[0], steps, coeffs.as_array(), (1.0 / w.dx ** 2,) * 3, dt)
    assert np.array_equal(old.to_global().cpu().numpy()[0], want)
    # after the last step the field the loop read last carries a whole fill, written in-kernel
    tm.fill_boundary(old, geom, plan)
    fin = old.data.cpu().numpy()  # settles
    ref = tm.MultiFab(ba, 1, 4)
    ref.from_global(old.to_global())
    tm.fill_boundary(ref, geom, plan)
    for u in old.local_units:
        fa, fb = old.fab(u), ref.fab(u)
        assert np.array_equal(fa.view(fa.abox, 0, 1).cpu().numpy(), fb.view(fb.abox, 0, 1).cpu().numpy())
    assert fin.shape == old._data.shape
