"""Every production kernel configuration, at the real shapes, against the
oracle -- the exact paths ``bench.py`` and DESIGN.md's numbers run:

* C2 at full size through ``HeatRunner`` as the bench drives it (fused
  neighbour-halo march, CUDA-graph step pairs, alternating direction,
  100 steps), every valid cell and the checksum against the C oracle
  (the reference's tag FillBoundary + four-loop heat, tm_oracle.c) and the
  checksum the reference itself printed;
* the 128-wide-box kernel instance (C3: 4 cells per lane, 32-row columns,
  one 17-warp CTA per SM, 4 components, 2 ghosts) in both march directions,
  at a reduced box count and at the full C3 shape;
* C4 at full size (colour-split and in-place fused GSRB) against the C
  oracle's red / FillBoundary / black / FillBoundary sweeps and residual;
* the C5 shape (32^3 boxes, 2 components, 2 ghosts, 4096 boxes at 512^3;
  the full 1024^3 case with TM_TEST_FULL_C5=1 -- it needs ~90 GB of device
  and ~60 GB of host memory);
* layouts the fused path must decline (66-, 70- and 98-wide boxes) through
  heat_step, HeatRunner and gsrb_solve.

Mirrors the reference's own pins: test_kernels.py:259-283 (tiling /
workers / layout transparency, bitwise) and test_acceptance.py:219-241.
"""

import os

import numpy as np
import pytest

from oracle import oracle as orc

pytestmark = pytest.mark.gpu

C2_REFERENCE_SUM = 16870634.63599003  # reference reduce_sum after 100 C2 steps


@pytest.fixture(scope="module")
def tm():
    import torch

    import paper_1604_03570_b200 as tm

    torch.cuda.set_device(0)
    return tm


def uniform_init(w, seed=5):
    rng = np.random.default_rng(seed)
    return rng.random((w.ncomp, w.n, w.n, w.n))


def oracle_run(tm, w, glob, steps):
    """The reference path restated in C (tag FillBoundary + per-component
    heat_tiles with the config's tiles), OpenMP over the host's threads."""
    from paper_1604_03570_b200.box import decompose
    from paper_1604_03570_b200.fillplan import build_fill_plan_units

    ba = tm.BoxArray.chop(w.domain, w.max_grid_size)
    valids = list(ba)
    geom = tm.Geometry(w.domain, (True, True, True), (w.dx,) * 3)
    plan = build_fill_plan_units(valids, geom, w.nghost, grids=valids)
    nt = orc.max_threads()
    old = orc.HostMF(valids, w.ncomp, w.nghost)
    old.from_global(glob)
    new = orc.HostMF(valids, w.ncomp, w.nghost)
    tags = orc.tags_array(plan.tags)
    tiles = orc.tiles_array([(u, t) for u in range(len(valids)) for t in decompose(valids[u], w.tile_size)])
    c = tm.HeatParams.stable(1.0, geom.dx).coefficients()
    for _ in range(steps):
        orc.fill_boundary(old, tags, nt)
        orc.heat_step(new, old, tiles, c[:3], c[3], nt)
        old, new = new, old
    return old


def device_setup(tm, w, glob):
    geom = tm.Geometry(w.domain, (True, True, True), (w.dx,) * 3)
    ba = tm.BoxArray.chop(w.domain, w.max_grid_size)
    mf = tm.MultiFab(ba, w.ncomp, w.nghost)
    mf.from_global(glob)
    return geom, ba, mf


def assert_ghosts_are_fresh_fill(tm, out, geom):
    import torch

    ref = out.clone_empty()
    ref.data.copy_(out.data)
    tm.fill_boundary(ref, geom)
    assert torch.equal(out.data.view(torch.int64), ref.data.view(torch.int64))


def assert_equal_oracle(out, host, w):
    got = out.to_global().cpu().numpy()
    exp = host.to_global((w.n,) * 3)
    bad = np.argwhere(got != exp)
    assert bad.size == 0, f"{len(bad)} cells differ from the oracle, first at (c,z,y,x)={tuple(bad[0])}"


def test_c2_bench_path_full_size(tm):
    """C2 exactly as bench.py runs it: default HeatRunner on 256^3 / 64 boxes,
    graph replay of step pairs, 100 steps."""
    from paper_1604_03570_b200 import _native
    from paper_1604_03570_b200.runner import HeatRunner

    w = tm.CONFIGS["C2"]
    glob = tm.make_init(w)
    geom, ba, mf = device_setup(tm, w, glob)
    sched = tm.build_schedule(mf, w.tile_size)
    r = HeatRunner(mf, geom, tm.HeatParams.stable(1.0, geom.dx), sched)
    assert r.fused and r.use_graph and r.fh.mode == _native.HALO_FUSED_NBR
    out = r.advance(w.steps)
    host = oracle_run(tm, w, glob, w.steps)
    assert_equal_oracle(out, host, w)
    s = out.reduce_sum()
    assert s == orc.reduce_sum(host) == C2_REFERENCE_SUM
    assert_ghosts_are_fresh_fill(tm, out, geom)
    # the bench's e2e job: re-upload, reset, advance again -> same bits
    mf2 = r.a
    mf2.from_global(glob)
    r.reset()
    assert r.advance(w.steps).reduce_sum() == C2_REFERENCE_SUM


@pytest.mark.parametrize("n,steps", [(256, 7), (512, 10)])
def test_c3_shape_128wide_fused(tm, n, steps):
    """The C3 kernel instance (128-wide boxes: CPL 4, 32-row columns, one
    17-warp CTA per SM, 4 comps, 2 ghosts), fused runner with graph and
    alternating direction; n = 512 is the full C3 shape (uniform init: the
    Gaussian init costs ~70 s of host time and changes no code path)."""
    from paper_1604_03570_b200.runner import HeatRunner

    w = tm.CONFIGS["C3"].scaled(n, 128, steps)
    glob = uniform_init(w)
    geom, ba, mf = device_setup(tm, w, glob)
    r = HeatRunner(mf, geom, tm.HeatParams.stable(1.0, geom.dx), w.tile_size)
    assert r.fused and r.fh.plan.columns["ny"].max() == 32 and r.fh.plan.columns["nx"].max() == 128
    out = r.advance(steps)
    assert_equal_oracle(out, oracle_run(tm, w, glob, steps), w)
    assert_ghosts_are_fresh_fill(tm, out, geom)


@pytest.mark.parametrize("reverse_pattern", ["fwd", "rev", "mixed"])
def test_c3_shape_fused_halo_directions(tm, reverse_pattern):
    """FusedHalo on 128-wide boxes, default rows: forward, reverse and mixed
    march directions all give the oracle's bits."""
    from paper_1604_03570_b200.march import FusedHalo

    steps = 4
    w = tm.CONFIGS["C3"].scaled(256, 128, steps)
    glob = uniform_init(w, 11)
    geom, ba, a = device_setup(tm, w, glob)
    b = a.clone_empty()
    p = tm.HeatParams.stable(1.0, geom.dx)
    fh = FusedHalo(a, b, geom)
    fh.prime(a)
    for k in range(steps):
        rev = {"fwd": False, "rev": True, "mixed": k % 3 != 1}[reverse_pattern]
        fh.step(b, a, p, reverse=rev)
        a, b = b, a
    tm.fill_boundary(a, geom)
    assert_equal_oracle(a, oracle_run(tm, w, glob, steps), w)


def gsrb_oracle(tm, w, rhs_g, sweeps):
    """Reference-shaped GSRB restated in C: (red, FillBoundary, black,
    FillBoundary) x sweeps, then the residual max-norm."""
    from paper_1604_03570_b200.box import decompose
    from paper_1604_03570_b200.fillplan import build_fill_plan_units

    ba = tm.BoxArray.chop(w.domain, w.max_grid_size)
    valids = list(ba)
    geom = tm.Geometry(w.domain, (True, True, True), (w.dx,) * 3)
    tags = orc.tags_array(build_fill_plan_units(valids, geom, 1, grids=valids).tags)
    tiles = orc.tiles_array([(u, t) for u in range(len(valids)) for t in decompose(valids[u], w.tile_size)])
    nt = orc.max_threads()
    phi = orc.HostMF(valids, 1, 1)
    rhs = orc.HostMF(valids, 1, 0)
    rhs.from_global(rhs_g)
    h2 = w.dx * w.dx
    for _ in range(sweeps):
        for color in (0, 1):
            orc.gsrb_color(phi, rhs, tiles, color, h2, nt)
            orc.fill_boundary(phi, tags, nt)
    return phi, orc.residual_max(phi, rhs, tiles, h2, nt)


@pytest.mark.parametrize("split", [True, False])
def test_c4_full_size_matches_oracle(tm, split):
    """BASELINE config 4 at full size (256^3, 64 boxes, 50 sweeps)."""
    w = tm.CONFIGS["C4"]
    rhs_g = tm.make_init(w)
    geom = tm.Geometry(w.domain, (True, True, True), (w.dx,) * 3)
    ba = tm.BoxArray.chop(w.domain, w.max_grid_size)
    phi = tm.MultiFab(ba, 1, 1)
    rhs = tm.MultiFab(ba, 1, 0)
    rhs.from_global(rhs_g)
    tm.gsrb_solve(phi, rhs, geom, w.steps, fused=True, split=split)
    host, res = gsrb_oracle(tm, w, rhs_g, w.steps)
    assert_equal_oracle(phi, host, w)
    assert tm.residual_maxnorm(phi, rhs, geom) == res


@pytest.mark.parametrize("n,steps", [(512, 6)] + ([(1024, 20)] if os.environ.get("TM_TEST_FULL_C5") == "1" else []))
def test_c5_shape_fused(tm, n, steps):
    """C5's kernel instance: 32^3 boxes (1 cell per lane), 2 comps, 2 ghosts,
    thousands of boxes, fused runner with graph (n = 1024 is the full C5)."""
    from paper_1604_03570_b200.runner import HeatRunner

    w = tm.CONFIGS["C5"].scaled(n, 32, steps)
    glob = uniform_init(w, 3)
    geom, ba, mf = device_setup(tm, w, glob)
    r = HeatRunner(mf, geom, tm.HeatParams.stable(1.0, geom.dx), w.tile_size)
    assert r.fused and len(mf.local_units) == (n // 32) ** 3
    out = r.advance(steps)
    host = oracle_run(tm, w, glob, steps)
    assert_equal_oracle(out, host, w)
    assert [out.reduce_sum(c) for c in range(w.ncomp)] == [orc.reduce_sum(host, c) for c in range(w.ncomp)]


@pytest.mark.parametrize("width", [66, 70, 98])
def test_widths_the_march_declines(tm, width):
    """Boxes wider than 64 whose width is not a multiple of 4 fall back to the
    tile kernel (heat_step), the unfused runner and the unfused GSRB -- and
    still give the oracle's bits (they used to raise)."""
    from paper_1604_03570_b200.march import fusable, march_eligible
    from paper_1604_03570_b200.runner import HeatRunner

    dom = tm.Box((0, 0, 0), (2 * width - 1, 127, 127))  # >= 2^21 cells: heat_step's march threshold
    geom = tm.Geometry(dom, (True, True, True), (1.0 / 128,) * 3)
    ba = tm.BoxArray.chop(dom, width)
    rng = np.random.default_rng(width)
    glob = rng.random((1, 128, 128, 2 * width))
    old = tm.MultiFab(ba, 1, 1)
    old.from_global(glob)
    assert not march_eligible(old) and not fusable(old, geom)
    p = tm.HeatParams.stable(1.0, geom.dx)
    c = p.coefficients()
    exp = orc.heat_periodic(glob, 2, c[:3], c[3])
    new = old.clone_empty()
    for _ in range(2):
        tm.fill_boundary(old, geom)
        tm.heat_step(new, old, geom, p, (1024, 8, 8))
        old, new = new, old
    assert np.array_equal(old.to_global().cpu().numpy(), exp)
    mf = tm.MultiFab(ba, 1, 1)
    mf.from_global(glob)
    r = HeatRunner(mf, geom, p, (1024, 8, 8))
    assert not r.fused
    assert np.array_equal(r.advance(2).to_global().cpu().numpy(), exp)
    phi = tm.MultiFab(ba, 1, 1)
    rhs = tm.MultiFab(ba, 1, 0)
    rhs.from_global(glob - 0.5)
    tm.gsrb_solve(phi, rhs, geom, 2)
    ref_phi, ref_res = orc.gsrb_periodic(np.zeros(glob.shape[1:]), glob[0] - 0.5, 2, geom.dx[0] * geom.dx[0])
    assert np.array_equal(phi.to_global().cpu().numpy()[0], ref_phi)
    assert tm.residual_maxnorm(phi, rhs, geom) == ref_res
