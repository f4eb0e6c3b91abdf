"""The reference-shaped step loop -- ``fill_boundary(old); heat_step(new,
old)`` per step, exactly as the reference's bench (_timed_loop,
/root/reference/pkg/src/tilemesh/bench.py:183-223) and INTEGRATION.md §1
drive it -- on its fast path: heat_step keeps packed x halos of the field it
writes, fill_boundary writes the x-face ghosts from them, and a heat_step
whose input has current halos and freshly filled ghosts reads y/z halos from
the neighbours' valid cells.  Every result must equal the oracle bit for
bit, every ghost must equal a regular FillBoundary's after each fill, and
any write to a field between the calls must send the next call back to the
general path (it reads what the caller wrote)."""

import numpy as np
import pytest

from oracle import oracle as orc

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def tm():
    import torch

    import paper_1604_03570_b200 as tm

    torch.cuda.set_device(0)
    return tm


def setup(tm, w):
    geom = tm.Geometry(w.domain, (True, True, True), (w.dx,) * 3)
    ba = tm.BoxArray.chop(w.domain, w.max_grid_size)
    rng = np.random.default_rng(17)
    glob = rng.random((w.ncomp,) + (w.n,) * 3)
    mf = tm.MultiFab(ba, w.ncomp, w.nghost)
    mf.from_global(glob)
    return geom, ba, glob, mf


def fresh_fill(tm, mf, geom):
    """Ghosts of ``mf`` as the general FillBoundary path writes them."""
    ref = mf.clone_empty()
    ref.data.copy_(mf.data)  # a torch write: ref's packed halos are not current
    assert not ref.xh_current()
    tm.fill_boundary(ref, geom)
    return ref


def assert_same_fabs(a, b):
    import torch

    for u in a.local_units:
        assert torch.equal(a.fab(u).data.contiguous().view(torch.int64), b.fab(u).data.contiguous().view(torch.int64))


@pytest.mark.parametrize("cfg,n,mgs,steps", [("C2", 128, 64, 6), ("C1", 128, 32, 5), ("C3", 256, 128, 4)])  # >= 2^21 cells: heat_step marches
def test_reference_loop_fast_path(tm, cfg, n, mgs, steps):
    w = tm.CONFIGS[cfg].scaled(n, mgs, steps)
    geom, ba, glob, old = setup(tm, w)
    new = old.clone_empty()
    p = tm.HeatParams.stable(1.0, geom.dx)
    sched = tm.build_schedule(old, w.tile_size)
    plan = tm.build_fill_plan(old, geom)
    for k in range(steps):
        tm.fill_boundary(old, geom, plan)
        assert old.ghosts_current()
        if k >= 1:  # the previous heat_step left current packed halos: fast fill + neighbour-halo sweep
            assert old.xh_current()
        assert_same_fabs(old, fresh_fill(tm, old, geom))
        tm.heat_step(new, old, geom, p, sched)
        assert new.xh_current() and not new.ghosts_current()
        old, new = new, old
    c = p.coefficients()
    assert np.array_equal(old.to_global().cpu().numpy(), orc.heat_periodic(glob, steps, c[:3], c[3]))


def test_writes_between_calls_take_the_general_path(tm):
    """A ghost the caller sets after fill_boundary is what heat_step reads; a
    valid cell set after heat_step is what the next fill copies."""
    from paper_1604_03570_b200 import stencil

    w = tm.CONFIGS["C2"].scaled(128, 64, 3)
    geom, ba, glob, old = setup(tm, w)
    new = old.clone_empty()
    p = tm.HeatParams.stable(1.0, geom.dx)
    for _ in range(2):  # reach the fast path
        tm.fill_boundary(old, geom)
        tm.heat_step(new, old, geom, p)
        old, new = new, old
    tm.fill_boundary(old, geom)
    assert old.xh_current() and old.ghosts_current()
    v = ba[0]
    old.fab(0).set_at(v.lo[0] - 1, v.lo[1] + 3, v.lo[2] + 5, 7.25)  # an x-face ghost
    old.fab(0).set_at(v.lo[0] + 2, v.hi[1] + 1, v.lo[2] + 1, -3.5)  # a y-face ghost
    assert not old.ghosts_current()
    # expected: the tile kernel (always reads the ghosts) on a copy of the same state
    twin = old.clone_empty()
    twin.data.copy_(old.data)
    twin_new = old.clone_empty()
    prev = stencil.SWEEP_KERNEL
    stencil.SWEEP_KERNEL = "tiled"
    try:
        tm.heat_step(twin_new, twin, geom, p)
    finally:
        stencil.SWEEP_KERNEL = prev
    tm.heat_step(new, old, geom, p)
    assert np.array_equal(new.to_global().cpu().numpy(), twin_new.to_global().cpu().numpy())
    # a valid cell written after the step: the next fill must copy it
    assert new.xh_current()
    new.fab(1).set_at(*ba[1].lo, 42.0)
    assert not new.xh_current()
    tm.fill_boundary(new, geom)
    assert_same_fabs(new, fresh_fill(tm, new, geom))
