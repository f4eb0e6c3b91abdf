"""The reference-shaped step loop -- ``fill_boundary(old); heat_step(new,
old)`` per step, exactly as the reference's bench (_timed_loop,
/root/reference/pkg/src/tilemesh/bench.py:183-223) and INTEGRATION.md §1
drive it -- on its fast path: heat_step keeps packed x halos of the field it
writes; fill_boundary of such a field runs only the edge/corner copies and
leaves the face ghosts pending; the next heat_step reads its halos from the
neighbours' valid cells and the packed halos and writes them into the face
ghosts as it goes.  Every result must equal the oracle bit for bit, every
ghost a caller can observe must equal a regular FillBoundary's, and any
write to a field between the calls must send the next call back to the
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
    """Nothing touches the fields between the calls: from the second step on, fill_boundary
    leaves the face ghosts pending (one ghost layer) and heat_step's sweep writes them; after
    every heat_step the input's ghosts must be exactly a regular FillBoundary's."""
    w = tm.CONFIGS[cfg].scaled(n, mgs, steps)
    geom, ba, glob, old = setup(tm, w)
    new = old.clone_empty()
    p = tm.HeatParams.stable(1.0, geom.dx)
    sched = tm.build_schedule(old, w.tile_size)
    plan = tm.build_fill_plan(old, geom)
    deferred = 0
    for k in range(steps):
        tm.fill_boundary(old, geom, plan)
        if k >= 1:  # the previous heat_step left current packed halos
            assert old.xh_current()
            deferred += old._pending_faces is not None
        settles = old.settles
        tm.heat_step(new, old, geom, p, sched)
        assert old.settles == settles, "heat_step settled the deferred faces instead of writing them"
        assert old._pending_faces is None and new.xh_current() and not new.ghosts_current()
        assert_same_fabs(old, fresh_fill(tm, old, geom))  # faces written by the sweep, edges by the fill
        old, new = new, old
    assert deferred == (steps - 1 if w.nghost == 1 else 0)
    c = p.coefficients()
    assert np.array_equal(old.to_global().cpu().numpy(), orc.heat_periodic(glob, steps, c[:3], c[3]))


def test_pending_faces_settle_on_access(tm):
    """A caller who looks at the storage between fill_boundary and heat_step sees every
    ghost filled (the deferred faces are written first), and the step is still exact."""
    w = tm.CONFIGS["C2"].scaled(128, 64, 3)
    geom, ba, glob, old = setup(tm, w)
    new = old.clone_empty()
    p = tm.HeatParams.stable(1.0, geom.dx)
    tm.fill_boundary(old, geom)
    tm.heat_step(new, old, geom, p)
    tm.fill_boundary(new, geom)
    assert new._pending_faces is not None
    v = ba[3]
    ghost = new.fab(3).at(v.lo[0] - 1, v.lo[1] + 5, v.lo[2] + 7)  # FAB view access settles
    assert new._pending_faces is None
    assert_same_fabs(new, fresh_fill(tm, new, geom))
    assert np.isfinite(ghost)
    tm.heat_step(old, new, geom, p)
    c = p.coefficients()
    assert np.array_equal(old.to_global().cpu().numpy(), orc.heat_periodic(glob, 2, c[:3], c[3]))


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


@pytest.mark.parametrize("cfg,n,mgs,steps", [("C2", 128, 64, 5), ("C2", 128, 64, 6), ("C1", 128, 32, 4)])
def test_every_ghost_matches_the_reference_loop(tm, cfg, n, mgs, steps):
    """The whole storage of BOTH fields -- valid cells and every ghost, including
    the ghosts a field keeps from its last fill while later steps overwrite its
    valid cells -- equals the reference loop's, restated in C (tag FillBoundary +
    heat_tiles on host FABs), after an uninterrupted run of the fast path."""
    from paper_1604_03570_b200.box import decompose
    from paper_1604_03570_b200.fillplan import build_fill_plan_units

    w = tm.CONFIGS[cfg].scaled(n, mgs, steps)
    geom, ba, glob, a = setup(tm, w)
    b = tm.MultiFab(ba, w.ncomp, w.nghost)  # zero storage on both sides
    p = tm.HeatParams.stable(1.0, geom.dx)
    plan = tm.build_fill_plan(a, geom)
    old, new = a, b
    for _ in range(steps):
        tm.fill_boundary(old, geom, plan)
        tm.heat_step(new, old, geom, p)
        old, new = new, old
    assert a.settles == 0 and b.settles == 0  # nothing was settled during the loop
    valids = list(ba)
    ha, hb = orc.HostMF(valids, w.ncomp, w.nghost), orc.HostMF(valids, w.ncomp, w.nghost)
    ha.from_global(glob)
    tags = orc.tags_array(build_fill_plan_units(valids, geom, w.nghost, grids=valids).tags)
    tiles = orc.tiles_array([(u, t) for u in range(len(valids)) for t in decompose(valids[u], w.tile_size)])
    c = p.coefficients()
    ho, hn = ha, hb
    for _ in range(steps):
        orc.fill_boundary(ho, tags, 4)
        orc.heat_step(hn, ho, tiles, c[:3], c[3], 4)
        ho, hn = hn, ho
    for dev, host in ((a, ha), (b, hb)):
        for u in range(len(valids)):
            got = dev.fab(u).to_numpy()
            assert np.array_equal(got.view(np.int64), host.fab(u).view(np.int64)), f"unit {u}"
