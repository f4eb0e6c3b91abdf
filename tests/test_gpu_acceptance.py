"""The reference's acceptance criteria for the path, run through the device
library (reference pkg/tests/test_acceptance.py):

* criterion 3 (test_acceptance.py:124-139): >= 200 randomized disjoint box
  layouts, random periodicity and ghost depth; after ONE device FillBoundary
  every fillable ghost (and every valid cell) of every allocation box holds
  the periodic image of a linear field and every unfillable ghost still holds
  the sentinel -- checked by a brute-force periodic-image search written here,
  independent of the fill plan;
* criterion 6 (test_acceptance.py:219-241): the checksum after 20 steps of
  fill_boundary + step on 64^3 is bitwise identical across tiling x workers x
  layout (3 x 3 x 2 = 18 variants) for both kernels -- and equal to the C
  oracle's / numpy oracle's checksum of the same run.
"""

import dataclasses

import numpy as np
import pytest

from oracle import oracle as orc

pytestmark = pytest.mark.gpu

SENTINEL = -987654.321


@pytest.fixture(scope="module")
def tm():
    import torch

    import paper_1604_03570_b200 as tm

    torch.cuda.set_device(0)
    return tm


def random_disjoint(tm, rng, domain):
    """A chop of the domain with ~30 % of the boxes dropped (holes make some
    ghosts unfillable)."""
    mgs = tuple(int(v) for v in rng.integers(2, 9, 3))
    cands = tm.BoxArray.chop(domain, mgs).boxes
    keep = [b for b in cands if rng.random() < 0.7]
    return keep or cands[:1]


def expected_allocation(tm, mf, geom, u):
    """Linear field at the periodic image of every cell of unit u's allocation
    box where some valid box covers that image, else the sentinel."""
    dom = geom.domain
    n = dom.extents
    b = mf.fab(u).abox
    axes = np.meshgrid(*[np.arange(b.lo[d], b.hi[d] + 1) for d in range(3)], indexing="ij")
    img = []
    for d in range(3):
        a = axes[d]
        if geom.periodic[d]:
            a = dom.lo[d] + (a - dom.lo[d]) % n[d]
        img.append(a)
    covered = np.zeros(img[0].shape, dtype=bool)
    for v in (x.valid for x in mf.units):
        m = np.ones(img[0].shape, dtype=bool)
        for d in range(3):
            m &= (img[d] >= v.lo[d]) & (img[d] <= v.hi[d])
        covered |= m
    return np.where(covered, img[0] + 10.0 * img[1] + 100.0 * img[2], SENTINEL)


def test_criterion_3_ghost_fill_randomized(tm):
    rng = np.random.default_rng(77)
    trials = 200
    for t in range(trials):
        hi = tuple(int(v) for v in rng.integers(3, 16, 3))
        dom = tm.Box((0, 0, 0), hi)
        geom = tm.Geometry(dom, tuple(bool(v) for v in rng.integers(0, 2, 3)))
        ng = int(rng.choice([1, 2, 4]))
        mf = tm.MultiFab(tm.BoxArray(random_disjoint(tm, rng, dom)), 1, ng)
        mf.fill(SENTINEL)
        mf.set_from_function(lambda i, j, k: i + 10.0 * j + 100.0 * k)
        tm.fill_boundary(mf, geom, workers=int(rng.choice([1, 3])))
        for u in mf.local_units:
            f = mf.fab(u)
            got = f.view(f.abox, 0, 1)[..., 0].cpu().numpy()
            assert np.array_equal(got, expected_allocation(tm, mf, geom, u)), (t, u)


@pytest.mark.parametrize("kernel", ["heat", "wide4"])
def test_criterion_6_transparency(tm, kernel):
    n, steps = 64, 20
    w = tm.CONFIGS["C1"].scaled(n, 32, steps)
    if kernel == "wide4":
        w = dataclasses.replace(w, nghost=4)
    glob = tm.make_init(w)
    geom = tm.Geometry(w.domain, (True, True, True), (w.dx,) * 3)
    params = tm.HeatParams.stable(1.0, geom.dx)
    dt4 = tm.wide4_stable_dt(1.0, geom.dx)
    coeffs = tm.derive_coeffs8()
    tilings = [None, (128, 4, 4), (32, 8, 8)]
    workers = [1, 4, 16]
    layouts = [(tm.CONTIGUOUS, None), (tm.REGIONAL, (64, 64, 64))]
    sums = set()
    variants = 0
    for ts in tilings:
        for nw in workers:
            for layout, region in layouts:
                ba = tm.BoxArray.chop(w.domain, w.max_grid_size)
                old = tm.MultiFab(ba, 1, w.nghost, layout, region)
                old.from_global(glob)
                new = old.clone_empty()
                sched = tm.build_schedule(old, ts) if ts is not None else None
                plan = tm.build_fill_plan(old, geom)
                for _ in range(steps):
                    tm.fill_boundary(old, geom, plan, workers=nw)
                    if kernel == "heat":
                        tm.heat_step(new, old, geom, params, sched, workers=nw)
                    else:
                        tm.wide4_step(new, old, geom, 1.0, dt4, sched, workers=nw, coeffs=coeffs)
                    old, new = new, old
                sums.add(old.reduce_sum())
                variants += 1
    assert variants == 18
    assert len(sums) == 1, sums
    # the same run on the CPU oracles: the serial reduce_sum chain of the final field
    if kernel == "heat":
        c = params.coefficients()
        want = orc.heat_periodic(glob, steps, c[:3], c[3])[0]
    else:
        want = orc.wide4_periodic(glob[0], steps, coeffs.as_array(), tuple(1.0 / d ** 2 for d in geom.dx), dt4)
    mf = tm.MultiFab(tm.BoxArray.chop(w.domain, w.max_grid_size), 1, w.nghost)
    mf.from_global(want[None])
    assert mf.reduce_sum() == sums.pop()
