"""The reference's per-tile heat operations on device FABs -- heat_flux and
heat_divergence_update (kernels.py:86-144; compiled.flux_x/y/z and
compiled.divergence, compiled.py:32-81) -- mirroring the reference's own tests
(test_kernels.py:123-200): zero flux of a constant field, the gradient of a
linear field, random data against a loop oracle (bitwise), rejected centring
and missing ghosts, and the divergence update against the loop oracle -- and,
bitwise, against heat_step on the same tile."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def tm():
    import torch

    import paper_1604_03570_b200 as tm

    torch.cuda.set_device(0)
    return tm


def one_box(tm, hi, nghost=1, fill=None, seed=None):
    """A MultiFab of the single box [0, hi] (non-periodic) and its device FAB."""
    import torch

    dom = tm.Box((0, 0, 0), hi)
    mf = tm.MultiFab(tm.BoxArray([dom]), 1, nghost)
    fab = mf.fab(0)
    if fill is not None:
        fab.fill(fill)
    if seed is not None:
        rng = np.random.default_rng(seed)
        fab.data.copy_(torch.from_numpy(rng.random(tuple(fab.data.shape))))
    return mf, fab


def flux_oracle(a, lo, face_box, d, dx):
    """Loop restatement of compiled.flux_x/y/z on a host copy ``a`` (x, y, z)
    whose first cell is ``lo``."""
    e = [0, 0, 0]
    e[d] = 1
    out = np.empty(face_box.extents)
    for k in range(face_box.lo[2], face_box.hi[2] + 1):
        for j in range(face_box.lo[1], face_box.hi[1] + 1):
            for i in range(face_box.lo[0], face_box.hi[0] + 1):
                hi_c = a[i - lo[0], j - lo[1], k - lo[2]]
                lo_c = a[i - e[0] - lo[0], j - e[1] - lo[1], k - e[2] - lo[2]]
                out[i - face_box.lo[0], j - face_box.lo[1], k - face_box.lo[2]] = (hi_c - lo_c) * (1.0 / dx)
    return out


def test_constant_field_zero_flux(tm):
    _, fab = one_box(tm, (3, 3, 3), fill=3.0)
    for d in range(3):
        f = tm.heat_flux(fab, tm.to_face(tm.Box((0, 0, 0), (3, 3, 3)), d), d, 0.5)
        assert bool((f == 0.0).all())


def test_linear_field_constant_gradient(tm):
    import torch

    _, fab = one_box(tm, (3, 3, 3))
    b = fab.abox
    I, J, K = np.ogrid[b.lo[0]:b.hi[0] + 1, b.lo[1]:b.hi[1] + 1, b.lo[2]:b.hi[2] + 1]
    fab.data[..., 0].copy_(torch.from_numpy(np.broadcast_to(2.0 * I + 3.0 * J + 5.0 * K, b.extents).copy()))
    dx = 0.25
    for d, g in enumerate((2.0, 3.0, 5.0)):
        f = tm.heat_flux(fab, tm.to_face(tm.Box((0, 0, 0), (3, 3, 3)), d), d, dx).cpu().numpy()
        assert np.allclose(f, g / dx, rtol=1e-14, atol=0.0)


def test_random_vs_loop_oracle(tm):
    _, fab = one_box(tm, (5, 4, 3), seed=11)
    a = fab.to_numpy()[..., 0]
    for d in range(3):
        fb = tm.to_face(tm.Box((0, 0, 0), (4, 3, 2)), d)
        got = tm.heat_flux(fab, fb, d, 0.125).cpu().numpy()
        assert np.array_equal(got, flux_oracle(a, fab.abox.lo, fb, d, 0.125))


def test_wrong_centering_and_missing_ghost_rejected(tm):
    _, fab = one_box(tm, (3, 3, 3), fill=1.0)
    with pytest.raises(ValueError):
        tm.heat_flux(fab, tm.Box((0, 0, 0), (3, 3, 3)), 0, 1.0)
    _, bare = one_box(tm, (3, 3, 3), nghost=0, fill=1.0)
    with pytest.raises(ValueError):
        tm.heat_flux(bare, tm.to_face(tm.Box((0, 0, 0), (3, 3, 3)), 0), 0, 1.0)


def step_on_tile(tm, mf_old, tile, params):
    mf_new = mf_old.clone_empty()
    mf_new.fill(0.0)
    fab_old, fab_new = mf_old.fab(0), mf_new.fab(0)
    fluxes = tuple(tm.heat_flux(fab_old, tm.to_face(tile, d), d, params.dx[d]) for d in range(3))
    tm.heat_divergence_update(fab_new, fab_old, fluxes, tile, params)
    return mf_new


def test_divergence_constant_field_unchanged(tm):
    mf, _ = one_box(tm, (3, 3, 3), fill=7.0)
    tile = tm.Box((0, 0, 0), (3, 3, 3))
    out = step_on_tile(tm, mf, tile, tm.HeatParams(1.0, 1e-3, (0.25,) * 3))
    assert bool((out.fab(0).view(tile) == 7.0).all())


def test_divergence_loop_oracle_and_heat_step(tm):
    mf, fab = one_box(tm, (3, 3, 3), seed=23)
    tile = tm.Box((0, 0, 0), (3, 3, 3))
    params = tm.HeatParams(2.0, 1e-3, (0.5, 0.25, 0.125))
    out = step_on_tile(tm, mf, tile, params)
    a = fab.to_numpy()[..., 0]
    o = out.fab(0).to_numpy()[..., 0]
    dtD = params.diffusivity * params.dt
    dxi = tuple(1.0 / d for d in params.dx)
    at = lambda i, j, k: a[i + 1, j + 1, k + 1]  # noqa: E731  (abox starts at -1)
    for k in range(4):
        for j in range(4):
            for i in range(4):
                div = ((at(i + 1, j, k) - 2 * at(i, j, k) + at(i - 1, j, k)) * dxi[0] ** 2
                       + (at(i, j + 1, k) - 2 * at(i, j, k) + at(i, j - 1, k)) * dxi[1] ** 2
                       + (at(i, j, k + 1) - 2 * at(i, j, k) + at(i, j, k - 1)) * dxi[2] ** 2)
                assert o[i + 1, j + 1, k + 1] == pytest.approx(at(i, j, k) + dtD * div, rel=1e-13)
    # the same bits as heat_step on the tile (the reference's flux form, same order)
    geom = tm.Geometry(tm.Box((0, 0, 0), (3, 3, 3)), (False, False, False), params.dx)
    ref = mf.clone_empty()
    ref.fill(0.0)
    tm.heat_step(ref, mf, geom, params)
    assert np.array_equal(out.fab(0).to_numpy(), ref.fab(0).to_numpy())
