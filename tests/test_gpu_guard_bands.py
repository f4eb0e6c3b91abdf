"""Out-of-bounds write check without compute-sanitizer (closed on this GPU
pool): every device allocation the package makes through ``torch.empty`` /
``torch.zeros`` while a case runs is placed between two canary bands, the
production kernels run over it, and every band must come back untouched.
Results are compared with the oracle as usual; the guarded tensors start on
odd multiples of 512 B (the allocator's minimum alignment, not the 2 MiB of a
fresh large block), a second placement of every TMA tensor map."""

import dataclasses

import numpy as np
import pytest

from oracle import oracle as orc

pytestmark = pytest.mark.gpu

BAND = (1 << 16) + 512  # bytes on each side of every allocation (an odd multiple of 512)
CANARY = 0xA5


class GuardBands:
    """Context manager: device allocations get canary bands; ``check()``
    returns the allocations whose bands changed."""

    def __init__(self):
        self.allocs = []

    def _wrap(self, orig, zero):
        import torch

        def alloc(*size, **kw):
            dev = kw.get("device")
            if set(kw) - {"dtype", "device"} or dev is None or torch.device(dev).type != "cuda":
                return orig(*size, **kw)
            shape = tuple(size[0]) if len(size) == 1 and not isinstance(size[0], int) else tuple(size)
            dtype = kw.get("dtype") or torch.get_default_dtype()
            nbytes = int(np.prod(shape, dtype=np.int64)) * dtype.itemsize
            body = -(-nbytes // 512) * 512  # the far band starts 512-B aligned, as a fresh block would
            raw = self._empty(body + 2 * BAND, dtype=torch.uint8, device=dev)
            raw[:BAND] = CANARY
            raw[BAND + nbytes:] = CANARY
            mid = raw[BAND:BAND + nbytes].view(dtype).view(shape)
            if zero:
                mid.zero_()
            self.allocs.append((raw, nbytes, shape, str(dtype)))
            return mid

        return alloc

    def __enter__(self):
        import torch

        self._empty, self._zeros = torch.empty, torch.zeros
        torch.empty = self._wrap(self._empty, False)
        torch.zeros = self._wrap(self._empty, True)
        return self

    def __exit__(self, *exc):
        import torch

        torch.empty, torch.zeros = self._empty, self._zeros

    def check(self):
        import torch

        torch.cuda.synchronize()
        bad = []
        for raw, nbytes, shape, dtype in self.allocs:
            lo_ok = bool((raw[:BAND] == CANARY).all())
            hi_ok = bool((raw[BAND + nbytes:] == CANARY).all())
            if not (lo_ok and hi_ok):
                bad.append((shape, dtype, "below" if not lo_ok else "above"))
        return bad


@pytest.fixture(scope="module")
def tm():
    import torch

    import paper_1604_03570_b200 as tm

    torch.cuda.set_device(0)
    return tm


def heat_oracle(tm, w, glob, steps):
    c = tm.HeatParams.stable(1.0, (w.dx,) * 3).coefficients()
    return orc.heat_periodic(glob, steps, c[:3], c[3])


def test_guard_detects_a_stray_write(tm):
    """The check itself: one double written past the end of a guarded tensor is reported."""
    import torch

    with GuardBands() as g:
        t = torch.zeros(1000, dtype=torch.float64, device="cuda")
        assert g.check() == []
        torch.as_strided(t, (1,), (1,), t.storage_offset() + 1000).fill_(1.0)  # element 1000: the far band's first
        assert g.check() == [((1000,), "torch.float64", "above")]
        torch.as_strided(t, (1,), (1,), t.storage_offset() - 1).fill_(1.0)  # element -1
        assert g.check() == [((1000,), "torch.float64", "below")]


@pytest.mark.parametrize("cfg,n,mgs,steps,rows", [
    ("C2", 128, 64, 5, None),   # the bench kernel instance (64-wide boxes, 2 cells per lane)
    ("C2", 96, 32, 4, 8),       # half-warp rows, several columns per box
    ("C3", 256, 128, 2, None),  # 128-wide boxes, 4 components, 2 ghosts
    ("C5", 64, 32, 4, None),    # 32^3 boxes, 2 components, 2 ghosts
    ("C5", 64, 16, 3, None),    # 16-wide boxes, 1 cell per lane
])
def test_fused_heat_runner_stays_inside_its_allocations(tm, cfg, n, mgs, steps, rows):
    from paper_1604_03570_b200.runner import HeatRunner

    w = tm.CONFIGS[cfg].scaled(n, mgs, steps)
    geom = tm.Geometry(w.domain, (True, True, True), (w.dx,) * 3)
    ba = tm.BoxArray.chop(w.domain, w.max_grid_size)
    glob = tm.make_init(w)
    with GuardBands() as g:
        mf = tm.MultiFab(ba, w.ncomp, w.nghost)
        mf.from_global(glob)
        r = HeatRunner(mf, geom, tm.HeatParams.stable(1.0, geom.dx), w.tile_size, fused=True, march_rows=rows,
                       use_graph=False)
        assert r.fused
        out = r.advance(steps)  # both march directions + the closing FillBoundary
        got = out.to_global().cpu().numpy()
        assert len(g.allocs) >= 3  # both fields and the packed x halos at least
        assert g.check() == []
    assert np.array_equal(got, heat_oracle(tm, w, glob, steps))


@pytest.mark.parametrize("n,mgs", [(128, 64), (64, 32), (48, 24)])
def test_reference_loop_stays_inside_its_allocations(tm, n, mgs):
    """fill_boundary; heat_step -- the deferred-ghost fast path on the large
    case (march + fill warp), Kernel B + the tile kernel on the small ones."""
    steps = 4
    w = tm.CONFIGS["C2"].scaled(n, mgs, steps)
    geom = tm.Geometry(w.domain, (True, True, True), (w.dx,) * 3)
    ba = tm.BoxArray.chop(w.domain, w.max_grid_size)
    glob = tm.make_init(w)
    p = tm.HeatParams.stable(1.0, geom.dx)
    with GuardBands() as g:
        old = tm.MultiFab(ba, w.ncomp, w.nghost)
        old.from_global(glob)
        new = old.clone_empty()
        plan = tm.build_fill_plan(old, geom)
        sched = tm.build_schedule(old, w.tile_size)
        for _ in range(steps):
            tm.fill_boundary(old, geom, plan)
            tm.heat_step(new, old, geom, p, sched)
            old, new = new, old
        tm.fill_boundary(old, geom, plan)
        old.settle()
        old.reduce_sum()  # the reduction kernels run under the bands too
        got = old.to_global().cpu().numpy()
        assert g.check() == []
    want = heat_oracle(tm, w, glob, steps)
    assert np.array_equal(got, want)


@pytest.mark.parametrize("n,mgs,split", [(128, 64, True), (128, 64, False), (64, 32, True), (48, 24, False)])
def test_gsrb_stays_inside_its_allocations(tm, n, mgs, split):
    sweeps = 3
    w = tm.CONFIGS["C4"].scaled(n, mgs, sweeps)
    rhs_g = tm.make_init(w)
    geom = tm.Geometry(w.domain, (True, True, True), (w.dx,) * 3)
    ba = tm.BoxArray.chop(w.domain, w.max_grid_size)
    with GuardBands() as g:
        phi = tm.MultiFab(ba, 1, 1)
        rhs = tm.MultiFab(ba, 1, 0)
        rhs.from_global(rhs_g)
        tm.gsrb_solve(phi, rhs, geom, sweeps, fused=True, split=split)
        res = tm.residual_maxnorm(phi, rhs, geom)
        got = phi.to_global().cpu().numpy()[0]
        assert g.check() == []
    ref_phi, ref_res = orc.gsrb_periodic(np.zeros((n,) * 3), rhs_g[0], sweeps, w.dx * w.dx)
    assert np.array_equal(got, ref_phi)
    assert res == ref_res


@pytest.mark.parametrize("n,mgs,fused", [(64, 32, True), (128, 64, True), (64, 32, False)])
def test_wide4_stays_inside_its_allocations(tm, n, mgs, fused):
    steps = 3
    w = dataclasses.replace(tm.CONFIGS["C1"].scaled(n, mgs, steps), nghost=4)
    glob = tm.make_init(w)
    geom = tm.Geometry(w.domain, (True, True, True), (w.dx,) * 3)
    ba = tm.BoxArray.chop(w.domain, w.max_grid_size)
    dt = tm.wide4_stable_dt(1.0, (w.dx,) * 3)
    coeffs = tm.derive_coeffs8()
    with GuardBands() as g:
        mf = tm.MultiFab(ba, 1, 4)
        mf.from_global(glob)
        r = tm.Wide4Runner(mf, geom, 1.0, dt, coeffs, fused=fused, use_graph=False)
        got = r.advance(steps).to_global().cpu().numpy()[0]
        r.close()
        assert g.check() == []
    want = orc.wide4_periodic(glob[0], steps, coeffs.as_array(), (1.0 / w.dx ** 2,) * 3, dt)
    assert np.array_equal(got, want)


@pytest.mark.parametrize("n,mgs,ranks,ncomp,nghost", [(128, 32, 8, 1, 1), (64, 32, 2, 2, 2)])
def test_peer_march_stays_inside_every_ranks_allocations(tm, n, mgs, ranks, ncomp, nghost):
    """Peer halos with emulated ranks on one GPU (tests/test_gpu_peer.py): every
    rank's fields, halo buffers and peer tables are guarded, so a march that
    reads a peer's face must not write outside its own rank's storage either."""
    import torch

    from paper_1604_03570_b200.boxarray import DistributionMapping
    from paper_1604_03570_b200.peer import PeerFused

    steps = 4
    w = tm.CONFIGS["C5"].scaled(n, mgs, steps)
    geom = tm.Geometry(w.domain, (True, True, True), (w.dx,) * 3)
    ba = tm.BoxArray.chop(w.domain, mgs)
    glob = np.random.default_rng(11).standard_normal((ncomp,) + tuple(w.domain.extents[::-1]))
    dm = DistributionMapping(ba, ranks)
    p = tm.HeatParams.stable(1.0, geom.dx)
    with GuardBands() as g:
        pairs = []
        for r in range(ranks):
            a = tm.MultiFab(ba, ncomp, nghost, dm=dm, rank=r)
            a.from_global(glob)
            pairs.append((a, a.clone_empty()))
        fields = {r: (pr[0].ptr, pr[1].ptr) for r, pr in enumerate(pairs)}
        pfs = [PeerFused(a, b, geom, fields) for a, b in pairs]
        for (a, _), pf in zip(pairs, pfs):
            pf.prime(a)
        for k in range(steps):
            for (a, b), pf in zip(pairs, pfs):
                old, new = (a, b) if k % 2 == 0 else (b, a)
                pf.step(new, old, p, reverse=k % 2 == 1)
        torch.cuda.synchronize()
        got = sum(pr[steps % 2].to_global().cpu().numpy() for pr in pairs)
        assert g.check() == []
    c = p.coefficients()
    assert np.array_equal(got, orc.heat_periodic(glob, steps, c[:3], c[3]))
