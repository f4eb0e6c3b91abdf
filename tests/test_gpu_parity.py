"""Device path (libtilemesh_b200.so through the public API) vs the oracle and
the reference's golden fixtures.  Bit-exact throughout: ghost fills are
copies and the heat/GSRB arithmetic follows the oracle operation for
operation with no FMA."""

import hashlib
import json
import os
import warnings

import numpy as np
import pytest

from oracle import oracle as orc

pytestmark = pytest.mark.gpu

G = os.path.join(os.path.dirname(__file__), "golden")
SENTINEL = -12345.6789


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a, dtype=np.float64).tobytes()).hexdigest()


def f_linear(i, j, k):
    return i + 10.0 * j + 100.0 * k


@pytest.fixture(scope="module")
def tm():
    import torch

    import paper_1604_03570_b200 as tm

    torch.cuda.set_device(0)
    return tm


def plan_case(z, name):
    from paper_1604_03570_b200 import Box

    v = z[name + "/valids"]
    d = z[name + "/domain"]
    return ([Box(r[:3], r[3:]) for r in v], Box(d[:3], d[3:]),
            tuple(bool(p) for p in z[name + "/periodic"]), int(z[name + "/nghost"][0]))


def device_flat(mf):
    return np.concatenate([u.fab.to_numpy().ravel(order="F") for u in mf.units])


def test_fill_boundary_matches_reference_golden(tm):
    z = np.load(os.path.join(G, "plans.npz"))
    fills = np.load(os.path.join(G, "fills.npz"))
    for name in fills.files:
        valids, dom, per, ng = plan_case(z, name)
        geom = tm.Geometry(dom, per)
        mf = tm.MultiFab(tm.BoxArray(valids), 1, ng)
        mf.fill(SENTINEL)
        mf.set_from_function(f_linear)
        tm.fill_boundary(mf, geom)
        assert np.array_equal(device_flat(mf), fills[name]), name
        tm.fill_boundary(mf, geom)  # idempotent
        assert np.array_equal(device_flat(mf), fills[name]), name


def test_fill_boundary_randomized_multicomp(tm):
    rng = np.random.default_rng(77)
    for trial in range(40):
        hi = tuple(int(v) for v in rng.integers(3, 16, 3))
        dom = tm.Box((0, 0, 0), hi)
        cands = tm.BoxArray.chop(dom, tuple(int(v) for v in rng.integers(2, 9, 3))).boxes
        keep = [b for b in cands if rng.random() < 0.7] or cands[:1]
        per = tuple(bool(v) for v in rng.integers(0, 2, 3))
        ng = int(rng.choice([1, 2, 4]))
        nc = int(rng.choice([1, 2, 3]))
        geom = tm.Geometry(dom, per)
        mf = tm.MultiFab(tm.BoxArray(keep), nc, ng)
        h = orc.HostMF(keep, nc, ng, fill=SENTINEL)
        mf.fill(SENTINEL)
        vals = rng.random(sum(v.ncells for v in keep) * nc)
        pos = 0
        for u, v in enumerate(keep):
            for c in range(nc):
                blk = vals[pos:pos + v.ncells].reshape(v.extents, order="F")
                pos += v.ncells
                h.valid_view(u, c)[...] = blk
                import torch

                mf.fab(u).view(v, c, 1)[..., 0].copy_(torch.from_numpy(np.ascontiguousarray(blk)))
        plan = tm.build_fill_plan(mf, geom)
        tm.fill_boundary(mf, geom, plan)
        orc.fill_boundary(h, plan.tags)
        assert np.array_equal(device_flat(mf), h.buf), trial


def workload_from_meta(meta):
    from paper_1604_03570_b200.configs import Workload

    m = json.loads(str(meta))
    return Workload("g", m["n"], m["mgs"], m["ng"], m["nc"], tuple(m["tile"]), m["steps"], "heat", m["init"])


def run_device(tm, w, steps, glob, tiling=None, zmerge=False, sums=None):
    geom = tm.Geometry(w.domain, (True, True, True), (w.dx,) * 3)
    ba = tm.BoxArray.chop(w.domain, w.max_grid_size)
    old = tm.MultiFab(ba, w.ncomp, w.nghost)
    old.from_global(glob)
    new = old.clone_empty()
    plan = tm.build_fill_plan(old, geom)
    sched = tm.build_schedule(old, w.tile_size if tiling is None else tiling)
    p = tm.HeatParams.stable(1.0, geom.dx)
    for _ in range(steps):
        tm.fill_boundary(old, geom, plan)
        tm.heat_step(new, old, geom, p, sched, zmerge=zmerge)
        old, new = new, old
        if sums is not None:
            sums.append([old.reduce_sum(c) for c in range(w.ncomp)])
    return old


def test_heat_matches_reference_golden(tm):
    z = np.load(os.path.join(G, "heat.npz"))
    names = sorted({k.split("/")[0] for k in z.files})
    for name in names:
        w = workload_from_meta(z[name + "/meta"])
        glob = tm.make_init(w)
        assert sha(glob) == str(z[name + "/init_sha"])
        sums = []
        mf = run_device(tm, w, w.steps, glob, sums=sums)
        fin = mf.to_global().cpu().numpy()
        assert sha(fin) == str(z[name + "/final_sha"]), name
        assert np.array_equal(np.array(sums), z[name + "/sums"]), name  # device checksum is bit-exact
        assert [mf.reduce_max(c) for c in range(w.ncomp)] == list(z[name + "/max"])
        assert [mf.reduce_min(c) for c in range(w.ncomp)] == list(z[name + "/min"])


@pytest.mark.parametrize("tiling,zmerge,kernel", [("off", False, "auto"), ((16, 4, 4), False, "auto"),
                                                  ((1024, 8, 8), True, "auto"), ((5, 3, 7), False, "auto"),
                                                  ((64, 64, 1), True, "auto"), ((16, 4, 4), False, "march")])
def test_heat_tiling_invariance(tm, tiling, zmerge, kernel, monkeypatch):
    from paper_1604_03570_b200 import stencil

    monkeypatch.setattr(stencil, "SWEEP_KERNEL", kernel)
    w = tm.CONFIGS["C1"].scaled(48, 24, 4)
    glob = tm.make_init(w)
    got = run_device(tm, w, 4, glob, tiling=tiling, zmerge=zmerge).to_global().cpu().numpy()
    p = tm.HeatParams.stable(1.0, (w.dx,) * 3).coefficients()
    assert np.array_equal(got, orc.heat_periodic(glob, 4, p[:3], p[3]))


def test_heat_c3_shape_multicomp_two_ghosts(tm):
    # C3's shape (128^3 boxes, 4 comps, 2 ghosts, tile (1024,16,16)) at 256^3
    w = tm.CONFIGS["C3"].scaled(256, 128, 2)
    glob = tm.make_init(w)
    got = run_device(tm, w, 2, glob).to_global().cpu().numpy()
    p = tm.HeatParams.stable(1.0, (w.dx,) * 3).coefficients()
    assert np.array_equal(got, orc.heat_periodic(glob, 2, p[:3], p[3]))


def test_heat_big_untiled_box_is_split(tm):
    w = tm.CONFIGS["C1"].scaled(200, 200, 1)  # one 200^3 box, tiling off -> CTA blocks split in x and y
    glob = tm.make_init(w)
    got = run_device(tm, w, 1, glob, tiling="off").to_global().cpu().numpy()
    p = tm.HeatParams.stable(1.0, (w.dx,) * 3).coefficients()
    assert np.array_equal(got, orc.heat_periodic(glob, 1, p[:3], p[3]))


@pytest.mark.parametrize("kernel", ["auto", "tiled"])
def test_heat_c2_full_size(tm, kernel, monkeypatch):
    """heat_step at C2 size: auto routes to the column march, "tiled" keeps
    the tile kernel covered at full size."""
    from paper_1604_03570_b200 import stencil

    monkeypatch.setattr(stencil, "SWEEP_KERNEL", kernel)
    w = tm.CONFIGS["C2"]
    glob = tm.make_init(w)
    p = tm.HeatParams.stable(1.0, (w.dx,) * 3).coefficients()
    mf = run_device(tm, w, 3, glob)
    assert np.array_equal(mf.to_global().cpu().numpy(), orc.heat_periodic(glob, 3, p[:3], p[3]))
    if kernel == "tiled":
        return
    # full 100 steps: the flux form conserves the checksum
    s0 = float(np.sum(glob))
    mf = run_device(tm, w, w.steps, glob)
    assert abs(mf.reduce_sum() - s0) <= 1e-11 * abs(s0)


def test_heat_random_layouts_vs_oracle(tm):
    rng = np.random.default_rng(3)
    for trial in range(12):
        n = tuple(int(v) for v in rng.integers(8, 40, 3))
        dom = tm.Box((0, 0, 0), tuple(v - 1 for v in n))
        ba = tm.BoxArray.chop(dom, tuple(int(v) for v in rng.integers(5, 20, 3)))
        per = tuple(bool(v) for v in rng.integers(0, 2, 3))
        ng = int(rng.integers(1, 3))
        nc = int(rng.integers(1, 3))
        dx = tuple(float(v) for v in rng.uniform(0.5, 2.0, 3))
        geom = tm.Geometry(dom, per, dx)
        params = tm.HeatParams.stable(0.7, dx)
        ts = tuple(int(v) for v in rng.integers(3, 40, 3))
        old = tm.MultiFab(ba, nc, ng)
        new = tm.MultiFab(ba, nc, ng)
        glob = rng.random((nc, n[2], n[1], n[0]))
        old.from_global(glob)
        h_old = orc.HostMF(list(ba), nc, ng)
        h_new = orc.HostMF(list(ba), nc, ng)
        h_old.from_global(glob)
        plan = tm.build_fill_plan(old, geom)
        sched = tm.build_schedule(old, ts)
        tiles = orc.tiles_array([(e.unit, e.tile) for e in sched.entries])
        c = params.coefficients()
        for _ in range(3):
            tm.fill_boundary(old, geom, plan)
            tm.heat_step(new, old, geom, params, sched)
            orc.fill_boundary(h_old, plan.tags)
            orc.heat_step(h_new, h_old, tiles, c[:3], c[3])
            old, new = new, old
            h_old, h_new = h_new, h_old
        assert np.array_equal(device_flat(old), h_old.buf), trial


def test_heat_amplification_and_conservation(tm):
    n = 32
    dom = tm.Box((0, 0, 0), (n - 1,) * 3)
    geom = tm.Geometry(dom, dx=(1.0 / n,) * 3)
    params = tm.HeatParams.stable(1.0, geom.dx[0])
    mf = tm.MultiFab(tm.BoxArray([dom]), 1, 1)
    tm.init_cosine(mf, geom, offset=1.0)
    u0 = mf.grid_valid_array(0).copy()
    work = mf.clone_empty()
    sched = tm.build_schedule(mf, (16, 8, 8))
    cur, nxt = mf, work
    s_prev = cur.reduce_sum()
    for _ in range(10):
        tm.fill_boundary(cur, geom)
        tm.heat_step(nxt, cur, geom, params, sched)
        cur, nxt = nxt, cur
        s = cur.reduce_sum()
        assert abs(s - s_prev) <= 1e-11 * abs(s_prev)
        s_prev = s
    expect = 1.0 + tm.heat_amplification(params, geom) ** 10 * (u0 - 1.0)
    err = np.max(np.abs(cur.grid_valid_array(0) - expect)) / np.max(np.abs(expect))
    assert err <= 1e-13


def test_gsrb_and_residual_vs_oracle(tm):
    w = tm.CONFIGS["C4"].scaled(64, 32, 5)
    rhs_g = tm.make_init(w)
    geom = tm.Geometry(w.domain, (True, True, True), (w.dx,) * 3)
    ba = tm.BoxArray.chop(w.domain, w.max_grid_size)
    phi = tm.MultiFab(ba, 1, 1)
    rhs = tm.MultiFab(ba, 1, 0)
    rhs.from_global(rhs_g)
    plan = tm.build_fill_plan(phi, geom)
    sched = tm.build_schedule(phi, w.tile_size)
    res = []
    for _ in range(w.steps):
        tm.gsrb_sweep(phi, rhs, geom, sched, plan)
        res.append(tm.residual_maxnorm(phi, rhs, geom, sched))
    ref_phi, ref_res = orc.gsrb_periodic(np.zeros((w.n,) * 3), rhs_g[0], w.steps, w.dx * w.dx)
    assert np.array_equal(phi.to_global().cpu().numpy()[0], ref_phi)
    assert res[-1] == ref_res
    assert res[-1] < res[0]


def test_reductions_bitwise(tm):
    w = tm.CONFIGS["C5"].scaled(64, 16, 1)
    glob = tm.make_init(w)
    ba = tm.BoxArray.chop(w.domain, w.max_grid_size)
    mf = tm.MultiFab(ba, w.ncomp, w.nghost)
    mf.from_global(glob)
    h = orc.HostMF(list(ba), w.ncomp, w.nghost)
    h.from_global(glob)
    for c in range(w.ncomp):
        assert mf.reduce_sum(c) == orc.reduce_sum(h, c)
        assert mf.reduce_max(c) == orc.reduce_max(h, c)
        assert mf.reduce_min(c) == orc.reduce_min(h, c)
    mf.fill(-3.5)
    assert mf.reduce_max(0) == -3.5 and mf.reduce_min(1) == -3.5


def test_error_behaviour(tm):
    dom = tm.Box((0, 0, 0), (7, 7, 7))
    geom = tm.Geometry(dom, dx=(1 / 8,) * 3)
    ba = tm.BoxArray([dom])
    mf0 = tm.MultiFab(ba, 1, 0)
    with pytest.raises(ValueError):
        tm.heat_step(mf0.clone_empty(), mf0, geom, tm.HeatParams.stable(1.0, 1 / 8), tm.build_schedule(mf0))
    mf = tm.MultiFab(ba, 1, 1)
    with pytest.warns(UserWarning):
        tm.heat_step(mf.clone_empty(), mf, geom, tm.HeatParams(1.0, 1.0, geom.dx), tm.build_schedule(mf),
                     verify=True)
    with pytest.raises(ValueError):
        tm.heat_step(mf, mf, geom, tm.HeatParams.stable(1.0, 1 / 8))
    with pytest.raises(IndexError):
        mf.fab(0).at(9, 0, 0)
    with pytest.raises(ValueError):
        tm.MultiFab(tm.BoxArray([]), 1, 0).reduce_sum(0)
    with pytest.raises(ValueError):
        tm.MultiFab(ba, 1, -1)


def test_mfiter_facade(tm):
    dom = tm.Box((0, 0, 0), (31, 31, 31))
    ba = tm.BoxArray.chop(dom, 16)
    mf = tm.MultiFab(ba, 1, 2)
    count = 0
    for mfi in tm.MFIter(mf, tiling=True):
        bx = mfi.tilebox()
        mf[mfi].view(bx).fill_(float(mfi.index()))
        assert mf[mfi].view(mfi.growntilebox(2)).shape[:3] == mfi.growntilebox(2).extents
        count += 1
    assert count == 8 * 2 * 2  # (1024,8,8) tiles of 16^3 boxes
    for g in range(len(ba)):
        assert np.all(mf.grid_valid_array(g) == g)


def test_halo_pack_unpack_loopback(tm):
    """Two ranks' halo messages exchanged by device copies on one GPU (no
    kernels wait on each other): ghosts must equal the single-rank fill."""
    import torch

    from paper_1604_03570_b200.halo import HaloExchange
    from paper_1604_03570_b200.multifab import _device_fill

    w = tm.CONFIGS["C5"].scaled(64, 16, 1)
    glob = tm.make_init(w)
    geom = tm.Geometry(w.domain, (True, True, True), (w.dx,) * 3)
    ba = tm.BoxArray.chop(w.domain, w.max_grid_size)
    ref = tm.MultiFab(ba, w.ncomp, w.nghost)
    ref.from_global(glob)
    plan = tm.build_fill_plan(ref, geom)
    tm.fill_boundary(ref, geom, plan)
    for nranks in (2, 3):
        dm = tm.DistributionMapping(ba, nranks)
        mfs = [tm.MultiFab(ba, w.ncomp, w.nghost, dm=dm, rank=r) for r in range(nranks)]
        for m in mfs:
            m.from_global(glob)
        halos = [HaloExchange(m, plan) for m in mfs]
        s = torch.cuda.current_stream().cuda_stream
        for m, h in zip(mfs, halos):
            h.pack.run(h.sendbuf.data_ptr(), (0, 0, 0), m.ptr, m.layout.side(), s)
        for r, h in enumerate(halos):
            for peer, off, n in h.send_spans:
                dst = halos[peer]
                roff = next(o for p, o, k in dst.recv_spans if p == r)
                assert next(k for p, o, k in dst.recv_spans if p == r) == n
                dst.recvbuf[roff:roff + n].copy_(h.sendbuf[off:off + n])
        for m, h in zip(mfs, halos):
            copy, _ = _device_fill(m, plan)
            copy.run(m.ptr, m.layout.side(), m.ptr, m.layout.side(), s)
            h.unpack.run(m.ptr, m.layout.side(), h.recvbuf.data_ptr(), (0, 0, 0), s)
        for m in mfs:
            for u in m.local_units:
                assert torch.equal(m.fab(u).data, ref.fab(u).data), (nranks, u)


def test_overlap_split_is_a_partition_and_exact(tm):
    """Interior/boundary split used to overlap NCCL with the sweep: the two
    block sets partition the tiles, interior tiles never touch a ghost cell a
    remote rank fills, and interior-then-boundary sweeps equal one sweep."""
    import torch

    from paper_1604_03570_b200.halo import HaloExchange
    from paper_1604_03570_b200.multifab import split_blocks, sweep_blocks
    from paper_1604_03570_b200.stencil import heat_sweep_plan
    from paper_1604_03570_b200 import _native

    w = tm.CONFIGS["C2"].scaled(64, 32, 2)  # 8 boxes over 4 ranks: x-pairs, y/z neighbours remote
    geom = tm.Geometry(w.domain, (True, True, True), (w.dx,) * 3)
    ba = tm.BoxArray.chop(w.domain, w.max_grid_size)
    dm = tm.DistributionMapping(ba, 4)
    mf = tm.MultiFab(ba, 1, 1, dm=dm, rank=1)
    plan = tm.build_fill_plan(mf, geom)
    halo = HaloExchange(mf, plan)
    sched = tm.build_schedule(mf, w.tile_size)
    blocks = sweep_blocks(mf, sched.entries)
    inner, outer = split_blocks(mf, blocks, halo.remote_dst)
    assert len(inner) + len(outer) == len(blocks) and len(inner) > 0 and len(outer) > 0
    # single-rank: interior + boundary sweeps == full sweep, bit for bit
    one = tm.MultiFab(ba, 1, 1)
    one.from_global(tm.make_init(w))
    tm.fill_boundary(one, geom)
    a, b = one.clone_empty(), one.clone_empty()
    p = tm.HeatParams.stable(1.0, geom.dx)
    sched1 = tm.build_schedule(one, w.tile_size)
    tm.heat_step(a, one, geom, p, sched1)
    blocks1 = sweep_blocks(one, sched1.entries)
    fake_remote = {u: [bx for bx in halo.remote_dst.get(u, [])] for u in range(len(ba))}
    i1, o1 = split_blocks(one, blocks1, fake_remote)
    heat_sweep_plan(b, one, p, _native.SweepPlan(i1))
    heat_sweep_plan(b, one, p, _native.SweepPlan(o1))
    for u in one.local_units:
        v = one.units[u].valid
        assert torch.equal(a.fab(u).view(v), b.fab(u).view(v))
