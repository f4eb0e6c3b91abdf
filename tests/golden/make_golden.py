"""Generate the golden fixtures in tests/golden/ by running the REFERENCE.

Run in the build container (the only place /root/reference exists):

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

Everything here drives the unmodified reference package ``tilemesh``
(``/root/reference/pkg/src/tilemesh``) through its public API:
``BoxArray.chop`` / ``MultiFab`` / ``build_fill_plan`` / ``fill_boundary``
/ ``heat_step`` / ``reduce_sum``.  For ncomp > 1 (configs C3, C5) it
drives ``compiled.heat_tiles`` once per component with ``comp(c)`` views,
exactly as ``heat_step`` does for component 0 (kernels.py:199-214),
because ``heat_step`` rejects ncomp != 1 (kernels.py:147-150).

Inputs come from ``paper_1604_03570_b200.configs.make_init`` (seeded,
host-independent).  Outputs:

* plans.npz  -- reference tags and exec_tags for several layouts
* fills.npz  -- reference FillBoundary results (sentinel + linear field)
* heat.npz   -- sha256 of initial/final global arrays, reduce_sum values,
                and full final arrays for the small cases
* wide4.npz  -- reference wide4_step runs (nghost 4): the coefficient and dt
                bits used, per-step reduce_sum, sha256 / full final arrays

* regional.npz -- REGIONAL-layout units, plans, a fill, heat / wide4 runs
* plotfile.npz -- reference write_plotfile output (HEADER + unit fab bytes)

``python tests/golden/make_golden.py wide4`` (or ``regional``, ...) regenerates one file.
"""

from __future__ import annotations

import hashlib
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.abspath(os.path.join(HERE, "..", "..")))

import tilemesh  # noqa: E402  (the reference)
from tilemesh import compiled  # noqa: E402
from tilemesh.box import Box  # noqa: E402
from tilemesh.iterator import build_schedule  # noqa: E402
from tilemesh.kernels import HeatParams, heat_step  # noqa: E402
from tilemesh.level import BoxArray, Geometry, MultiFab, build_fill_plan, fill_boundary  # noqa: E402

from paper_1604_03570_b200.configs import CONFIGS, make_init  # noqa: E402

SENTINEL = -12345.6789


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a, dtype=np.float64).tobytes()).hexdigest()


def tag_rows(tags):
    out = np.empty((len(tags), 17), dtype=np.int64)
    for n, t in enumerate(tags):
        out[n] = [t.dst_unit, *t.dst_box.lo, *t.dst_box.hi, t.src_unit, *t.src_box.lo, *t.src_box.hi, *t.shift]
    return out


def random_layout(rng):
    dom_hi = tuple(int(v) for v in rng.integers(3, 12, 3))
    domain = Box((0, 0, 0), dom_hi)
    mgs = tuple(int(v) for v in rng.integers(2, 9, 3))
    cands = BoxArray.chop(domain, mgs).boxes
    keep = [b for b in cands if rng.random() < 0.7] or [cands[0]]
    periodic = tuple(bool(v) for v in rng.integers(0, 2, 3))
    ng = int(rng.choice([1, 2, 4]))
    return domain, keep, periodic, ng


def plan_cases():
    cases = []
    c1 = Box((0, 0, 0), (63, 63, 63))
    cases.append(("c1_layout", c1, BoxArray.chop(c1, 32).boxes, (True, True, True), 1))
    d32 = Box((0, 0, 0), (31, 31, 31))
    cases.append(("c5_like_32_mgs16_ng2", d32, BoxArray.chop(d32, 16).boxes, (True, True, True), 2))
    d3 = Box((0, 0, 0), (2, 2, 2))
    cases.append(("wrap_wider_than_domain", d3, [d3], (True, True, True), 4))
    d8 = Box((0, 0, 0), (7, 7, 7))
    cases.append(("nonperiodic_z", d8, [d8], (True, True, False), 1))
    d16 = Box((0, 0, 0), (15, 7, 7))
    cases.append(("abutting_two", d16, [Box((0, 0, 0), (7, 7, 7)), Box((8, 0, 0), (15, 7, 7))],
                  (True, False, True), 2))
    uneven = Box((0, 0, 0), (20, 13, 9))
    cases.append(("uneven_chop", uneven, BoxArray.chop(uneven, (8, 6, 5)).boxes, (True, True, True), 1))
    d64 = Box((0, 0, 0), (63, 63, 63))
    cases.append(("split_single_64_ng1", d64, [d64], (True, True, True), 1))
    d48 = Box((0, 0, 0), (47, 47, 47))
    cases.append(("split_48_ng2", d48, [d48], (True, True, True), 2))
    d40 = Box((0, 0, 0), (79, 39, 39))
    cases.append(("split_two_ng3_partial_periodic", d40, BoxArray.chop(d40, 40).boxes, (True, False, True), 3))
    rng = np.random.default_rng(42)
    for t in range(12):
        dom, keep, per, ng = random_layout(rng)
        cases.append((f"random_{t}", dom, keep, per, ng))
    c2 = Box((0, 0, 0), (255, 255, 255))
    cases.append(("c2_layout", c2, BoxArray.chop(c2, 64).boxes, (True, True, True), 1))
    return cases


def f_linear(i, j, k):
    return i + 10.0 * j + 100.0 * k


def make_plans_and_fills():
    plans = {}
    fills = {}
    meta = []
    for name, dom, boxes, per, ng in plan_cases():
        geom = Geometry(dom, per)
        ba = BoxArray(boxes)
        mf = MultiFab(ba, 1, ng)
        plan = build_fill_plan(mf, geom)
        plans[name + "/tags"] = tag_rows(plan.tags)
        plans[name + "/exec"] = tag_rows(plan.exec_tags)
        plans[name + "/valids"] = np.array([[*b.lo, *b.hi] for b in boxes], dtype=np.int64)
        plans[name + "/domain"] = np.array([*dom.lo, *dom.hi], dtype=np.int64)
        plans[name + "/periodic"] = np.array(per, dtype=np.int64)
        plans[name + "/nghost"] = np.array([ng], dtype=np.int64)
        meta.append(name)
        if len(boxes) <= 64 and name != "c2_layout":
            mf.fill(SENTINEL)
            mf.set_from_function(f_linear)
            fill_boundary(mf, geom, plan)
            fills[name] = np.concatenate([u.fab.flat for u in mf.units])
        print(f"plan {name}: {len(plan.tags)} tags, {len(plan.exec_tags)} exec", flush=True)
    plans["names"] = np.array(meta)
    np.savez_compressed(os.path.join(HERE, "plans.npz"), **plans)
    np.savez_compressed(os.path.join(HERE, "fills.npz"), **fills)


def set_global(mf, glob):
    for u in mf.units:
        lo, hi = u.valid.lo, u.valid.hi
        for c in range(mf.ncomp):
            blk = glob[c, lo[2]:hi[2] + 1, lo[1]:hi[1] + 1, lo[0]:hi[0] + 1]
            u.fab.view(u.valid, c, 1)[..., 0] = blk.transpose(2, 1, 0)


def get_global(mf, n):
    out = np.zeros((mf.ncomp, n, n, n))
    for u in mf.units:
        lo, hi = u.valid.lo, u.valid.hi
        for c in range(mf.ncomp):
            out[c, lo[2]:hi[2] + 1, lo[1]:hi[1] + 1, lo[0]:hi[0] + 1] = \
                u.fab.view(u.valid, c, 1)[..., 0].transpose(2, 1, 0)
    return out


def run_reference(w, steps, glob):
    """Reference step loop (bench._timed_loop shape): fill; step; swap."""
    dom = w.domain
    geom = Geometry(dom, (True, True, True), (w.dx,) * 3)
    ba = BoxArray.chop(dom, w.max_grid_size)
    old = MultiFab(ba, w.ncomp, w.nghost)
    set_global(old, glob)
    new = old.clone_empty()
    plan = build_fill_plan(old, geom)
    sched = build_schedule(old, w.tile_size)
    params = HeatParams.stable(1.0, geom.dx)
    sums = []
    for _ in range(steps):
        fill_boundary(old, geom, plan)
        if w.ncomp == 1:
            heat_step(new, old, geom, params, sched)
        else:
            dxi = tuple(1.0 / d for d in params.dx)
            dtD = params.diffusivity * params.dt
            tx, ty, tz = sched.max_tile_extents()
            fx = np.empty((tx + 1, ty, tz), order="F")
            fy = np.empty((tx, ty + 1, tz), order="F")
            fz = np.empty((tx, ty, tz + 1), order="F")
            for unit, tiles in sched.worker_runs(1, 0):
                uo = old.units[unit].fab
                un = new.units[unit].fab
                au = uo.abox.lo
                for c in range(w.ncomp):
                    compiled.heat_tiles(un.comp(c), uo.comp(c), au[0], au[1], au[2],
                                        fx, fy, fz, tiles, dxi[0], dxi[1], dxi[2], dtD)
        old, new = new, old
        sums.append([old.reduce_sum(c) for c in range(w.ncomp)])
    return old, np.array(sums)


def make_heat():
    out = {}
    cases = [
        ("C1", CONFIGS["C1"], CONFIGS["C1"].steps, True),
        ("small16", CONFIGS["C1"].scaled(16, 8, 5), 5, True),
        ("c3_like", CONFIGS["C3"].scaled(32, 16, 3), 3, False),
        ("c5_like", CONFIGS["C5"].scaled(64, 16, 2), 2, False),
        ("uneven", CONFIGS["C1"].scaled(30, 13, 4), 4, True),
    ]
    for name, w, steps, keep_full in cases:
        glob = make_init(w)
        mf, sums = run_reference(w, steps, glob)
        fin = get_global(mf, w.n)
        out[name + "/init_sha"] = np.array(sha(glob))
        out[name + "/final_sha"] = np.array(sha(fin))
        out[name + "/sums"] = sums
        out[name + "/max"] = np.array([mf.reduce_max(c) for c in range(w.ncomp)])
        out[name + "/min"] = np.array([mf.reduce_min(c) for c in range(w.ncomp)])
        out[name + "/meta"] = np.array(json.dumps(dict(n=w.n, mgs=w.max_grid_size, ng=w.nghost,
                                                       nc=w.ncomp, tile=list(w.tile_size), steps=steps,
                                                       init=w.init)))
        if keep_full and w.n <= 32:
            out[name + "/final"] = fin
        print(f"heat {name}: sum {sums[-1]} sha {sha(fin)[:16]}", flush=True)
    np.savez_compressed(os.path.join(HERE, "heat.npz"), **out)


WIDE4_CASES = [  # (name, n, max_grid_size, steps, keep full field)
    ("w16_single", 16, 16, 3, True),
    ("w32_boxes", 32, 16, 3, True),
    ("w32_small_boxes", 32, 8, 2, False),
    ("w30_uneven", 30, 13, 2, True),
    ("w64_c2like", 64, 32, 2, False),
]


def make_wide4():
    """Reference wide4 runs (kernels.wide4_step): fill;
    step; swap, nghost 4, fully periodic, seeded gauss+noise init."""
    import dataclasses

    from tilemesh.kernels import derive_coeffs8, wide4_stable_dt, wide4_step

    out = {}
    coeffs = derive_coeffs8()
    out["coeffs"] = coeffs.as_array()
    for name, n, mgs, steps, keep_full in WIDE4_CASES:
        w = dataclasses.replace(CONFIGS["C1"].scaled(n, mgs, steps), nghost=4)
        glob = make_init(w)
        dom = w.domain
        geom = Geometry(dom, (True, True, True), (w.dx,) * 3)
        old = MultiFab(BoxArray.chop(dom, w.max_grid_size), 1, 4)
        set_global(old, glob)
        new = old.clone_empty()
        plan = build_fill_plan(old, geom)
        sched = build_schedule(old, w.tile_size)
        dt = wide4_stable_dt(1.0, geom.dx)
        sums = []
        for _ in range(steps):
            fill_boundary(old, geom, plan)
            wide4_step(new, old, geom, 1.0, dt, sched, 1, coeffs)
            old, new = new, old
            sums.append(old.reduce_sum(0))
        fin = get_global(old, n)
        out[name + "/init_sha"] = np.array(sha(glob))
        out[name + "/final_sha"] = np.array(sha(fin))
        out[name + "/sums"] = np.array(sums)
        out[name + "/dt"] = np.array(dt)
        out[name + "/meta"] = np.array(json.dumps(dict(n=n, mgs=mgs, steps=steps)))
        if keep_full:
            out[name + "/final"] = fin
        print(f"wide4 {name}: sum {sums[-1]} sha {sha(fin)[:16]}", flush=True)
    np.savez_compressed(os.path.join(HERE, "wide4.npz"), **out)


REGIONAL_CASES = [  # (name, domain hi, max_grid_size or None, region, nghost, periodic, kernel, steps)
    ("r24_one_grid", (23, 23, 23), None, (12, 12, 12), 1, (True, True, True), "heat", 5),
    ("r32_uneven", (31, 31, 31), 16, (8, 16, 5), 2, (True, True, True), "heat", 3),
    ("r_two_grids", (15, 7, 7), 8, (4, 4, 4), 2, (True, False, True), "fill", 0),
    ("r32_wide4", (31, 31, 31), None, (16, 16, 16), 4, (True, True, True), "wide4", 2),
]


def make_regional():
    """Reference runs on the REGIONAL layout (level.py:116-133; SURVEY.md §8f
    row 3): the unit list, the FillBoundary plan over regions, a fill of a
    linear field, and heat / wide4 runs with their reduce_sum values."""
    from tilemesh.kernels import derive_coeffs8, wide4_stable_dt, wide4_step
    from tilemesh.level import REGIONAL

    out = {}
    for name, hi, mgs, region, ng, per, kernel, steps in REGIONAL_CASES:
        dom = Box((0, 0, 0), hi)
        n = hi[0] + 1
        geom = Geometry(dom, per, (1.0 / n,) * 3)
        ba = BoxArray.chop(dom, (mgs,) * 3) if mgs else BoxArray([dom])
        mf = MultiFab(ba, 1, ng, REGIONAL, region)
        plan = build_fill_plan(mf, geom)
        out[name + "/units"] = np.array([[u.grid, *u.valid.lo, *u.valid.hi] for u in mf.units], dtype=np.int64)
        out[name + "/tags"] = tag_rows(plan.tags)
        out[name + "/meta"] = np.array(json.dumps(dict(hi=hi, mgs=mgs, region=region, ng=ng, periodic=per,
                                                       kernel=kernel, steps=steps)))
        if kernel == "fill":
            mf.fill(SENTINEL)
            mf.set_from_function(f_linear)
            fill_boundary(mf, geom, plan)
            out[name + "/fill"] = np.concatenate([u.fab.flat for u in mf.units])
            print(f"regional {name}: {len(mf.units)} units, {len(plan.tags)} tags", flush=True)
            continue
        w = CONFIGS["C1"].scaled(n, n, steps)
        glob = make_init(w)
        set_global(mf, glob)
        new = mf.clone_empty()
        sched = build_schedule(mf, (8, 8, 8))
        sums = []
        old = mf
        for _ in range(steps):
            fill_boundary(old, geom, plan)
            if kernel == "heat":
                heat_step(new, old, geom, HeatParams.stable(1.0, geom.dx), sched)
            else:
                wide4_step(new, old, geom, 1.0, wide4_stable_dt(1.0, geom.dx), sched, 1, derive_coeffs8())
            old, new = new, old
            sums.append(old.reduce_sum(0))
        fin = get_global(old, n)
        out[name + "/init_sha"] = np.array(sha(glob))
        out[name + "/final_sha"] = np.array(sha(fin))
        out[name + "/sums"] = np.array(sums)
        print(f"regional {name}: {len(mf.units)} units, {len(plan.tags)} tags, sum {sums[-1]}", flush=True)
    np.savez_compressed(os.path.join(HERE, "regional.npz"), **out)


def make_plotfiles():
    """Reference plotfile-lite dumps (level.py:326-345, fab.py:86-90): the
    HEADER text and every unit file's bytes."""
    import tempfile

    from tilemesh.level import REGIONAL, write_plotfile

    out = {}
    cases = [
        ("p_two_comp", Box((0, 0, 0), (5, 5, 5)), None, 2, 1, None, False),
        ("p_chop_ng2", Box((0, 0, 0), (11, 11, 11)), 6, 1, 2, None, True),
        ("p_regional", Box((0, 0, 0), (15, 15, 15)), None, 1, 1, (8, 8, 16), True),
    ]
    for name, dom, mgs, nc, ng, region, fill in cases:
        n = dom.hi[0] + 1
        geom = Geometry(dom, (True, True, True), (1.0 / n,) * 3)
        ba = BoxArray.chop(dom, (mgs,) * 3) if mgs else BoxArray([dom])
        mf = MultiFab(ba, nc, ng, REGIONAL if region else "contiguous", region)
        for c in range(nc):
            mf.set_from_function(lambda i, j, k, c=c: f_linear(i, j, k) + 1000.0 * c + 0.125, comp=c)
        if fill:
            fill_boundary(mf, geom)
        with tempfile.TemporaryDirectory() as d:
            write_plotfile(mf, geom, d)
            out[name + "/HEADER"] = np.array(open(os.path.join(d, "HEADER")).read())
            files = sorted(f for f in os.listdir(d) if f.endswith(".fab"))
            out[name + "/files"] = np.array(files)
            for f in files:
                out[name + "/" + f] = np.frombuffer(open(os.path.join(d, f), "rb").read(), dtype=np.uint8)
        out[name + "/meta"] = np.array(json.dumps(dict(hi=dom.hi, mgs=mgs, nc=nc, ng=ng, region=region,
                                                       fill=fill)))
        print(f"plotfile {name}: {len(files)} unit files", flush=True)
    np.savez_compressed(os.path.join(HERE, "plotfile.npz"), **out)


if __name__ == "__main__":
    print("reference:", tilemesh.__file__)
    which = sys.argv[1:] or ["plans", "heat", "wide4", "regional", "plotfile"]
    if "plans" in which:
        make_plans_and_fills()
    if "heat" in which:
        make_heat()
    if "wide4" in which:
        make_wide4()
    if "regional" in which:
        make_regional()
    if "plotfile" in which:
        make_plotfiles()
