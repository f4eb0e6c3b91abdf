"""Run BASELINE configs C1-C5 at full size on one GPU: rates + size-independent
parity properties.

    python tools/run_configs.py [C1 C2 C3 C4 C5] [--oracle]

Per heat config: fused and unfused step paths (independent kernels) must agree
bit for bit; each component's sum is conserved (flux form) to 1e-11
relative; C1/C2 checksums equal the reference's (golden / SURVEY value).
C4 (GSRB): residual decreases; with --oracle the final phi and residual are
compared bit for bit with the whole-domain numpy restatement.  With --oracle
the heat configs also run the reference path restated in C (oracle/tm_oracle.c,
OpenMP) at full size and compare every valid cell and each component's serial
checksum bit for bit with the device result.
Prints one JSON line per config.
"""

import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1604_03570_b200 as tm  # noqa: E402
from paper_1604_03570_b200.runner import HeatRunner  # noqa: E402

REF_SUMS = {"C2": 16870634.63599003}  # SURVEY.md §8a a10 (reference run)


def ev_time(fn):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) * 1e-3


def oracle_heat(name, w, glob, ba, geom, plan, p):
    """The reference path restated in C (oracle/tm_oracle.c: tag FillBoundary +
    per-component heat_tiles, OpenMP over all host threads) at full size.
    Returns the host MultiFab holding the final field."""
    from oracle import oracle as orc
    from paper_1604_03570_b200.box import decompose

    nt = orc.max_threads()
    valids = list(ba)
    old = orc.HostMF(valids, w.ncomp, w.nghost)
    old.from_global(glob)
    new = orc.HostMF(valids, w.ncomp, w.nghost)
    tags = orc.tags_array(plan.tags)
    tiles = orc.tiles_array([(u, t) for u in range(len(valids)) for t in decompose(valids[u], w.tile_size)])
    c = p.coefficients()
    for _ in range(w.steps):
        orc.fill_boundary(old, tags, nt)
        orc.heat_step(new, old, tiles, c[:3], c[3], nt)
        old, new = new, old
    del new
    return old, nt


def compare_with_oracle(res, out_global, host, ba, w):
    """Bit-compare every valid cell of the device result with the oracle's, box by box."""
    from oracle import oracle as orc

    bad = 0
    maxdiff = 0.0
    for u, v in enumerate(ba):
        sl = tuple(slice(v.lo[d], v.hi[d] + 1) for d in (2, 1, 0))
        for c in range(w.ncomp):
            d = out_global[(c,) + sl].cpu().numpy()
            h = host.valid_view(u, c).transpose(2, 1, 0)
            if not np.array_equal(d, h):
                bad += 1
                maxdiff = max(maxdiff, float(np.max(np.abs(d - h))))
    res["phi_equals_oracle"] = bad == 0
    res["oracle_mismatched_box_comps"] = bad
    if bad:
        res["oracle_max_abs_diff"] = maxdiff
    res["oracle_sums"] = [orc.reduce_sum(host, c) for c in range(w.ncomp)]
    res["sums_equal_oracle"] = res["oracle_sums"] == res["fused_sums"]


def heat_config(name, oracle=False):
    w = tm.CONFIGS[name]
    t0 = time.time()
    glob = tm.make_init(w)
    t_init = time.time() - t0
    geom = tm.Geometry(w.domain, (True, True, True), (w.dx,) * 3)
    ba = tm.BoxArray.chop(w.domain, w.max_grid_size)
    t0 = time.time()
    mf = tm.MultiFab(ba, w.ncomp, w.nghost)
    plan = tm.build_fill_plan(mf, geom)
    t_plan = time.time() - t0
    g = torch.from_numpy(glob).cuda()
    host = None
    if oracle:
        t0 = time.time()
        host, nt = oracle_heat(name, w, glob, ba, geom, plan, tm.HeatParams.stable(1.0, geom.dx))
        res_oracle = {"oracle_s": time.time() - t0, "oracle_threads": nt}
    del glob
    sums0 = [float(torch.sum(g[c]).item()) for c in range(w.ncomp)]
    p = tm.HeatParams.stable(1.0, geom.dx)
    sched = tm.build_schedule(mf, w.tile_size)
    res = {"config": name, "cells": w.cells * w.ncomp, "steps": w.steps, "init_s": t_init, "plan_s": t_plan}
    finals = {}
    for fused in (True, False):
        mf.from_global(g)
        r = HeatRunner(mf, geom, p, sched, plan, fused=fused)
        r.advance(2)  # warm + capture
        mf.from_global(g)
        r.reset()
        secs = ev_time(lambda: r.advance(w.steps))
        out = r.current
        key = "fused" if fused else "unfused"
        res[key + "_rate"] = w.cells * w.ncomp * w.steps / secs
        res[key + "_ms_per_step"] = secs / w.steps * 1e3
        finals[key] = out.to_global()
        res[key + "_sums"] = [out.reduce_sum(c) for c in range(w.ncomp)]
        del r
        torch.cuda.empty_cache()
    res["fused_equals_unfused"] = bool(torch.equal(finals["fused"], finals["unfused"]))
    if host is not None:
        res.update(res_oracle)
        compare_with_oracle(res, finals["fused"], host, ba, w)
    res["conservation_max_rel"] = max(abs(s - s0) / abs(s0) for s, s0 in zip(res["fused_sums"], sums0))
    if name in REF_SUMS:
        res["checksum_equals_reference"] = res["fused_sums"][0] == REF_SUMS[name]
    if name == "C1":
        z = np.load(os.path.join(os.path.dirname(__file__), "..", "tests", "golden", "heat.npz"))
        res["checksum_equals_reference"] = res["fused_sums"][0] == float(z["C1/sums"][-1][0])
    return res


def gsrb_config(oracle: bool):
    w = tm.CONFIGS["C4"]
    rhs_g = tm.make_init(w)
    geom = tm.Geometry(w.domain, (True, True, True), (w.dx,) * 3)
    ba = tm.BoxArray.chop(w.domain, w.max_grid_size)
    phi = tm.MultiFab(ba, 1, 1)
    rhs = tm.MultiFab(ba, 1, 0)
    rhs.from_global(rhs_g)
    plan = tm.build_fill_plan(phi, geom)
    sched = tm.build_schedule(phi, w.tile_size)
    tm.gsrb_solve(phi, rhs, geom, 2, sched, plan, fused=True)  # warm (plans, halo tables, graph)
    tm.gsrb_solve(phi, rhs, geom, 2, sched, plan, fused=True, split=False)
    tm.gsrb_sweep(phi, rhs, geom, sched, plan)
    phi.fill(0.0)
    r0 = tm.residual_maxnorm(phi, rhs, geom, sched)
    res = {"config": "C4", "cells": w.cells, "sweeps": w.steps, "residual0": r0}
    finals = {}
    for key, fused, split in (("fused", True, None), ("inplace", True, False), ("unfused", False, False)):
        phi.fill(0.0)
        secs = ev_time(lambda: tm.gsrb_solve(phi, rhs, geom, w.steps, sched, plan, fused=fused, split=split))
        res[key + "_rate"] = w.cells * w.steps / secs
        res[key + "_ms_per_sweep"] = secs / w.steps * 1e3
        res[key + "_residual"] = tm.residual_maxnorm(phi, rhs, geom, sched)
        finals[key] = phi.to_global()
    res["fused_equals_unfused"] = bool(torch.equal(finals["fused"], finals["unfused"]) and
                                       torch.equal(finals["inplace"], finals["unfused"]))
    r1 = res["fused_residual"]
    res["residual_decreased"] = r1 < r0
    if oracle:
        from oracle import oracle as orc

        ref_phi, ref_res = orc.gsrb_periodic(np.zeros((w.n,) * 3), rhs_g[0], w.steps, w.dx * w.dx)
        res["phi_equals_oracle"] = bool(np.array_equal(phi.to_global().cpu().numpy()[0], ref_phi))
        res["residual_equals_oracle"] = r1 == ref_res
    return res


def main():
    names = [a for a in sys.argv[1:] if a.startswith("C")] or ["C1", "C2", "C3", "C4", "C5"]
    torch.cuda.set_device(0)
    for n in names:
        t0 = time.time()
        res = gsrb_config("--oracle" in sys.argv) if n == "C4" else heat_config(n, "--oracle" in sys.argv)
        res["wall_s"] = time.time() - t0
        print(json.dumps(res), flush=True)
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
