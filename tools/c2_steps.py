"""Eager C2 step loop for profiling (ncu): python tools/c2_steps.py [steps] [--zmerge] [--config C2]."""

import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_1604_03570_b200 as tm  # noqa: E402


def main():
    steps = int(sys.argv[1]) if len(sys.argv) > 1 and sys.argv[1].isdigit() else 10
    zmerge = "--zmerge" in sys.argv
    cfg = sys.argv[sys.argv.index("--config") + 1] if "--config" in sys.argv else "C2"
    w = tm.CONFIGS[cfg]
    geom = tm.Geometry(w.domain, (True, True, True), (w.dx,) * 3)
    ba = tm.BoxArray.chop(w.domain, w.max_grid_size)
    old = tm.MultiFab(ba, w.ncomp, w.nghost)
    old.from_global(tm.make_init(w))
    new = old.clone_empty()
    plan = tm.build_fill_plan(old, geom)
    sched = tm.build_schedule(old, w.tile_size)
    p = tm.HeatParams.stable(1.0, geom.dx)
    for _ in range(steps):
        tm.fill_boundary(old, geom, plan)
        tm.heat_step(new, old, geom, p, sched, zmerge=zmerge)
        old, new = new, old
    torch.cuda.synchronize()
    print("done", cfg, steps, "sum", old.reduce_sum())


if __name__ == "__main__":
    main()
